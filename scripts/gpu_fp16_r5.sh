mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 1200 python -m pytest tests/test_gpu_fp16.py tests/test_gpu_canary.py tests/test_gpu_bench.py -m gpu -q -s -p no:cacheprovider > gpurun_out/pytest_fp16e.log 2>&1; echo pytest_rc=$?; grep -E "passed|failed|threshold|adversarial" gpurun_out/pytest_fp16e.log | tail -8; grep -E "^FAILED" gpurun_out/pytest_fp16e.log | head
PROBE_ACC=0 PROBE_TERMS=4 PROBE_SHAPES=32768x32768x32768 timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm|prep|fix" -c 8 --csv --log-file gpurun_out/launches_c5_randn_r6.csv python scripts/fp16_probe.py > /dev/null 2>&1; echo ncu_rc=$?
PROBE_ACC=0 PROBE_TERMS=4,3 PROBE_SHAPES=32768x32768x32768,16384x16384x16384,262144x1024x1024 python scripts/fp16_probe.py
