mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_fp16.py tests/test_gpu_canary.py -m gpu -q -s -p no:cacheprovider > gpurun_out/pytest_fp16d.log 2>&1; echo pytest_rc=$?; grep -E "passed|failed|threshold" gpurun_out/pytest_fp16d.log | tail -3; grep -E "^FAILED" gpurun_out/pytest_fp16d.log | head
for sh in 32768x32768x32768 262144x1024x1024; do
PROBE_ACC=0 PROBE_TERMS=4 PROBE_SHAPES=$sh timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm|prep|fix" -c 8 --csv --log-file gpurun_out/launches_${sh}_r4.csv python scripts/fp16_probe.py > /dev/null 2>&1; echo ncu_rc=$?
done
PROBE_ACC=0 PROBE_TERMS=4 PROBE_SHAPES=32768x32768x32768,16384x16384x16384,262144x1024x1024 python scripts/fp16_probe.py
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r4.json 2> gpurun_out/bench_r4.err; echo bench_rc=$?; head -c 700 gpurun_out/bench_r4.json
