mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 1500 python -m pytest tests/test_gpu_fp16.py tests/test_gpu_canary.py tests/test_gpu_bench.py tests/test_gpu_fullc.py -m gpu -q -s -p no:cacheprovider > gpurun_out/pytest_fp16f.log 2>&1; echo pytest_rc=$?; grep -E "passed|failed|threshold" gpurun_out/pytest_fp16f.log | tail -4; grep -E "^FAILED" gpurun_out/pytest_fp16f.log | head
bash scripts/gpu_sanitize.sh 2>&1 | tail -40
