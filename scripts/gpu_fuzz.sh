mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout -s KILL 900 python -m pytest tests/test_gpu_fuzz.py -m gpu -q > gpurun_out/pytest_fuzz.log 2>&1; echo fuzz_rc=$?
grep -E "passed|failed|FAILED|Error|assert" gpurun_out/pytest_fuzz.log | tail -20
