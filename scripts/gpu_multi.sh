mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout -s KILL 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -x > gpurun_out/pytest_multi.log 2>&1; echo multi_rc=$?
grep -E "passed|failed|FAILED|Error|assert|GigaError" gpurun_out/pytest_multi.log | tail -25
