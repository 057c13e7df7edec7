mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout -s KILL 900 python -m pytest tests/test_gpu_vec.py -m gpu -q -x > gpurun_out/pytest_vec.log 2>&1; echo vec_rc=$?
grep -E "passed|failed|FAILED|Error|assert" gpurun_out/pytest_vec.log | tail -15
