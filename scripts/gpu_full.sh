mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout -s KILL 300 python -m pytest tests -m gpu -q -x -k "pipeline" > gpurun_out/pytest_pipe.log 2>&1; echo pipe_rc=$?
grep -E "passed|failed|FAILED|Error|error" gpurun_out/pytest_pipe.log | tail -10
timeout -s KILL 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED" gpurun_out/pytest_gpu.log | tail -10
