mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -3 gpurun_out/build.log
timeout -s KILL 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -20 gpurun_out/smoke.log
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -s -k "probe or split or golden or integer" > gpurun_out/pytest_gpu1.log 2>&1; echo rc=$?; tail -40 gpurun_out/pytest_gpu1.log
