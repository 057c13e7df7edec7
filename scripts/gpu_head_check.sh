mkdir -p gpurun_out
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/smoke.log
timeout -s KILL 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_all.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed" gpurun_out/pytest_gpu_all.log | tail -2; grep -E "^FAILED|^ERROR" gpurun_out/pytest_gpu_all.log | head -30
timeout -s KILL 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench_rc=$?; head -c 400 gpurun_out/bench_default.json; echo
