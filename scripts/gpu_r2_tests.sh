# Round-2 GPU check: build, smoke, full GPU suite (new parity tests included), default bench.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -3 gpurun_out/smoke.log
timeout -s KILL 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|error" gpurun_out/pytest_gpu.log | tail -5
grep -E "^FAILED|^ERROR|adversarial|Error" gpurun_out/pytest_gpu.log | head -30
if [ -z "$NO_BENCH" ]; then
timeout -s KILL 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench_rc=$?
tail -c 3000 gpurun_out/bench_default.json
fi
