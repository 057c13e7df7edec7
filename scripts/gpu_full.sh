mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout -s KILL 900 python -m pytest tests/test_gpu.py -m gpu -q -k "host or golden or tolerance or smoke" > gpurun_out/pytest_host.log 2>&1; echo host_rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_host.log | tail -10
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 5 > gpurun_out/bench.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'])"
for P in 40 50 70; do GIGA_HOST_EARLY_PCT=$P timeout -s KILL 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$P', d['e2e']['value'], d['e2e']['ms_per_step'])"; done
