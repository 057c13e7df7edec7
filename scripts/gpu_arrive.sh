# Fence-free TMEM-empty arrive: short-K probe, parity suites, bench lines (peak choice).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
SHAPES="16384,32768,1024;262144,1024,1024;16384,32768,4096;32768,32768,32768" TERMS=4 REPS=3 timeout -s KILL 600 python scripts/shortk_probe.py 2>&1 | tail -4
timeout -s KILL 1500 python -m pytest tests/test_gpu.py tests/test_gpu_fp16.py tests/test_gpu_schemes.py tests/test_gpu_fullc.py tests/test_gpu_sched.py -q -p no:cacheprovider -x > gpurun_out/pytest_arrive.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_arrive.log
timeout -s KILL 900 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_arrive.json 2>/dev/null; echo bench_rc=$?; python -c "
import json; d=json.loads(open('gpurun_out/bench_arrive.json').read().splitlines()[-1]); r=d['roofline']; print(d['value'], r['peak_kind'], r['frac'], d['clocks'])"
timeout -s KILL 600 python bench.py --config c3_16384 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_arrive_c3.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/bench_arrive_c3.json').read().splitlines()[-1]); r=d['roofline']; print(d['value'], r['peak_kind'], r['frac'], d['clocks'])"
