# 3xFP16 with exception fixes: its GPU tests, the canary / scheduler tests, the scheme
# crossover for all three schemes, the ncu launch list of a forced 3xFP16 bench step.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
timeout -s KILL 1200 python -m pytest tests/test_gpu_fp16.py tests/test_gpu_canary.py tests/test_gpu_sched.py -m gpu -q -s -p no:cacheprovider > gpurun_out/pytest_fp16.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed" gpurun_out/pytest_fp16.log | tail -3; grep -E "^FAILED|^ERROR|threshold worst" gpurun_out/pytest_fp16.log | head -30
for s in 3xtf32 tf32bf16 3xfp16; do GIGA_SCHEME=$s timeout -s KILL 600 python scripts/scheme_crossover.py >> gpurun_out/scheme_crossover_r02.jsonl 2>>gpurun_out/xo.err; done
cat gpurun_out/scheme_crossover_r02.jsonl | python -c "
import sys,json
d={}
for l in sys.stdin:
    r=json.loads(l); d.setdefault(tuple(r['shape']),{})[r['scheme']]=r['tflops']
for k,v in d.items(): print(k, v)
"
GIGA_SCHEME=3xfp16 timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm|prep|fix" -c 40 --csv --log-file gpurun_out/launches_c3_3xfp16.csv python bench.py --config c3_16384 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1; echo ncu_rc=$?
