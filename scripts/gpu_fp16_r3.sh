mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_fp16.py tests/test_gpu_canary.py -m gpu -q -s -p no:cacheprovider > gpurun_out/pytest_fp16c.log 2>&1; echo pytest_rc=$?; grep -E "passed|failed|threshold" gpurun_out/pytest_fp16c.log | tail -3; grep -E "^FAILED" gpurun_out/pytest_fp16c.log | head
rm -f gpurun_out/scheme_crossover_r02b.jsonl
for s in 3xtf32 tf32bf16 3xfp16; do GIGA_SCHEME=$s timeout -s KILL 600 python scripts/scheme_crossover.py >> gpurun_out/scheme_crossover_r02b.jsonl 2>>gpurun_out/xo.err; done
cat gpurun_out/scheme_crossover_r02b.jsonl | python -c "
import sys,json
d={}
for l in sys.stdin:
    r=json.loads(l); d.setdefault(tuple(r['shape']),{})[r['scheme']]=r['tflops']
for k,v in d.items(): print(k, v)
"
PROBE_ACC=0 PROBE_TERMS=4 PROBE_SHAPES=32768x32768x32768 timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm|prep|fix" -c 8 --csv --log-file gpurun_out/launches_c5_fp16.csv python scripts/fp16_probe.py > /dev/null 2>&1; echo ncu_rc=$?
