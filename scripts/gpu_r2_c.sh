mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_fp16.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_fp16g.log 2>&1; echo fp16_rc=$?; tail -1 gpurun_out/pytest_fp16g.log
for pk in 8 16; do
GIGA_PROMOTE_KBLOCKS=$pk PROBE_TERMS=4 PROBE_SHAPES=32768x32768x32768,16384x16384x16384 timeout -s KILL 900 python scripts/fp16_probe.py 2>&1 | grep -E "longk|rate" | grep -v '"terms": 2' | sed "s/^/pk=$pk /"
GIGA_PROMOTE_KBLOCKS=$pk timeout -s KILL 300 python -m pytest tests/test_gpu_fp16.py -k "threshold" -m gpu -q -s -p no:cacheprovider 2>&1 | grep "threshold worst" | sed "s/^/pk=$pk /"
done
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"prep|compact|fix" -c 12 --csv --log-file gpurun_out/launches_prep_c5b.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1; echo launches_rc=$?
timeout -s KILL 900 python bench.py > gpurun_out/bench_default2.json 2>/dev/null; echo bench_rc=$?; python -c "
import json; d=json.loads(open('gpurun_out/bench_default2.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['prep_ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step'], d['clocks'])"
GIGA_TRACE=1 timeout -s KILL 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 2> gpurun_out/trace_e2e.err > /dev/null; grep '"trace": "host' gpurun_out/trace_e2e.err | tail -1 | head -c 1500
