# After the prep16_b change: the 3xFP16 suites, full-size parity, a default bench line and the
# c5 launch list.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 2000 python -m pytest tests/test_gpu_fp16.py tests/test_gpu_schemes.py tests/test_gpu_fullc.py tests/test_gpu_fuzz.py tests/test_gpu_canary.py tests/test_gpu_mcast.py tests/test_gpu.py -q -p no:cacheprovider > gpurun_out/pytest_prepb.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_prepb.log; grep -E "^FAILED" gpurun_out/pytest_prepb.log | head
timeout -s KILL 900 python bench.py --no-cpu-baseline > gpurun_out/bench_prepb.json 2>/dev/null; echo bench_rc=$?; python -c "
import json; d=json.loads(open('gpurun_out/bench_prepb.json').read().splitlines()[-1]); r=d['roofline']; print(d['value'], r['prep_ms_per_step'], r['frac'], d['clocks'], d['e2e']['value'])"
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm|prep|fix|compact" --csv --log-file gpurun_out/launches_bench_c5_prepb.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1; echo launches_rc=$?
