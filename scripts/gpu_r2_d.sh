mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 900 python -m pytest "tests/test_gpu.py::test_full_size_sampled_rows" -m gpu -q -s -p no:cacheprovider > gpurun_out/pytest_full_d5.log 2>&1; echo full_rc=$?; grep -E "max rel|passed|failed" gpurun_out/pytest_full_d5.log | tail -8
for bps in 2 8; do GIGA_PREPB_BLOCKS_PER_SM=$bps timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"prep16_b_kernel" -c 3 --csv --log-file gpurun_out/launches_prepb_$bps.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1; grep -o '"[0-9.]*"$' gpurun_out/launches_prepb_$bps.csv | tail -2 | sed "s/^/bps=$bps /"; done
timeout -s KILL 900 python bench.py --dist d5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_d5.json 2>/dev/null; echo bench_d5_rc=$?; python -c "
import json; d=json.loads(open('gpurun_out/bench_d5.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['prep_ms_per_step'], d['clocks'])"
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm|prep|fix|compact" -c 8 --csv --log-file gpurun_out/launches_c5_d5.csv python bench.py --dist d5 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1; echo rc=$?
