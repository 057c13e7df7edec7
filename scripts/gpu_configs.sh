mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
for C in c1_512 c2_4096 c3_16384 c4_tall c5_32768; do
  E=0; [ $C = c3_16384 ] && E=3; [ $C = c2_4096 ] && E=3; [ $C = c4_tall ] && E=3
  timeout -s KILL 600 python bench.py --config $C --steps 5 --warmup 3 --e2e-steps $E --no-cpu-baseline > gpurun_out/bench_$C.log 2>&1
  tail -1 gpurun_out/bench_$C.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$C', d['value'], d['ms_per_step'], r['achieved'], r['frac'], r['kernel_ms'], r['split_ms_per_step'], d['clocks']['sm_mhz'], (d['e2e'] or {}).get('value'))"
done
timeout -s KILL 900 python -m pytest tests/test_gpu.py -q -s -k "full_size" 2>&1 | grep -E "max rel|passed|failed"
