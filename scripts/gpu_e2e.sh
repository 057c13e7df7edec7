mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout -s KILL 900 python -m pytest tests/test_gpu.py tests/test_gpu_vec.py -q -x -k "host or paper_api or matmul" 2>&1 | tail -2
for C in c5_32768 c3_16384 c2_4096 c4_tall c1_512; do
  timeout -s KILL 600 python bench.py --config $C --steps 3 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/bench_e2e_$C.log 2>&1
  tail -1 gpurun_out/bench_e2e_$C.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$C', d['value'], d['e2e'])"
done
