# Multi-GPU bring-up and scaling (for a box with several GPUs): the physical-GPU tests, then
# bench.py at N = 1, 2, 4, 8 with both transports, and one traced call per N (GIGA_TRACE=1:
# per-rank JSON timelines of the broadcast / GEMM / gather chunks on stderr).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
NG=$(python -c "import torch; print(torch.cuda.device_count())")
echo "GPUs: $NG"
timeout -s KILL 1800 python -m pytest tests/test_gpu_multi.py tests/test_gpu_mcast.py -q -rs > gpurun_out/pytest_multi.log 2>&1; tail -3 gpurun_out/pytest_multi.log
CFG=${CFG:-c5_32768}
for T in nccl p2p; do
  for N in 1 2 4 8; do
    [ $N -gt $NG ] && continue
    if [ $N = 1 ]; then
      timeout -s KILL 900 python bench.py --config $CFG --transport $T > gpurun_out/scale_${T}_$N.json 2> gpurun_out/scale_${T}_$N.err
    else
      timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + N)) bench.py --gpus $N --config $CFG --transport $T > gpurun_out/scale_${T}_$N.json 2> gpurun_out/scale_${T}_$N.err
      GIGA_TRACE=1 timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + N)) bench.py --gpus $N --config $CFG --transport $T --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2> gpurun_out/trace_${T}_$N.err
    fi
    tail -1 gpurun_out/scale_${T}_$N.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$T', $N, d['value'], d['ms_per_step'], d['roofline_step']['frac'])"
  done
done
# the multicast gather (N4): C_full bound into an NVLink multicast team (falls back to the
# unicast gather, noted in config.gather, where the driver refuses multicast)
for N in 2 4 8; do
  [ $N -gt $NG ] && continue
  timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29700 + N)) bench.py --gpus $N --config $CFG --transport p2p --gather mc > gpurun_out/scale_mc_$N.json 2> gpurun_out/scale_mc_$N.err
  tail -1 gpurun_out/scale_mc_$N.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('p2p+mc', $N, d['value'], d['ms_per_step'], d['config'].get('gather'))"
done
