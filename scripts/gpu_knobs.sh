mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
for rep in 1 2; do
for sz in 16384 32768; do
for knob in "GIGA_WAVE_SYNC=1" "GIGA_WAVE_SYNC=0" "GIGA_GROUP_M=4" "GIGA_GROUP_M=16" "GIGA_L2_PROMO=3" "GIGA_PROMOTE_KBLOCKS=16"; do
  echo -n "$sz $knob: "; env $knob SIZE=$sz PKS=-1 timeout -s KILL 300 python scripts/sweep_gemm.py 2>&1 | tail -1
done; done; done
