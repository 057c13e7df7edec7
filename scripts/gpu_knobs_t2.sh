# knob sweep of the TF32 + BF16 GEMM (raster group, L2 promotion, wave barrier)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
export PROBE_ACC=0 PROBE_SHAPES=16384x16384x16384,32768x32768x32768 PROBE_TERMS=2
for env in "GIGA_GROUP_M=8" "GIGA_GROUP_M=4" "GIGA_GROUP_M=16" "GIGA_L2_PROMO=3" "GIGA_WAVE_SYNC=0" "GIGA_PROMOTE_KBLOCKS=16" "GIGA_GROUP_M=8"; do
  echo "$env"; env $env timeout -s KILL 300 python scripts/tf32bf16_probe.py 2>&1 | grep -o '"shape.*'
done
