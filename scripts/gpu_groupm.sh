# L2 raster group (M-tiles walked before the next N-tile) of the 3xFP16 GEMM: bench.py c5 at
# GIGA_GROUP_M = 4 / 8 / 16, same box, alternating twice; DRAM bytes per launch from ncu.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in 1 2; do for gm in 4 8 16; do
  GIGA_GROUP_M=$gm timeout -s KILL 600 python bench.py --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('group_m=$gm', d['value'], d['clocks']['sm_mhz'])"
done; done
for gm in 4 16; do
  GIGA_GROUP_M=$gm MNK=32768,32768,32768 PKS=8 TERMS=4 timeout -s KILL 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_3xtf32 -s 2 -c 1 --csv python scripts/sweep_gemm.py 2>/dev/null | grep -E "dram__bytes|duration" | sed "s/^/group_m=$gm /" | cut -c1-160
done
