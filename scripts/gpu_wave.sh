mkdir -p gpurun_out
python -c "from paper_2504_01266_b200 import build; build.build()" > gpurun_out/build.log 2>&1
for W in 0 1 0 1; do
  echo -n "WAVE=$W c3: "; GIGA_WAVE_SYNC=$W MNK=16384,16384,16384 PKS=8 timeout -s KILL 120 python scripts/sweep_gemm.py 2>&1 | tail -1
done
for W in 0 1; do
  echo "WAVE=$W"; GIGA_WAVE_SYNC=$W MNK=16384,16384,16384 PKS=8 timeout -s KILL 300 ncu --clock-control none --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,gpc__cycles_elapsed.avg.per_second -k regex:gemm_3xtf32 -s 2 -c 1 python scripts/sweep_gemm.py 2>&1 | grep -E "dram__bytes_read|hit_rate|duration|tensor|per_second"
done
GIGA_WAVE_SYNC=1 MNK=32768,32768,32768 PKS=8 timeout -s KILL 120 python scripts/sweep_gemm.py 2>&1 | tail -1
GIGA_WAVE_SYNC=0 MNK=32768,32768,32768 PKS=8 timeout -s KILL 120 python scripts/sweep_gemm.py 2>&1 | tail -1
