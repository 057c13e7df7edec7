mkdir -p gpurun_out
python -c "from paper_2504_01266_b200 import build; build.build()" > gpurun_out/build.log 2>&1
for P in 3 2 0; do
 for G in 8 4; do
  echo "PROMO=$P GROUP=$G"
  GIGA_L2_PROMO=$P GIGA_GROUP_M=$G PKS=8 timeout -s KILL 300 ncu --clock-control none --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,gpc__cycles_elapsed.avg.per_second -k regex:gemm_3xtf32 -s 2 -c 1 python scripts/sweep_gemm.py 2>&1 | grep -E "dram__bytes_read|hit_rate|duration|tensor|per_second"
 done
done
