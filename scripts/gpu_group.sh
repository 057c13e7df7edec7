mkdir -p gpurun_out
python -c "from paper_2504_01266_b200 import build; build.build()" > gpurun_out/build.log 2>&1
for G in 2 4 8 16 64; do
  echo "GROUP_M=$G"; GIGA_GROUP_M=$G PKS=8 timeout -s KILL 300 python scripts/sweep_gemm.py 2>&1 | tail -1
  GIGA_GROUP_M=$G PKS=8 timeout -s KILL 300 ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum -k regex:gemm_3xtf32 -s 2 -c 1 python scripts/sweep_gemm.py 2>&1 | grep -E "dram__bytes_read|hit_rate|duration" 
done
