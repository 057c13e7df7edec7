mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo launches_rc=$?
MNK=16384,16384,16384 PKS=8 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_3xtf32 -s 2 -c 1 -o gpurun_out/prof_c3_wave python scripts/sweep_gemm.py > gpurun_out/ncu_c3.log 2>&1; echo ncu_rc=$?
MNK=32768,32768,32768 PKS=8 timeout -s KILL 600 ncu --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,gpc__cycles_elapsed.avg.per_second -k regex:gemm_3xtf32 -s 2 -c 1 python scripts/sweep_gemm.py > gpurun_out/ncu_c5.log 2>&1; echo ncu5_rc=$?
grep -E "dram__|hit_rate|duration|tensor|per_second" gpurun_out/ncu_c5.log
MNK=16384,16384,16384 timeout -s KILL 300 ncu --set full --clock-control none -k regex:split_lo -c 1 -o gpurun_out/prof_split python scripts/sweep_gemm.py > gpurun_out/ncu_split.log 2>&1; echo ncu2_rc=$?
