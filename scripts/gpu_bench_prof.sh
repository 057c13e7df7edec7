mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/bench.log
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo launches_rc=$?
SIZE=16384 PKS=8 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_3xtf32 -s 2 -c 1 -o gpurun_out/prof_cg2 python scripts/sweep_gemm.py > gpurun_out/ncu_cg2.log 2>&1; echo ncu_rc=$?
timeout -s KILL 300 ncu --set full --clock-control none -k regex:split_lo -s 2 -c 1 -o gpurun_out/prof_split python scripts/sweep_gemm.py > gpurun_out/ncu_split.log 2>&1; echo ncu2_rc=$?
