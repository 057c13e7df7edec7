mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
for N in 67108864 1073741824; do timeout -s KILL 300 python bench.py --workload dot --n $N > gpurun_out/bench_vec_$N.log 2>&1; tail -1 gpurun_out/bench_vec_$N.log; done
timeout -s KILL 300 ncu --set full --clock-control none -k regex:dot_kernel -s 3 -c 1 -o gpurun_out/prof_dot python bench.py --workload dot --n 1073741824 --steps 2 > /dev/null 2>&1; echo ncu_rc=$?
