mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
T0=$(date +%s); timeout -s KILL 900 python bench.py > gpurun_out/bench_c5.log 2> gpurun_out/bench_c5.err; echo bench_rc=$? wall=$(( $(date +%s) - T0 ))s
tail -2 gpurun_out/bench_c5.err; tail -1 gpurun_out/bench_c5.log
