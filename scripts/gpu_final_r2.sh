# Round-2 final state: build, smoke, whole GPU suite, bench lines (c5 default incl. e2e and
# cpu_baseline; c3, c2, c4), reference arm, c5 launch list, sanitizers (incl. the store modes).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -1 gpurun_out/build.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
timeout -s KILL 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/pytest_gpu_all.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed" gpurun_out/pytest_gpu_all.log | tail -2; grep -E "^FAILED|^ERROR" gpurun_out/pytest_gpu_all.log | head -30
timeout -s KILL 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench_rc=$?; head -c 300 gpurun_out/bench_default.json; echo
for c in c3_16384 c2_4096 c4_tall; do timeout -s KILL 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_${c}_rc=$?; head -c 200 gpurun_out/bench_$c.json; echo; done
timeout -s KILL 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo ref_rc=$?; head -c 300 gpurun_out/bench_reference.json; echo
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm|prep|fix|compact" --csv --log-file gpurun_out/launches_bench_c5.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1; echo launches_rc=$?
echo "(compute-sanitizer is closed on this pool)"
