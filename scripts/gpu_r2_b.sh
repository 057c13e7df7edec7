# overlap test, c4 scheme comparison (bench), prep kernel timings after batching the loads
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_overlap.py tests/test_gpu.py::test_trace_timelines -m gpu -q -s -p no:cacheprovider > gpurun_out/pytest_overlap.log 2>&1; echo overlap_rc=$?; grep -E "overlap:|passed|failed" gpurun_out/pytest_overlap.log | tail -3; grep -E "^E " gpurun_out/pytest_overlap.log | head -10
for s in 3xtf32 3xfp16; do GIGA_SCHEME=$s timeout -s KILL 600 python bench.py --config c4_tall --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c4_$s.json 2>/dev/null; echo c4 $s; head -c 250 gpurun_out/bench_c4_$s.json; echo; done
XO_SHAPES=262144x1024x1024,131072x1024x1024,65536x2048x2048,32768x4096x4096,16384x8192x8192,8192x16384x2048,32768x32768x2048,16384x16384x2048 bash -c 'for s in 3xtf32 3xfp16; do GIGA_SCHEME=$s timeout -s KILL 600 python scripts/scheme_crossover.py; done' > gpurun_out/xo_c.jsonl 2>/dev/null; cat gpurun_out/xo_c.jsonl
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"prep|compact|fix" -c 12 --csv --log-file gpurun_out/launches_prep_c5.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1; echo launches_rc=$?
