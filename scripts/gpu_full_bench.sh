mkdir -p gpurun_out
bash scripts/gpu_full.sh
timeout -s KILL 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench_rc=$?
tail -c 3000 gpurun_out/bench_default.json
