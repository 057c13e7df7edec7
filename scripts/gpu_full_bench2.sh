# gpu_full_bench.sh + the c3 line
mkdir -p gpurun_out
bash scripts/gpu_full.sh
timeout -s KILL 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench_rc=$?
timeout -s KILL 600 python bench.py --config c3_16384 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench3_rc=$?
tail -c 2500 gpurun_out/bench_default.json; tail -c 1500 gpurun_out/bench_c3.json
