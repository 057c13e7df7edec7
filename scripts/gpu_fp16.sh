# 3xFP16 bring-up: accuracy + rates (scripts/fp16_probe.py), then the product bench with the
# scheme forced.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
timeout -s KILL 900 python scripts/fp16_probe.py > gpurun_out/fp16_probe.jsonl 2> gpurun_out/fp16_probe.err; echo probe_rc=$?
cat gpurun_out/fp16_probe.jsonl; tail -5 gpurun_out/fp16_probe.err
if [ -z "$NO_BENCH" ]; then
GIGA_SCHEME=3xfp16 timeout -s KILL 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_fp16.json 2> gpurun_out/bench_fp16.err; echo bench_rc=$?
tail -c 1500 gpurun_out/bench_fp16.json; tail -3 gpurun_out/bench_fp16.err
fi
