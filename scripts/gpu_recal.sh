# Recalibration after the 3xFP16 epilogue fix: scheme crossover (3xfp16 / 3xtf32 / tf32bf16)
# over small, tall and short-K shapes, and the chunk-rate sweep behind make_plan's model.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
export XO_SHAPES="512x512x512,1024x1024x1024,2048x2048x2048,4096x4096x4096,2048x4096x4096,4096x4096x2048,8192x8192x1024,8192x8192x2048,32768x1024x1024,65536x1024x1024,262144x1024x1024,131072x2048x1024,16384x32768x576,16384x32768x1024,16384x16384x1024,8192x16384x1024,4096x32768x1024,2048x16384x16384,4096x4096x8192,8192x8192x8192,16384x16384x16384,16384x32768x256,16384x32768x512,2048x32768x2048"
for s in 3xfp16 3xtf32 tf32bf16; do
  GIGA_SCHEME=$s timeout -s KILL 900 python scripts/scheme_crossover.py > gpurun_out/xo_$s.jsonl 2> gpurun_out/xo_$s.err; echo xo_${s}_rc=$?
done
timeout -s KILL 1500 python scripts/chunk_rate_sweep.py 16384 32768 > gpurun_out/chunk_rate_sweep.jsonl 2> gpurun_out/chunk_rate.err; echo sweep_rc=$?
