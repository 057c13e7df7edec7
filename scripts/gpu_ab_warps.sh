# Same-box A/B of the 3xTF32 rate: 16-warp layout (libgiga.so) vs the 12-warp build
# (abtest/libgiga_12w.so), alternating.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
export PROBE_ACC=0 PROBE_SHAPES=16384x16384x16384,32768x32768x32768 PROBE_TERMS=3
for i in 1 2; do
  echo "16w"; timeout -s KILL 300 python scripts/tf32bf16_probe.py 2>&1 | cut -c1-40,120-
  echo "12w"; GIGA_LIB_PATH=abtest/libgiga_12w.so timeout -s KILL 300 python scripts/tf32bf16_probe.py 2>&1 | cut -c1-40,120-
done
PROBE_TERMS=2 timeout -s KILL 300 python scripts/tf32bf16_probe.py 2>&1 | cut -c1-40,120-
