# MMA order of the TF32 + BF16 stage: interleaved (bf16, tf32 per k8) vs grouped by kind
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
GIGA_MMA_GROUPED=1 timeout -s KILL 600 python -m pytest -q tests/test_gpu_schemes.py -k "bit_exact or tolerance or coherent" 2>&1 | tail -2
export PROBE_ACC=0 PROBE_SHAPES=16384x16384x16384,32768x32768x32768 PROBE_TERMS=2
for g in 1 0 1 0; do
  echo "grouped=$g"; GIGA_MMA_GROUPED=$g timeout -s KILL 300 python scripts/tf32bf16_probe.py 2>&1 | grep -o '"shape.*'
done
