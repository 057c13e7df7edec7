mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout -s KILL 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for v in 0 1; do
  echo "GIGA_TAIL_SPLIT=$v"
  GIGA_TAIL_SPLIT=$v timeout -s KILL 300 python scripts/gemm_shapes.py 2>&1 | tail -10
done
STRESS_SECONDS=180 timeout -s KILL 400 python scripts/stress_lo_smem.py | tail -1
