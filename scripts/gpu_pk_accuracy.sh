mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for pk in 8 12 16; do
  echo "pk=$pk"
  GIGA_PROMOTE_KBLOCKS=$pk timeout -s KILL 900 python -m pytest tests/test_gpu.py -q -s -k "full_size and 32768" 2>&1 | grep -E "max rel|passed|failed"
  SIZE=32768 PKS=$pk timeout -s KILL 300 python scripts/sweep_gemm.py 2>&1 | tail -1
done
