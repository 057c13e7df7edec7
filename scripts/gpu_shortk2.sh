# Short-K epilogue changes: probe (default promotion interval and 16), fp16 / scheme parity.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
export SHAPES="16384,32768,1024;262144,1024,1024;16384,32768,4096;32768,32768,32768" TERMS=4 REPS=3
for v in "X=1" "GIGA_PROMOTE_KBLOCKS=16"; do
  echo "== $v"; env $v timeout -s KILL 600 python scripts/shortk_probe.py 2>&1 | tail -4
done
timeout -s KILL 900 python -m pytest tests/test_gpu_fp16.py tests/test_gpu_schemes.py tests/test_gpu_mcast.py -q -p no:cacheprovider -x > gpurun_out/pytest_shortk.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_shortk.log
SHAPES="16384,32768,1024" TERMS=4 REPS=1 timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_3xtf32 -s 2 -c 1 -o gpurun_out/prof_shortk2 python scripts/shortk_probe.py > gpurun_out/ncu_shortk2.log 2>&1; echo ncu_rc=$?
