# 3xFP16: fix-kernel rework check (tests), then the promotion interval (4 vs 8 k-blocks of 32)
# for speed and long-K accuracy.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_fp16.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_fp16b.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_fp16b.log
for pk in 4 8; do
GIGA_PROMOTE_KBLOCKS=$pk PROBE_TERMS=4 PROBE_SHAPES=262144x1024x1024,4096x4096x4096,16384x32768x1024,16384x16384x16384,32768x32768x32768 timeout -s KILL 900 python scripts/fp16_probe.py 2>&1 | grep -v '"probe": "acc"' | sed "s/^/pk=$pk /"
done
PROBE_ACC=0 PROBE_TERMS=4 PROBE_SHAPES=262144x1024x1024 timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm|prep|fix" -c 8 --csv --log-file gpurun_out/launches_c4_fix2.csv python scripts/fp16_probe.py > /dev/null 2>&1; echo ncu_rc=$?
