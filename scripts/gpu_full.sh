mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout -s KILL 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -10
for S in 262144,1024,1024 4096,4096,4096 16384,16384,16384; do MNK=$S PKS=8 timeout -s KILL 120 python scripts/sweep_gemm.py 2>&1 | tail -1; done
