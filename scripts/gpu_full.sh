mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout -s KILL 200 python -m pytest tests -m gpu -q -x -k "cta_group" > gpurun_out/pytest_cg.log 2>&1; echo cg_rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_cg.log | tail -10
PKS=8,16 timeout -s KILL 300 python scripts/sweep_gemm.py 2>&1 | tail -3
GIGA_CTA_GROUP=1 PKS=16 timeout -s KILL 300 python scripts/sweep_gemm.py 2>&1 | tail -2
timeout -s KILL 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -10
