mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x -s > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|Error|max rel err" gpurun_out/pytest_gpu.log | tail -12
for S in 262144,1024,1024 4096,4096,4096 16384,16384,16384 32768,32768,32768; do for W in 0 1; do echo -n "W=$W $S "; GIGA_WAVE_SYNC=$W MNK=$S PKS=8 timeout -s KILL 120 python scripts/sweep_gemm.py 2>&1 | tail -1; done; done
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/bench.log
