# k-split (deterministic stream-K) on the GPU: its tests, then the shard-GEMM time per shape
# with the split off, planned, and forced to s parts.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout -s KILL 900 python -m pytest tests/test_gpu.py -q -x -k "ksplit or tail_split" 2>&1 | tail -3
: > gpurun_out/ksplit_sweep.jsonl
GIGA_TAIL_SPLIT=0 timeout -s KILL 300 python scripts/ksplit_sweep.py >> gpurun_out/ksplit_sweep.jsonl
timeout -s KILL 300 python scripts/ksplit_sweep.py >> gpurun_out/ksplit_sweep.jsonl
for s in 2 3 4 6 8 12 16; do
  GIGA_KSPLIT_S=$s timeout -s KILL 300 python scripts/ksplit_sweep.py >> gpurun_out/ksplit_sweep.jsonl
done
cat gpurun_out/ksplit_sweep.jsonl
