# 3xFP16 promotion interval, same box, alternating: bench.py c5 / c3 at 8 and 16 k-blocks,
# then the constructed worst cases and the threshold case at 16.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in 1 2; do for pk in 8 16; do for cfg in c5_32768 c3_16384; do
  GIGA_PROMOTE_KBLOCKS_T4=$pk timeout -s KILL 600 python bench.py --config $cfg --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('pk=$pk $cfg', d['value'], d['clocks']['sm_mhz'])"
done; done; done
GIGA_PROMOTE_KBLOCKS_T4=16 timeout -s KILL 900 python -m pytest tests/test_gpu_fullc.py -k worst tests/test_gpu_fp16.py -m gpu -q -s -p no:cacheprovider 2>&1 | grep -E "threshold worst|product_3xfp16|passed|failed" | sed 's/.tf32bf16.*//' | tail -6
