# The 3xFP16 scheme on one GPU: its GPU tests, accuracy + rates of every scheme
# (fp16_probe.py), the promotion-interval trade (PK="4 8 16"), the product-path crossover of
# the three schemes (scheme_crossover.py), launch lists of the c5 step on d2 and d5 inputs.
# Sections can be skipped: NO_TESTS=1, NO_PK=1, NO_XO=1, NO_NCU=1.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [ -z "$NO_TESTS" ]; then
  timeout -s KILL 1200 python -m pytest tests/test_gpu_fp16.py tests/test_gpu_canary.py tests/test_gpu_fullc.py -m gpu -q -s -p no:cacheprovider > gpurun_out/pytest_3xfp16.log 2>&1
  echo tests_rc=$?; grep -E "passed|failed|threshold|adversarial" gpurun_out/pytest_3xfp16.log | tail -6
fi
if [ -z "$NO_PK" ]; then
  for pk in ${PK:-8 16}; do
    GIGA_PROMOTE_KBLOCKS=$pk PROBE_TERMS=4 PROBE_SHAPES=32768x32768x32768,16384x16384x16384 timeout -s KILL 900 python scripts/fp16_probe.py 2>&1 | grep -E "longk|rate" | sed "s/^/pk=$pk /"
  done
fi
if [ -z "$NO_XO" ]; then
  rm -f gpurun_out/scheme_crossover.jsonl
  for s in 3xtf32 tf32bf16 3xfp16; do GIGA_SCHEME=$s timeout -s KILL 900 python scripts/scheme_crossover.py >> gpurun_out/scheme_crossover.jsonl 2>/dev/null; done
  python - <<'PY'
import json
d = {}
for l in open("gpurun_out/scheme_crossover.jsonl"):
    r = json.loads(l); d.setdefault(tuple(r["shape"]), {})[r["scheme"]] = r["tflops"]
for k, v in d.items(): print(k, v)
PY
fi
if [ -z "$NO_NCU" ]; then
  for dist in d2 d5; do
    timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm|prep|fix|compact" -c 8 --csv --log-file gpurun_out/launches_c5_$dist.csv python bench.py --dist $dist --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1; echo ncu_${dist}_rc=$?
  done
fi
