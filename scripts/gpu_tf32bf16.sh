# TF32 + BF16 scheme: the GPU tests of both schemes and the touched pipeline test, then the
# rates of the two schemes (RN and truncated hi).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout -s KILL 900 python -m pytest -q -s tests/test_gpu_schemes.py "tests/test_gpu.py::test_rank_compute_only_is_the_pipeline_arithmetic" > gpurun_out/pytest_schemes.log 2>&1; echo pytest_rc=$?
GIGA_HI_RN=0 timeout -s KILL 300 python -m pytest -q -s tests/test_gpu_schemes.py -k coherent 2>&1 | grep coherent
grep -E "coherent|passed|failed|FAILED|Error" gpurun_out/pytest_schemes.log | tail -12
export PROBE_ACC=0 PROBE_SHAPES=16384x16384x16384,32768x32768x32768
timeout -s KILL 300 python scripts/tf32bf16_probe.py > gpurun_out/tf32bf16_rates.jsonl 2>&1
GIGA_HI_RN=0 PROBE_TERMS=2 timeout -s KILL 300 python scripts/tf32bf16_probe.py >> gpurun_out/tf32bf16_rates.jsonl 2>&1
cat gpurun_out/tf32bf16_rates.jsonl
