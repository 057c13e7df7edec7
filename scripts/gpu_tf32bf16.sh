# TF32 + BF16 scheme: GPU tests (schemes, full-size parity), then rates vs 3xTF32.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout -s KILL 900 python -m pytest -q -s tests/test_gpu_schemes.py "tests/test_gpu.py::test_full_size_sampled_rows" > gpurun_out/pytest_schemes.log 2>&1; echo pytest_rc=$?
grep -E "coherent|max rel|passed|failed|FAILED|Error" gpurun_out/pytest_schemes.log | tail -12
export PROBE_ACC=0 PROBE_SHAPES=16384x16384x16384,32768x32768x32768
timeout -s KILL 300 python scripts/tf32bf16_probe.py > gpurun_out/tf32bf16_rates.jsonl 2>&1
cut -c1-40,120- gpurun_out/tf32bf16_rates.jsonl
