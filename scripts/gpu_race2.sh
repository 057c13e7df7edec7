mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout -s KILL 300 compute-sanitizer --tool racecheck --racecheck-report hazard python scripts/racecheck_gemm_cg2.py 2>&1 | tail -3
bash scripts/gpu_sanitize.sh
timeout -s KILL 900 python -m pytest tests/test_gpu.py -q -x 2>&1 | tail -2
