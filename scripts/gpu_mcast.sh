# N4 store paths: the new store-mode / multicast tests, the p2p / fused-gather suites, a
# default bench (no regression of the product kernel), the NVLS probe.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
timeout -s KILL 1500 python -m pytest tests/test_gpu_mcast.py tests/test_gpu_multi.py tests/test_gpu_fp16.py tests/test_gpu_canary.py -q -p no:cacheprovider -rs > gpurun_out/pytest_mcast.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/pytest_mcast.log
timeout -s KILL 900 python bench.py --no-cpu-baseline > gpurun_out/bench_mcast.json 2> gpurun_out/bench_mcast.err; echo bench_rc=$?; head -c 300 gpurun_out/bench_mcast.json; echo
