# Round 2: the racy two-stream test re-run, the TMA fill-ceiling sweep, the NVLS multicast probe.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 300 python -m pytest tests/test_gpu_sched.py -m gpu -q -s -p no:cacheprovider > gpurun_out/sched.log 2>&1; echo sched_rc=$?; tail -3 gpurun_out/sched.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/nvls_probe scripts/nvls_probe.cu -lcuda && timeout -s KILL 120 /tmp/nvls_probe > gpurun_out/nvls_probe.jsonl 2>&1; echo nvls_rc=$?; cat gpurun_out/nvls_probe.jsonl
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_fill_sweep scripts/tma_fill_sweep.cu -lcuda && timeout -s KILL 600 /tmp/tma_fill_sweep 4000 4096 0 1 > gpurun_out/tma_fill_sweep.jsonl 2>&1; echo sweep_rc=$?
nvidia-smi -q | grep -i -A3 "fabric\|nvlink" | head -30
