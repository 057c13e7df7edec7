# Round 2 final-state check: build, smoke, whole GPU suite, benches (c5 default, c3, c2, c4),
# launch list, sanitizers (incl. initcheck), the NVLS probe.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; tail -2 gpurun_out/build.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/smoke.log
timeout -s KILL 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_all.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed" gpurun_out/pytest_gpu_all.log | tail -2; grep -E "^FAILED|^ERROR" gpurun_out/pytest_gpu_all.log | head -30
timeout -s KILL 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench_rc=$?; head -c 300 gpurun_out/bench_default.json; echo
for c in c3_16384 c2_4096 c4_tall; do timeout -s KILL 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_${c}_rc=$?; head -c 200 gpurun_out/bench_$c.json; echo; done
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm|prep|fix|compact" --csv --log-file gpurun_out/launches_bench_c5.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1; echo launches_rc=$?
bash scripts/gpu_sanitize.sh > /dev/null 2>&1; head -12 gpurun_out/compute_sanitizer.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/nvls_probe scripts/nvls_probe.cu -lcuda && timeout -s KILL 120 /tmp/nvls_probe > gpurun_out/nvls_probe.jsonl 2>&1; cat gpurun_out/nvls_probe.jsonl
MNK=32768,32768,32768 PKS=8 TERMS=4 timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_3xtf32 -s 2 -c 1 -o gpurun_out/prof_c5_fp16 python scripts/sweep_gemm.py > gpurun_out/ncu_c5.log 2>&1; echo ncu_full_rc=$?
python scripts/ncu_summary.py gpurun_out/prof_c5_fp16.ncu-rep > gpurun_out/prof_c5_fp16_summary.json 2>&1; head -30 gpurun_out/prof_c5_fp16_summary.json
