# ncu evidence of the product path with the TF32 + BF16 scheme: launch lists of the default
# (c5) and c3 bench commands, one --set full capture of the GEMM at c3 and c5 (terms = 2).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo launches_rc=$?
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3_16384 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launches3.log 2>&1; echo launches_rc=$?
TERMS=2 SIZE=16384 PKS=8 timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_3xtf32 -s 2 -c 1 -o gpurun_out/prof_c3_final python scripts/sweep_gemm.py > gpurun_out/ncu_c3.log 2>&1; echo ncu_rc=$?
TERMS=2 MNK=32768,32768,32768 PKS=8 timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_3xtf32 -s 2 -c 1 -o gpurun_out/prof_c5_final python scripts/sweep_gemm.py > gpurun_out/ncu_c5.log 2>&1; echo ncu_rc=$?
TERMS=2 SIZE=16384 PKS=8 timeout -s KILL 600 ncu --set full --clock-control none -k regex:prep_ -c 2 -o gpurun_out/prof_prep_c3 python scripts/sweep_gemm.py > gpurun_out/ncu_prep.log 2>&1; echo ncu_rc=$?
ls -la gpurun_out/*.ncu-rep
timeout -s KILL 900 python -m pytest -q -s "tests/test_gpu.py::test_full_size_sampled_rows" 2>&1 | grep -E "rel err|passed|failed"
