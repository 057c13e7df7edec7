mkdir -p gpurun_out
python -c "from paper_2504_01266_b200 import build; build.build()" > gpurun_out/build.log 2>&1
MNK=262144,1024,1024 PKS=8 timeout -s KILL 120 python scripts/sweep_gemm.py 2>&1 | tail -1
MNK=4096,4096,4096 PKS=8 timeout -s KILL 120 python scripts/sweep_gemm.py 2>&1 | tail -1
MNK=262144,1024,1024 PKS=8 timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:gemm_3xtf32 -s 2 -c 1 -o gpurun_out/prof_c4 python scripts/sweep_gemm.py > /dev/null 2>&1; echo rc=$?
MNK=4096,4096,4096 PKS=8 timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:gemm_3xtf32 -s 2 -c 1 -o gpurun_out/prof_c2 python scripts/sweep_gemm.py > /dev/null 2>&1; echo rc=$?
