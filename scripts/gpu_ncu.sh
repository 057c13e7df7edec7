mkdir -p gpurun_out
python -c "from paper_2504_01266_b200 import build; build.build()" > gpurun_out/build.log 2>&1
PKS=0,2,64 timeout -s KILL 300 python scripts/sweep_gemm.py 2>&1 | tail -4
SIZE=16384 PKS=16 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_3xtf32 -s 2 -c 1 -o gpurun_out/prof_pk16 python scripts/sweep_gemm.py > gpurun_out/ncu_pk16.log 2>&1; echo ncu_rc=$?
tail -3 gpurun_out/ncu_pk16.log
