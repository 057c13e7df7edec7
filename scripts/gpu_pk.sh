mkdir -p gpurun_out
python -c "from paper_2504_01266_b200 import build; build.build()" > gpurun_out/build.log 2>&1
for R in 1 2; do
MNK=16384,16384,16384 PKS=8,16,32,8 timeout -s KILL 300 python scripts/sweep_gemm.py 2>&1 | tail -4
done
MNK=32768,32768,32768 PKS=8,16,8,16 timeout -s KILL 300 python scripts/sweep_gemm.py 2>&1 | tail -4
