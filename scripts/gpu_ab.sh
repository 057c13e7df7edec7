mkdir -p gpurun_out
for R in 1 2; do
for L in libgiga_prev.so libgiga.so; do
  for S in 16384,16384,16384 262144,1024,1024; do echo -n "$L $S: "; GIGA_LIB_PATH=paper_2504_01266_b200/$L MNK=$S PKS=8 timeout -s KILL 120 python scripts/sweep_gemm.py 2>&1 | tail -1; done
done; done
