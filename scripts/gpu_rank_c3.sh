# Launch lists of rank W-1's GEMM launches at c3 for W = 2 and 8 (what the N > 1 per-GPU
# compute spends its time on after the epilogue fix).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for w in 2 8; do
S=16384 W=$w timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm|prep|fix|compact" --csv --log-file gpurun_out/launches_rank_c3_w$w.csv python scripts/rank_compute_probe.py > gpurun_out/rank_c3_w$w.log 2>&1; echo w${w}_rc=$?
done
S=32768 W=8 timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm|prep|fix|compact" --csv --log-file gpurun_out/launches_rank_c5_w8.csv python scripts/rank_compute_probe.py > gpurun_out/rank_c5_w8.log 2>&1; echo c5w8_rc=$?
