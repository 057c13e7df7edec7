mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
cat > /tmp/tr.py <<'PY'
import sys, torch, synth
from paper_2504_01266_b200 import giga
M = N = K = int(sys.argv[1])
giga.init(1)
Ah = synth.gen_rows_torch(0, M, K, 1, "d2", device="cuda").cpu().pin_memory()
Bh = synth.gen_rows_torch(0, K, N, 2, "d2", device="cuda").cpu().pin_memory()
Ch = torch.empty((M, N)).pin_memory()
for _ in range(3):
    giga.matmul(Ah, Bh, Ch, M, N, K, 1)
PY
for S in 32768 16384; do GIGA_TRACE=1 PYTHONPATH=. timeout -s KILL 300 python /tmp/tr.py $S 2> gpurun_out/trace_$S.txt; tail -1 gpurun_out/trace_$S.txt | cut -c1-3000; done
