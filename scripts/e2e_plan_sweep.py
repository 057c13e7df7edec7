"""giga_matmul on pinned host buffers at 32768^3 (the paper's call, bench.py's e2e) under the
host plans $GIGA_HOST_PLAN forces, vs the planner's own choice: wall ms per call (median of
3 after a warm call). One JSON line per plan."""
import json, os, statistics, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
M = N = K = int(os.environ.get("E2E_SIZE", "32768"))
plans = os.environ.get("E2E_PLANS", "auto").split(";")
code = r'''
import os, sys, time, statistics, json
import torch
sys.path.insert(0, os.getcwd())
import synth
from paper_2504_01266_b200 import giga
M = N = K = int(sys.argv[1])
A = torch.empty((M, K), dtype=torch.float32).pin_memory()
B = torch.empty((K, N), dtype=torch.float32).pin_memory()
C = torch.empty((M, N), dtype=torch.float32).pin_memory()
synth.gen_rows_torch(0, M, K, synth.MATRIX_A, "d2", out=A)
synth.gen_rows_torch(0, K, N, synth.MATRIX_B, "d2", out=B)
giga.init(1)
giga.matmul(A, B, C, M, N, K, 1)
ts = []
for _ in range(3):
    t0 = time.perf_counter(); giga.matmul(A, B, C, M, N, K, 1); ts.append((time.perf_counter() - t0) * 1e3)
giga.finalize()
ms = statistics.median(ts)
print(json.dumps({"ms": round(ms, 2), "tflops": round(2 * M * N * K / ms / 1e9, 1)}))
'''
for pl in plans:
    env = dict(os.environ)
    if pl != "auto":
        env["GIGA_HOST_PLAN"] = pl
    r = subprocess.run([sys.executable, "-c", code, str(M)], env=env, capture_output=True,
                       text=True, cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    line = [x for x in r.stdout.splitlines() if x.startswith("{")]
    out = json.loads(line[-1]) if line else {"err": r.stderr[-300:]}
    print(json.dumps({"plan": pl, **out}), flush=True)
