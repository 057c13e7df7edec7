"""cuBLAS reference points on this box (context for the roofline; SURVEY.md 8(d) asks for a real
TF32 probe): torch.matmul fp32 with TF32 tensor cores (1 MMA per product, not fp32-accurate)
and without (SGEMM), burst (best of 10) and sustained (back to back for ~4 s), CUDA events."""
import json, time, torch
res = {}
def run(n, tf32, sustained_s=0.0):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.rand(n, n, device="cuda") * 2 - 1
    b = torch.rand(n, n, device="cuda") * 2 - 1
    c = torch.empty(n, n, device="cuda")
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); torch.matmul(a, b, out=c); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    out = {"burst_tflops": round(2 * n ** 3 / best / 1e9, 1)}
    if sustained_s:
        reps = max(1, int(sustained_s / (best / 1e3)))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            torch.matmul(a, b, out=c)
        e1.record(); e1.synchronize()
        out["sustained_tflops"] = round(2 * n ** 3 * reps / e0.elapsed_time(e1) / 1e9, 1)
        out["sustained_reps"] = reps
    return out
res["tf32_8192"] = run(8192, True, 4.0)
res["tf32_16384"] = run(16384, True, 4.0)
res["sgemm_fp32_8192"] = run(8192, False)
res["sgemm_fp32_16384"] = run(16384, False, 4.0)
res["torch"] = torch.__version__
res["how"] = "torch.matmul fp32, allow_tf32 on/off; U[-1,1) inputs; best of 10 (burst), back-to-back ~4 s (sustained)"
print(json.dumps(res))
