"""Pinned host <-> device copy rates on this box: contiguous, cudaMemcpy2DAsync column blocks
(the host pipeline's phase-1 copies), and both directions at once."""
import json, torch
from cuda.bindings import runtime as rt
dev = torch.device("cuda", 0)
GiB = 1 << 30
h = torch.empty(GiB // 4, dtype=torch.float32).pin_memory()
d = torch.empty(GiB // 4, dtype=torch.float32, device=dev)
h2 = torch.empty(GiB // 4, dtype=torch.float32).pin_memory()
d2 = torch.empty(GiB // 4, dtype=torch.float32, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
H2D, D2H = rt.cudaMemcpyKind.cudaMemcpyHostToDevice, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record(); fn(); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return best
cs = torch.cuda.current_stream().cuda_stream
res = {}
res["h2d_GBs"] = GiB / t(lambda: rt.cudaMemcpyAsync(d.data_ptr(), h.data_ptr(), GiB, H2D, cs)) / 1e9
res["d2h_GBs"] = GiB / t(lambda: rt.cudaMemcpyAsync(h.data_ptr(), d.data_ptr(), GiB, D2H, cs)) / 1e9
def duplex():
    rt.cudaMemcpyAsync(d.data_ptr(), h.data_ptr(), GiB, H2D, s1.cuda_stream)
    rt.cudaMemcpyAsync(h2.data_ptr(), d2.data_ptr(), GiB, D2H, s2.cuda_stream)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
res["duplex_each_GBs"] = GiB / t(duplex) / 1e9
for w in (256, 512, 1024, 2048, 4096):
    sec = t(lambda: rt.cudaMemcpy2DAsync(d.data_ptr(), 16384 * 4, h.data_ptr(), 16384 * 4, w * 4,
                                         16384, H2D, cs))
    res[f"h2d_2d_w{w}_GBs"] = 16384 * w * 4 / sec / 1e9
print(json.dumps({k: round(v, 1) for k, v in res.items()}))
