"""compute-sanitizer racecheck target: only the cta_group::2 TMEM alloc/dealloc the GEMM does
(libgiga_debug.so giga_dbg_tmem_pair_alloc), to tell the toolchain's alloc handshake apart from
the GEMM's own shared-memory protocol."""
import ctypes, os
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_2504_01266_b200", "libgiga_debug.so"))
out = torch.zeros(18, dtype=torch.int32, device="cuda")
rc = lib.giga_dbg_tmem_pair_alloc(9, ctypes.c_void_p(out.data_ptr()))
print("pair alloc rc", rc, "tmem bases", sorted(set(out.cpu().tolist())))
