"""Bring-up probe: TMA swizzled tile layouts and single-UMMA descriptor variants (kind::tf32).

Runs on a GPU box; prints which layouts/descriptors reproduce A[:, :8] @ B[:8, :] exactly.
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_2504_01266_b200", "libgiga_debug.so"))
p, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
lib.giga_dbg_tma_dump.argtypes = [p, i64, i64, i32, i32, i32, i32, i32, p]
lib.giga_dbg_mma_once.argtypes = [p, i32, p, i32, i32, i32, i32, i32, i32, i32, ctypes.c_uint, i32, p]
res = {}


def swz(o, bits):  # physical byte offset of logical o under Swizzle<bits,4,3>
    if bits == "32b":  # Swizzle<2,5,2>: 32 B granules in 128 B rows, 4-row period
        return o ^ ((o >> 2) & 0x60)
    mask = ((1 << bits) - 1) << 4
    return o ^ ((o >> 3) & mask)


def tma_dump(M, box_cols, box_rows, sw, c0=0, c1=0):
    d = torch.from_numpy(np.ascontiguousarray(M)).cuda()
    out = torch.zeros(box_cols * box_rows, device="cuda")
    rc = lib.giga_dbg_tma_dump(d.data_ptr(), M.shape[0], M.shape[1], box_cols, box_rows, sw, c0, c1,
                               out.data_ptr())
    assert rc == 0, rc
    return out.cpu().numpy()


def check_swizzle(name, M, box_cols, box_rows, sw, bits, c0=0, c1=0):
    img = tma_dump(M, box_cols, box_rows, sw, c0, c1)
    exp = np.zeros_like(img)
    for r in range(box_rows):
        for c in range(box_cols):
            o = (r * box_cols + c) * 4
            exp[swz(o, bits) // 4] = M[c1 + r, c0 + c] if (c1 + r < M.shape[0] and c0 + c < M.shape[1]) else 0
    ok = bool(np.array_equal(img, exp))
    res[name] = ok
    print(name, "matches swizzle formula:", ok, flush=True)
    return img


def mma(a_img, b_img, a_lbo, a_sbo, a_lay, b_lbo, b_sbo, b_lay, b_major, n=256):
    idesc = (1 << 4) | (2 << 7) | (2 << 10) | (0 << 15) | (b_major << 16) | ((n >> 3) << 17) | ((128 >> 4) << 24)
    da = torch.from_numpy(np.ascontiguousarray(a_img, dtype=np.float32)).cuda()
    db = torch.from_numpy(np.ascontiguousarray(b_img, dtype=np.float32)).cuda()
    D = torch.full((128, n), float("nan"), device="cuda")
    rc = lib.giga_dbg_mma_once(da.data_ptr(), a_img.size * 4, db.data_ptr(), b_img.size * 4, a_lbo, a_sbo,
                               a_lay, b_lbo, b_sbo, b_lay, idesc, n, D.data_ptr())
    assert rc == 0, rc
    return D.cpu().numpy()


i = np.arange(128)[:, None]
k = np.arange(32)[None, :]
A = (((i * 3 + k) % 7) - 3).astype(np.float32)          # 128 x 32
kk = np.arange(32)[:, None]
j = np.arange(256)[None, :]
B = (((kk * 5 + j) % 9) - 4).astype(np.float32)         # 32 x 256
ref8 = A[:, :8].astype(np.float64) @ B[:8, :].astype(np.float64)

# TMA images
idx = np.arange(128 * 32, dtype=np.float32).reshape(128, 32)
check_swizzle("tma_A_sw64_box16x128", idx, 16, 128, 64, 2)
check_swizzle("tma_A_sw128_box32x128", idx, 32, 128, 128, 3)
idxb = np.arange(32 * 256, dtype=np.float32).reshape(32, 256)
check_swizzle("tma_B_sw128_box32x16", idxb, 32, 16, 128, 3, c0=64, c1=0)

check_swizzle("tma_B_sw128atom32_box32x16", idxb, 32, 16, 132, "32b", c0=64, c1=0)
b32 = np.concatenate([tma_dump(B, 32, 16, 132, c0=32 * c) for c in range(8)])  # 8 x 2 KiB
a64 = tma_dump(A, 16, 128, 64)                          # 8 KiB, K-major SW64
a128 = tma_dump(A, 32, 128, 128)                        # 16 KiB, K-major SW128
b128 = np.concatenate([tma_dump(B, 32, 16, 128, c0=32 * c) for c in range(8)])  # 8 x 2 KiB
Bt = np.ascontiguousarray(B.T)                          # 256 x 32 (K-major B)
bt64 = tma_dump(Bt, 16, 256, 64)                        # 16 KiB

# no-swizzle K-major images built by hand: core matrix = 8 rows x 16 B
def interleave_kmajor(X, kdim=8, lbo=128, sbo=256):
    rows = X.shape[0]
    img = np.zeros((rows // 8) * sbo // 4 + 64, np.float32)
    for r in range(rows):
        for c in range(kdim):
            off = (r // 8) * sbo + (c // 4) * lbo + (r % 8) * 16 + (c % 4) * 4
            img[off // 4] = X[r, c]
    return img

variants = {
    "A_sw64_B_mn_base32b(lbo2048,sbo512)": (a64, b32, 16, 512, 4, 2048, 512, 1, 1),
    "A_sw64_B_mn_base32b(lbo512,sbo2048)": (a64, b32, 16, 512, 4, 512, 2048, 1, 1),
    "A_sw128_B_mn_base32b(lbo2048,sbo512)": (a128, b32, 16, 1024, 2, 2048, 512, 1, 1),
    "A_sw64_B_mn_sw128(lbo2048,sbo1024)": (a64, b128, 16, 512, 4, 2048, 1024, 2, 1),
    "A_sw64_B_mn_sw128(lbo1024,sbo2048)": (a64, b128, 16, 512, 4, 1024, 2048, 2, 1),
    "A_sw128_B_mn_sw128(lbo2048,sbo1024)": (a128, b128, 16, 1024, 2, 2048, 1024, 2, 1),
    "A_sw64_B_k_sw64": (a64, bt64, 16, 512, 4, 16, 512, 4, 0),
    "A_sw128_B_k_sw64": (a128, bt64, 16, 1024, 2, 16, 512, 4, 0),
    "A_none_B_none_kmajor": (interleave_kmajor(A), interleave_kmajor(Bt), 128, 256, 0, 128, 256, 0, 0),
}
for name, v in variants.items():
    try:
        D = mma(*v)
        ok = bool(np.array_equal(D.astype(np.float64), ref8))
        nz = int(np.count_nonzero(D))
        res[name] = {"exact": ok, "nonzero": nz, "d00": float(D[0, 0]), "ref00": float(ref8[0, 0]),
                     "maxdiff": float(np.nanmax(np.abs(D - ref8)))}
    except AssertionError as e:
        res[name] = {"error": str(e)}
    print(name, res[name], flush=True)

os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "debug_umma.json"), "w") as f:
    json.dump(res, f, indent=1)
