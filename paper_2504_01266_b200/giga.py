"""Thin ctypes binding of libgiga.so (include/giga.h). Argument marshalling only.

Every step of the matrix multiply runs inside libgiga's CUDA kernels and NCCL calls; this
module converts numpy arrays / torch tensors to raw pointers and status codes to
exceptions. There is no fallback: if libgiga.so is missing or cannot load, importing this
module raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GIGA_LIB_PATH") or os.path.join(_HERE, "libgiga.so")  # A/B runs

GIGA_OK = 0
STATUS = {
    0: "GIGA_OK", -1: "GIGA_ERR_INVALID_ARG", -2: "GIGA_ERR_NOT_INITIALIZED",
    -3: "GIGA_ERR_ALREADY_INITIALIZED", -4: "GIGA_ERR_NO_DEVICE", -5: "GIGA_ERR_OOM",
    -6: "GIGA_ERR_CUDA", -7: "GIGA_ERR_COMM", -8: "GIGA_ERR_UNSUPPORTED",
}
EXPORTS = (
    "giga_init", "giga_num_devices", "giga_finalize", "giga_partition", "giga_matmul",
    "giga_matmul_sharded", "giga_last_error", "giga_comm_unique_id", "giga_rank_init",
    "giga_matmul_rank", "giga_split_lo", "giga_gemm_3xtf32", "giga_gemm_3xtf32_ex",
    "giga_timing_enable", "giga_timing_reset", "giga_timing_read", "giga_pipeline_plan",
    "giga_plan_block", "giga_dot", "giga_l2norm", "giga_dot_rank", "giga_init_devices",
    "giga_rank_p2p_export", "giga_rank_p2p_import", "giga_host_plan", "giga_gemm_schedule",
    "giga_rank_compute_only", "giga_product_scheme", "giga_gemm_gather_ex", "giga_mc_alloc",
    "giga_mc_free", "giga_rank_mc_create", "giga_rank_mc_join", "giga_rank_mc_bind",
)
P2P_BLOB_BYTES = 256
MC_BLOB_BYTES = 64


class GigaError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.status = STATUS.get(code, str(code))


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (there is no CPU fallback)")
    # NCCL is dlopen'ed lazily by libgiga; make the torch wheel's copy resolvable first.
    try:
        import torch  # noqa: F401  (loads libnccl.so.2 into the process)
    except Exception:
        pass
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    i64, i32, p = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
    P64 = ctypes.POINTER(ctypes.c_int64)
    sig = {
        "giga_init": ([i32], i32),
        "giga_num_devices": ([], i32),
        "giga_finalize": ([], i32),
        "giga_partition": ([i64, i32, i32, P64, P64], i32),
        "giga_matmul": ([p, p, p, i64, i64, i64, i32], i32),
        "giga_matmul_sharded": ([p, p, p, i64, i64, i64, i32], i32),
        "giga_last_error": ([], ctypes.c_char_p),
        "giga_comm_unique_id": ([p], i32),
        "giga_rank_init": ([i32, i32, i32, p], i32),
        "giga_matmul_rank": ([p, p, p, i64, i64, i64, p], i32),
        "giga_split_lo": ([p, p, i64, p], i32),
        "giga_gemm_3xtf32": ([p, p, p, p, p, i64, i64, i64, i64, p], i32),
        "giga_gemm_3xtf32_ex": ([p, p, p, p, p, i64, i64, i64, i64, i32, i32, i32, p], i32),
        "giga_timing_enable": ([i32], i32),
        "giga_timing_reset": ([], i32),
        "giga_timing_read": ([ctypes.POINTER(ctypes.c_double), P64,
                              ctypes.POINTER(ctypes.c_double), P64], i32),
        "giga_pipeline_plan": ([i64, i64, i64, i32, ctypes.POINTER(i32), P64,
                                ctypes.POINTER(i32)], i32),
        "giga_plan_block": ([i64, i32, i32, i32, i32, P64, P64], i32),
        "giga_dot": ([p, p, i64, i32, ctypes.POINTER(ctypes.c_double)], i32),
        "giga_l2norm": ([p, i64, i32, ctypes.POINTER(ctypes.c_double)], i32),
        "giga_dot_rank": ([p, p, i64, ctypes.POINTER(ctypes.c_double), p], i32),
        "giga_init_devices": ([p, i32], i32),
        "giga_rank_p2p_export": ([p, p, p], i32),
        "giga_rank_p2p_import": ([p, i32], i32),
        "giga_host_plan": ([i64, i64, i64, i32, P64, ctypes.POINTER(ctypes.c_int), P64,
                            ctypes.POINTER(ctypes.c_int), P64,
                            ctypes.POINTER(ctypes.c_double)], i32),
        "giga_gemm_schedule": ([i64, i64, i64, i32, P64], i32),
        "giga_product_scheme": ([i64, i64, i64, ctypes.POINTER(ctypes.c_int)], i32),
        "giga_rank_compute_only": ([p, p, p, i64, i64, i64, i32, i32, p], i32),
        "giga_gemm_gather_ex": ([p, p, p, p, i32, i64, i64, i64, i64, i32, i32, p], i32),
        "giga_mc_alloc": ([i32, ctypes.c_size_t, p], i32),
        "giga_mc_free": ([p], i32),
        "giga_rank_mc_create": ([ctypes.c_size_t, p], i32),
        "giga_rank_mc_join": ([p], i32),
        "giga_rank_mc_bind": ([p], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


lib = _load()


def last_error() -> str:
    return lib.giga_last_error().decode()


def _check(rc: int):
    if rc != GIGA_OK:
        raise GigaError(rc, last_error())


def _ptr(x):
    """Raw address of a numpy array / torch tensor (contiguous fp32) or an int."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        if not x.flags.c_contiguous:
            raise ValueError("arrays must be C-contiguous")
        return x.ctypes.data
    if hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise ValueError("tensors must be contiguous")
        return x.data_ptr()
    raise TypeError(f"cannot take the address of {type(x)}")


def _stream(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream  # torch.cuda.Stream


# ---- single-process API -----------------------------------------------------------------

def init(ngpus_max: int = 0):
    _check(lib.giga_init(ngpus_max))


def init_devices(devices):
    """giga_init_devices: library GPU g on CUDA device devices[g] (repeats allowed)."""
    arr = (ctypes.c_int * len(devices))(*devices)
    _check(lib.giga_init_devices(ctypes.cast(arr, ctypes.c_void_p), len(devices)))


def num_devices() -> int:
    return lib.giga_num_devices()


def finalize():
    _check(lib.giga_finalize())


def partition(M: int, ngpus: int, g: int):
    r0, rows = ctypes.c_int64(), ctypes.c_int64()
    _check(lib.giga_partition(M, ngpus, g, ctypes.byref(r0), ctypes.byref(rows)))
    return r0.value, rows.value


def matmul(A, B, C, M: int, N: int, K: int, ngpus: int = 1):
    """giga_matmul: A, B, C all host (numpy / pinned torch) or all device (GPU 0)."""
    _check(lib.giga_matmul(_ptr(A), _ptr(B), _ptr(C), M, N, K, ngpus))


def matmul_sharded(A_shards, B_bufs, C_fulls, M: int, N: int, K: int):
    n = len(C_fulls)
    arr = ctypes.c_void_p * n
    a = arr(*[_ptr(x) if x is not None else None for x in A_shards])
    b = arr(*[_ptr(x) for x in B_bufs])
    c = arr(*[_ptr(x) for x in C_fulls])
    _check(lib.giga_matmul_sharded(ctypes.cast(a, ctypes.c_void_p), ctypes.cast(b, ctypes.c_void_p),
                                   ctypes.cast(c, ctypes.c_void_p), M, N, K, n))


# ---- multi-process API ------------------------------------------------------------------

def comm_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(lib.giga_comm_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
    return bytes(buf)


def rank_init(rank: int, world: int, device: int, uid: bytes | None):
    buf = (ctypes.c_uint8 * 128)(*uid) if uid is not None else None
    _check(lib.giga_rank_init(rank, world, device,
                              ctypes.cast(buf, ctypes.c_void_p) if buf is not None else None))


def p2p_export(B, C_full) -> bytes:
    """giga_rank_p2p_export: this rank's registration blob (CUDA IPC handles)."""
    buf = (ctypes.c_uint8 * P2P_BLOB_BYTES)()
    _check(lib.giga_rank_p2p_export(_ptr(B), _ptr(C_full), ctypes.cast(buf, ctypes.c_void_p)))
    return bytes(buf)


def p2p_import(blobs):
    """giga_rank_p2p_import: every rank's blob, in rank order."""
    raw = b"".join(blobs)
    buf = (ctypes.c_uint8 * len(raw)).from_buffer_copy(raw)
    _check(lib.giga_rank_p2p_import(ctypes.cast(buf, ctypes.c_void_p), len(blobs)))


class _DevBuf:
    """A library-owned device buffer seen through __cuda_array_interface__ (torch.as_tensor
    wraps it without a copy)."""

    def __init__(self, ptr: int, numel: int):
        self.__cuda_array_interface__ = {"shape": (numel,), "typestr": "<f4",
                                         "data": (ptr, False), "version": 3}


def as_float_tensor(ptr: int, numel: int, device):
    """A float32 torch view of `numel` floats at device pointer `ptr` on `device`."""
    import torch
    with torch.cuda.device(device):
        return torch.as_tensor(_DevBuf(ptr, numel), device=device)


def mc_alloc(ngpus: int, nbytes: int):
    """giga_mc_alloc: device pointers (ints) of ngpus C_full buffers bound into one NVLink
    multicast team (GigaError GIGA_ERR_UNSUPPORTED where the driver has no multicast)."""
    out = (ctypes.c_void_p * ngpus)()
    _check(lib.giga_mc_alloc(ngpus, nbytes, ctypes.cast(out, ctypes.c_void_p)))
    return [int(x) for x in out]


def mc_free(C_full0: int):
    _check(lib.giga_mc_free(ctypes.c_void_p(C_full0)))


def rank_mc_alloc(nbytes: int, group=None) -> int:
    """The rank API's multicast C_full (giga_rank_mc_create / _join / _bind, include/giga.h):
    rank 0's blob is broadcast and every phase ends in a barrier over torch.distributed.
    Collective: every rank calls it, and every rank raises if any rank failed."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    blob = (ctypes.c_uint8 * MC_BLOB_BYTES)()
    rc = 0
    if rank == 0:
        rc = lib.giga_rank_mc_create(nbytes, ctypes.cast(blob, ctypes.c_void_p))
    msg = [(rc, last_error() if rc else "", bytes(blob))]
    dist.broadcast_object_list(msg, src=0, group=group)
    rc0, err0, raw = msg[0]
    if rc0:
        raise GigaError(rc0, f"rank 0: {err0}")
    buf = (ctypes.c_uint8 * MC_BLOB_BYTES).from_buffer_copy(raw)
    for phase in ("join", "bind"):
        ptr = ctypes.c_void_p()
        rc = (lib.giga_rank_mc_join(ctypes.cast(buf, ctypes.c_void_p)) if phase == "join"
              else lib.giga_rank_mc_bind(ctypes.byref(ptr)))
        codes = [None] * dist.get_world_size(group)
        dist.all_gather_object(codes, (rc, last_error() if rc else ""), group=group)
        for q, (c, e) in enumerate(codes):
            if c:
                raise GigaError(c, f"rank {q} ({phase}): {e}")
    return int(ptr.value)


def gemm_gather_ex(A, B, C, peers, M: int, N: int, K: int, ldc=None, terms=0, store_mode=0,
                   stream=None):
    """giga_gemm_gather_ex: C (and every peer buffer) = A * B through the fused-gather
    epilogue with store_mode 0 TMA / 1 st.global / 2 multimem.st."""
    arr = (ctypes.c_void_p * max(1, len(peers)))(*[_ptr(q) for q in peers])
    _check(lib.giga_gemm_gather_ex(_ptr(A), _ptr(B), _ptr(C), ctypes.cast(arr, ctypes.c_void_p),
                                   len(peers), M, N, K, N if ldc is None else ldc, terms,
                                   store_mode, _stream(stream)))


def matmul_rank(A_shard, B, C_full, M: int, N: int, K: int, stream=None):
    _check(lib.giga_matmul_rank(_ptr(A_shard), _ptr(B), _ptr(C_full), M, N, K, _stream(stream)))


def dot(x, y, n: int | None = None, ngpus: int = 1) -> float:
    """giga_dot: x, y both host (numpy / torch CPU) or both device (GPU 0)."""
    n = (x.size if isinstance(x, np.ndarray) else x.numel()) if n is None else n
    r = ctypes.c_double()
    _check(lib.giga_dot(_ptr(x), _ptr(y), n, ngpus, ctypes.byref(r)))
    return r.value


def l2norm(x, n: int | None = None, ngpus: int = 1) -> float:
    n = (x.size if isinstance(x, np.ndarray) else x.numel()) if n is None else n
    r = ctypes.c_double()
    _check(lib.giga_l2norm(_ptr(x), n, ngpus, ctypes.byref(r)))
    return r.value


def dot_rank(x_shard, y_shard, n: int, stream=None) -> float:
    r = ctypes.c_double()
    _check(lib.giga_dot_rank(_ptr(x_shard), _ptr(y_shard), n, ctypes.byref(r), _stream(stream)))
    return r.value


def pipeline_plan(M: int, N: int, K: int, world: int):
    """(kbounds, rchunks): B K-chunk bounds and the number of C gather rounds."""
    kc, rc = ctypes.c_int(), ctypes.c_int()
    kb = (ctypes.c_int64 * 17)()
    _check(lib.giga_pipeline_plan(M, N, K, world, ctypes.byref(kc), kb, ctypes.byref(rc)))
    return [kb[i] for i in range(kc.value + 1)], rc.value


def plan_block(M: int, world: int, rchunks: int, owner: int, q: int):
    r0, rows = ctypes.c_int64(), ctypes.c_int64()
    _check(lib.giga_plan_block(M, world, rchunks, owner, q, ctypes.byref(r0), ctypes.byref(rows)))
    return r0.value, rows.value


def rank_compute_only(A_shard, B, C_full, M: int, N: int, K: int, world: int, rank: int,
                      stream=None):
    """Rank `rank`'s GEMM launches of the world-`world` pipeline, without communication."""
    _check(lib.giga_rank_compute_only(_ptr(A_shard), _ptr(B), _ptr(C_full), M, N, K, world,
                                      rank, _stream(stream)))


def gemm_schedule(M: int, N: int, K: int, num_sms: int = 148) -> dict:
    """The tiling and k-split unit schedule of one GEMM launch (see include/giga.h)."""
    out = (ctypes.c_int64 * 8)()
    _check(lib.giga_gemm_schedule(M, N, K, num_sms, out))
    keys = ("cta_group", "tiles", "clusters", "n_kb", "first_split", "s", "units", "mode")
    return dict(zip(keys, list(out)))


def product_scheme(M: int, N: int, K: int) -> int:
    """3 (3xTF32) or 2 (TF32 + BF16): the scheme the product path uses for this launch."""
    t = ctypes.c_int(0)
    _check(lib.giga_product_scheme(M, N, K, ctypes.byref(t)))
    return t.value


def host_plan(M: int, N: int, K: int, num_sms: int = 148):
    """The host-buffer schedule of giga_matmul on one GPU (see include/giga.h)."""
    Me, P, Q, t = ctypes.c_int64(), ctypes.c_int(), ctypes.c_int(), ctypes.c_double()
    kb, rb = (ctypes.c_int64 * 17)(), (ctypes.c_int64 * 17)()
    _check(lib.giga_host_plan(M, N, K, num_sms, ctypes.byref(Me), ctypes.byref(P), kb,
                              ctypes.byref(Q), rb, ctypes.byref(t)))
    return {"Me": Me.value, "kb": list(kb[:P.value + 1]), "rb": list(rb[:Q.value + 1]),
            "t_model": t.value}


# ---- building blocks --------------------------------------------------------------------

def split_lo(x, lo, n: int | None = None, stream=None):
    n = x.numel() if n is None else n
    _check(lib.giga_split_lo(_ptr(x), _ptr(lo), n, _stream(stream)))


def gemm_3xtf32(A, A_lo, B, B_lo, C, M, N, K, ldc=None, terms=3, promote_kblocks=-1,
                cta_group=0, stream=None):
    _check(lib.giga_gemm_3xtf32_ex(_ptr(A), _ptr(A_lo), _ptr(B), _ptr(B_lo), _ptr(C), M, N, K,
                                   N if ldc is None else ldc, terms, promote_kblocks,
                                   cta_group, _stream(stream)))


# ---- timing -----------------------------------------------------------------------------

def timing_enable(on: bool = True):
    _check(lib.giga_timing_enable(1 if on else 0))


def timing_reset():
    _check(lib.giga_timing_reset())


def timing_read():
    gm, sm = ctypes.c_double(), ctypes.c_double()
    gn, sn = ctypes.c_int64(), ctypes.c_int64()
    _check(lib.giga_timing_read(ctypes.byref(gm), ctypes.byref(gn), ctypes.byref(sm),
                                ctypes.byref(sn)))
    return {"gemm_ms": gm.value, "gemm_launches": gn.value, "split_ms": sm.value,
            "split_launches": sn.value}
