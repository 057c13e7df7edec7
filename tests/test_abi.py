"""CPU-side checks of the C ABI: the library loads, exports every symbol include/giga.h
declares, and its pure host logic (partition rule, argument validation) behaves."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "giga.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(giga_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def giga():
    from paper_2504_01266_b200 import build
    build.build()
    from paper_2504_01266_b200 import giga as g
    return g


def test_exports_every_declared_symbol(giga):
    declared = _declared()
    assert len(declared) >= 15
    lib = ctypes.CDLL(giga.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(giga.EXPORTS)


def test_library_is_sm100a_and_uses_tcgen05(giga):
    import subprocess
    sass = subprocess.run(["cuobjdump", "-sass", giga.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", giga.LIB_PATH],
                                       capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass


@pytest.mark.parametrize("M,ng", [(10, 1), (10, 3), (2, 4), (0, 2), (16384, 8), (7, 7)])
def test_partition_rule(giga, M, ng):
    # contiguous blocks, floor split, the last device takes the remainder
    rows = [giga.partition(M, ng, g) for g in range(ng)]
    assert rows[0][0] == 0
    for g in range(1, ng):
        assert rows[g][0] == rows[g - 1][0] + rows[g - 1][1]
    assert rows[-1][0] + rows[-1][1] == M
    base = M // ng
    assert all(r[1] == base for r in rows[:-1])
    assert rows[-1][1] == M - (ng - 1) * base


def test_partition_bad_args(giga):
    for args in [(-1, 2, 0), (10, 0, 0), (10, 2, 2), (10, 2, -1)]:
        with pytest.raises(giga.GigaError) as e:
            giga.partition(*args)
        assert e.value.status == "GIGA_ERR_INVALID_ARG"


def test_not_initialized_paths(giga):
    import numpy as np
    a = np.ones((2, 2), np.float32)
    with pytest.raises(giga.GigaError) as e:
        giga.matmul(a, a, np.empty_like(a), 2, 2, 2, 1)
    assert e.value.status == "GIGA_ERR_NOT_INITIALIZED"
    with pytest.raises(giga.GigaError) as e:
        giga.matmul_rank(a, a, a, 2, 2, 2)
    assert e.value.status == "GIGA_ERR_NOT_INITIALIZED"
    # multicast teams (N4) need an initialised library; no driver call is made before that
    with pytest.raises(giga.GigaError) as e:
        giga.mc_alloc(1, 1 << 20)
    assert e.value.status == "GIGA_ERR_NOT_INITIALIZED"
    import ctypes
    blob = (ctypes.c_uint8 * giga.MC_BLOB_BYTES)()
    assert giga.lib.giga_rank_mc_create(1 << 20, blob) == -2
    assert giga.lib.giga_rank_mc_join(blob) == -2
    assert giga.lib.giga_rank_mc_bind(ctypes.byref(ctypes.c_void_p())) == -2
    with pytest.raises(giga.GigaError) as e:
        giga.mc_free(4096)
    assert e.value.status == "GIGA_ERR_INVALID_ARG"
    giga.finalize()  # finalize when not initialised is OK


def test_init_without_gpu_reports_no_device(giga):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by tests/test_gpu.py")
    with pytest.raises(giga.GigaError) as e:
        giga.init(1)
    assert e.value.status == "GIGA_ERR_NO_DEVICE"
    assert giga.num_devices() == 0


def test_product_scheme_selection():
    """giga_product_scheme (host-only): 3xFP16 where its per-launch operand preparation is
    amortised (>= 2^35 multiply-adds, K >= 512), 3xTF32 for the small, shallow and thin configs
    (profiles/r02_scheme_crossover_e.jsonl). TF32 + BF16 is forced only."""
    from paper_2504_01266_b200 import giga
    for shape in [(16384, 16384, 16384), (32768, 32768, 32768), (4096, 32768, 32768),
                  (8192, 8192, 2048), (2048, 16384, 16384), (16384, 32768, 1024),
                  (65536, 2048, 2048), (8192, 16384, 1024), (4096, 4096, 4096),
                  (32768, 1024, 1024), (262144, 1024, 1024), (2048, 4096, 4096),
                  (16384, 32768, 576), (32768, 16384, 1000), (65536, 4096, 512),
                  (4096, 32768, 768)]:
        assert giga.product_scheme(*shape) == 4, shape
    for shape in [(512, 512, 512), (2048, 2048, 2048), (16384, 16384, 256),
                  (1024, 32768, 32768), (4096, 4096, 1024), (32768, 512, 2048)]:
        assert giga.product_scheme(*shape) == 3, shape
    with pytest.raises(Exception):
        giga.product_scheme(0, 4, 4)
