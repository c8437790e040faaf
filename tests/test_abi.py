"""The C-ABI boundary (include/mdr.h): the built library loads without a GPU
and exports every function the header declares, and the Python binding
declares a prototype for each of them.  No compute calls (CPU suite)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "mdr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mdr_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_function():
    from paper_2410_10447_b200 import build

    lib = ctypes.CDLL(build.build())
    names = header_functions()
    assert len(names) > 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    from paper_2410_10447_b200 import _lib

    declared = set(_lib.exported_symbols()) | set(_lib._OPTIONAL)
    missing = [n for n in header_functions() if n not in declared]
    assert not missing, missing


def test_site_chunking_policy():
    """Host-only policy of the chunked site mapping (capi.cpp pick_chunks):
    FP64-fast only, chunk lengths a multiple of the 8-site batch, at most 256
    (atom, chunk) items, lane per atom when chunking does not pay."""
    from paper_2410_10447_b200 import PAIR_FP32, PAIR_FP64, PAIR_FP64_FAST, build

    lib = ctypes.CDLL(build.build())

    def pick(pair, na, ns):
        n, ln = ctypes.c_int(), ctypes.c_int()
        assert lib.mdr_site_chunking(pair, na, ns, ctypes.byref(n), ctypes.byref(ln)) == 0
        return n.value, ln.value

    def pick_search(pair, na, ns, warps, group=False):
        n, ln, g = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        assert lib.mdr_search_chunking(pair, na, ns, warps, ctypes.byref(n), ctypes.byref(ln), ctypes.byref(g)) == 0
        return (n.value, ln.value, g.value) if group else (n.value, ln.value)

    assert pick(PAIR_FP64_FAST, 20, 64) == (3, 24)  # C3 on one warp: 60 items in 2 rounds of 24 sites
    # C3's search on 2 warps: 8 chunks of 8 sites, one atom per item (160 items, 3 rounds of 64 lanes)
    assert pick_search(PAIR_FP64_FAST, 20, 64, 2, group=True) == (8, 8, 1)
    assert pick_search(PAIR_FP64_FAST, 20, 64, 3, group=True) == (8, 8, 1)  # the pooled form: same policy
    assert pick_search(PAIR_FP64_FAST, 20, 64, 1) == pick(PAIR_FP64_FAST, 20, 64)
    assert pick(PAIR_FP64, 20, 64) == (1, 64)
    assert pick(PAIR_FP32, 20, 64) == (1, 64)
    assert pick_search(PAIR_FP32, 20, 64, 2) == (1, 64)
    assert pick(PAIR_FP64_FAST, 200, 64) == (1, 64)  # items would exceed 256
    assert pick(PAIR_FP64_FAST, 20, 6) == (1, 6)  # fewer sites than one batch
    for warps in (1, 2):
        for na in (1, 5, 16, 31, 40, 100, 128):
            for ns in (8, 30, 64, 200):
                n, ln, g = pick_search(PAIR_FP64_FAST, na, ns, warps, group=True)
                if n > 1:
                    # the warp-per-pose policy stages at most 256 items, the two-warp search 512
                    assert ln % 8 == 0 and na * n <= (256 if warps == 1 else 512) and (n - 1) * ln < ns <= n * ln
                    if warps == 1:
                        assert g == 1 and ((na * n + 31) // 32) * (ln + 4) < ((na + 31) // 32) * ns
                    else:
                        assert g in (1, 3) and na * n > 32
                        assert ((-(-na // g) * n + 63) // 64) * g * ln < ((na + 31) // 32) * ns
    assert lib.mdr_search_chunking(PAIR_FP64_FAST, 20, 64, 4, ctypes.byref(ctypes.c_int()),
                                   ctypes.byref(ctypes.c_int()), None) != 0
    assert lib.mdr_site_chunking(7, 20, 64, ctypes.byref(ctypes.c_int()), ctypes.byref(ctypes.c_int())) != 0
