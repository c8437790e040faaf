"""ctypes binding of libmdr_b200.so (the C-ABI of include/mdr.h).

There is no CPU fallback: if the library is missing or no CUDA device is
present, loading fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# MDR_LIB_PATH selects an experiment build (variants/<name>/, see build.py)
LIB_PATH = os.environ.get("MDR_LIB_PATH") or os.path.join(HERE, "libmdr_b200.so")

_lib = None

P = C.c_void_p
I = C.c_int
D = C.c_double
F = C.c_float
U64 = C.c_uint64
SZ = C.c_size_t

# name -> (restype, argtypes)
_SIGS = {
    "mdr_version": (C.c_char_p, []),
    "mdr_phase_prof": (I, [P, I]),
    "mdr_phase_prof_sm": (I, [P, I]),
    "mdr_ctx_create": (P, [I]),
    "mdr_ctx_destroy": (None, [P]),
    "mdr_ctx_set_stream": (I, [P, P]),
    "mdr_ctx_stream": (P, [P]),
    "mdr_ctx_set_pair_precision": (I, [P, I]),
    "mdr_ctx_set_warps_per_block": (I, [P, I]),
    "mdr_ctx_set_cta_warps": (I, [P, I]),
    "mdr_ctx_set_exact_torsion": (I, [P, I]),
    "mdr_site_chunking": (I, [I, I, I, P, P]),
    "mdr_search_chunking": (I, [I, I, I, I, P, P, P]),
    "mdr_ctx_set_ls_warps": (I, [P, I]),
    "mdr_last_error": (C.c_char_p, [P]),
    "mdr_ctx_launch_count": (U64, [P]),
    "mdr_ctx_synchronize": (I, [P]),
    "mdr_f32_to_half_batch": (I, [P, P, SZ, P]),
    "mdr_half_to_f32_batch": (I, [P, P, SZ, P]),
    "mdr_mma_batch": (I, [P, P, P, P, I, I, P]),
    "mdr_reduce4_batch": (I, [P, P, I, I, I, I, P, P]),
    "mdr_block_reduce_batch": (I, [P, P, I, I, P, P]),
    "mdr_warp_reduce_batch": (I, [P, P, I, P, P]),
    "mdr_reduce7_batch": (I, [P, P, I, I, I, I, P, P]),
    "mdr_reduce4_dev": (I, [P, P, I, I, I, I, P]),
    "mdr_reduce7_dev": (I, [P, P, I, I, I, I, P]),
    "mdr_reduce_uses_tc05": (I, [P, I, I, I]),
    "mdr_ctx_set_tc05": (I, [P, I]),
    "mdr_score_batch": (I, [P, P, P, I, I, I, I, P, P, P, P]),
    "mdr_score_reference_batch": (I, [P, P, P, I, P, P, P]),
    "mdr_adadelta_step_batch": (I, [P, I, I, D, D, P, P, P, P]),
    "mdr_local_search_batch": (I, [P, P, P, I, I, D, I, I, I, P, P, P, P, P]),
    "mdr_lga_defaults": (None, [P]),
    "mdr_lga_max_records": (I, [P]),
    "mdr_lga_run_batch": (I, [P, P, I, I, P, P, I, P, P, P, P, P, P, P]),
    "mdr_instance_upload": (P, [P, P]),
    "mdr_instance_free": (None, [P, P]),
    "mdr_score_dev": (I, [P, P, P, I, I, I, I, P, P, P]),
    "mdr_local_search_dev": (I, [P, P, P, I, I, D, I, I, I, P, P, P, P, P]),
    "mdr_lga_batch_create": (P, [P, P, I, I, P, I]),
    "mdr_lga_batch_destroy": (None, [P, P]),
    "mdr_lga_batch_run_dev": (I, [P, P, P]),
    "mdr_lga_batch_download": (I, [P, P, P, P, P, P, P, P, P]),
    "mdr_lga_batch_total_evals_dev": (I, [P, P, P]),
    "mdr_lga_batch_profile_dev": (I, [P, P, P, P, P, P]),
    "mdr_selftest_ddiv": (I, [P, U64, C.c_int64, P]),
    "mdr_selftest_dsqrt": (I, [P, U64, C.c_int64, P]),
    "mdr_selftest_sincos": (I, [P, U64, C.c_int64, P]),
    "mdr_selftest_crmath": (I, [P, C.c_int64, P]),
    "mdr_crmath_values": (I, [P, C.c_int64, I, P]),
    "mdr_reduce_bench_dev": (I, [P, I, I, P, I, I, P]),
    "mdr_fill_uniform_dev": (I, [P, U64, C.c_char_p, C.c_int64, P]),
    "mdr_reduce_bench_chain_cycles_dev": (I, [P, I, I, P, I, I, P, P]),
    "mdr_reduce_bench_kernels": (I, []),
    "mdr_reduce_bench_kernel_name": (C.c_char_p, [I]),
    "mdr_grid_upload": (P, [P, P]),
    "mdr_grid_build": (P, [P, P, P, P]),
    "mdr_grid_download": (I, [P, P, P]),
    "mdr_grid_free": (None, [P, P]),
    "mdr_instance_set_grid": (I, [P, P, P, P]),
    "mdr_grid_score_batch": (I, [P, P, P, P, P, I, I, I, P, P, P]),
    "mdr_grid_local_search_batch": (I, [P, P, P, P, P, I, I, D, I, I, P, P, P, P]),
    "mdr_grid_lga_run_batch": (I, [P, P, P, P, I, P, P, I, P, P, P, P, P, P]),
    "mdr_pose_coords_batch": (I, [P, P, P, I, P]),
    "mdr_grid_screen_batch": (I, [P, P, P, P, I, I, I, P, P, D, P, P, P, P, P, P, P]),
    "mdr_multi_lga_run_batch": (I, [P, I, P, I, I, I, P, P, I, P, P, P, P]),
    "mdr_multi_screen": (I, [P, I, P, P, P, P, P, I, I, I, P, P, D, I, P, P, P, P, P, P]),
    "mdr_multi_last_error": (C.c_char_p, []),
    "mdr_multi_set_fault_injection": (None, [I, I]),
    "mdr_cluster_poses": (I, [P, P, P, P, I, D, P, P, P]),
    "mdr_cluster_segments_dev": (I, [P, P, P, P, P, I, I, D, P, P, P]),
    "mdr_lga_batch_cluster": (I, [P, P, D, P, P, P]),
}

# Optional entry points (present once their module is built).
_OPTIONAL = {
    "mdr_reduce_bench_dev": (I, [P, I, I, P, I, I, P]),
    "mdr_reduce_bench_kernels": (I, []),
    "mdr_reduce_bench_kernel_name": (C.c_char_p, [I]),
}


def exported_symbols():
    return sorted(_SIGS)


def load():
    """Load the library (build it first if it is missing, e.g. a fresh
    checkout on a box that has nvcc)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        from . import build

        build.build()
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    for name, (res, args) in _OPTIONAL.items():
        if hasattr(lib, name):
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
    _lib = lib
    return lib
