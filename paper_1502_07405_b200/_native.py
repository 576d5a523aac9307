"""ctypes loader for libhssmf_b200.so (the C-ABI of include/hssmf_b200.h).

The product path has no CPU fallback: if the shared library is missing this
module raises at import time of any numeric entry point.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhssmf_b200.so")

i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
f64c = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
vp = C.c_void_p


class Status(C.Structure):
    _fields_ = [("code", C.c_int), ("front", C.c_int), ("column", C.c_int),
                ("msg", C.c_char * 512)]


class ProbeStat(C.Structure):
    _fields_ = [("launches", C.c_longlong), ("ms", C.c_double), ("flops", C.c_double),
                ("bytes", C.c_double)]


class Options(C.Structure):
    _fields_ = [("ls", C.c_int), ("eps", C.c_double), ("leaf", C.c_int), ("d0", C.c_int),
                ("dd", C.c_int), ("p", C.c_int), ("min_hss", C.c_int),
                ("max_rank", C.c_int), ("mode", C.c_int)]


_lib = None

_SIGS = {
    "hssmf_version": (C.c_char_p, []),
    "hssmf_launch_count": (C.c_longlong, []),
    "hssmf_csr_grid": (C.c_int, [C.c_int, C.c_int, C.c_double, C.POINTER(vp), i32p,
                                 C.POINTER(C.c_int), C.POINTER(Status)]),
    "hssmf_csr_convdiff3d": (C.c_int, [C.c_int, C.c_double, C.POINTER(vp), C.POINTER(Status)]),
    "hssmf_csr_create": (C.c_int, [C.c_int, i32p, i32p, f64c, C.POINTER(vp),
                                   C.POINTER(Status)]),
    "hssmf_csr_permuted": (C.c_int, [vp, i32p, C.POINTER(vp), C.POINTER(Status)]),
    "hssmf_csr_info": (None, [vp, C.POINTER(C.c_int), C.POINTER(C.c_longlong)]),
    "hssmf_csr_get": (None, [vp, i32p, i32p, f64c]),
    "hssmf_csr_matvec": (None, [vp, f64c, f64c]),
    "hssmf_csr_free": (None, [vp]),
    "hssmf_nd_geometric": (C.c_int, [i32p, C.c_int, C.c_int, i32p, C.POINTER(vp),
                                     C.POINTER(Status)]),
    "hssmf_tree_create": (C.c_int, [C.c_int, C.c_int, i32p, i32p, i32p, i32p, i32p, vp, vp,
                                    C.POINTER(vp), C.POINTER(Status)]),
    "hssmf_symbolic": (C.c_int, [vp, vp, C.POINTER(Status)]),
    "hssmf_tree_info": (None, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int),
                               C.POINTER(C.c_longlong)]),
    "hssmf_tree_get": (None, [vp, i32p, i32p, i32p, i32p, i32p, i32p, i32p, i32p]),
    "hssmf_tree_free": (None, [vp]),
    "hssmf_csr_read_mm": (C.c_int, [C.c_char_p, C.POINTER(vp), C.POINTER(Status)]),
    "hssmf_csr_write_mm": (C.c_int, [vp, C.c_char_p, C.POINTER(Status)]),
    "hssmf_equilibrate": (C.c_int, [vp, C.POINTER(vp), vp, vp, vp, C.POINTER(C.c_int),
                                    C.POINTER(Status)]),
    "hssmf_nd_graph": (C.c_int, [vp, C.c_int, i32p, C.POINTER(vp), C.POINTER(Status)]),
    "hssmf_reorder_separators": (C.c_int, [vp, vp, vp, C.c_int, i32p, C.POINTER(Status)]),
    "hssmf_tree_sep_clusters": (C.c_int, [vp, C.c_int, vp, vp, vp, vp, vp]),
    "hssmf_tree_set_sep_clusters": (C.c_int, [vp, C.c_int, C.c_int, vp, vp, vp, vp,
                                              C.POINTER(Status)]),
    "hssmf_front_cluster_tree": (C.c_int, [C.c_int, C.c_int, C.c_int, vp, vp, vp, vp, vp]),
    "hssmf_factor": (C.c_int, [C.c_int, vp, vp, C.POINTER(Options), C.POINTER(vp),
                               C.POINTER(Status)]),
    "hssmf_refactor": (C.c_int, [vp, vp, C.c_int, C.POINTER(Status)]),
    "hssmf_gmres": (C.c_int, [vp, vp, vp, vp, C.c_int, C.c_double, C.c_double, C.c_int, vp, vp,
                              C.c_int, C.POINTER(Status)]),
    "hssmf_refine": (C.c_int, [vp, vp, vp, vp, C.c_double, C.c_double, C.c_int, vp, vp, C.c_int,
                               C.POINTER(Status)]),
    "hssmf_analyze_owned": (C.c_int, [C.c_int, vp, vp, vp, vp, C.POINTER(vp), C.POINTER(Status)]),
    "hssmf_nlevels": (C.c_int, [vp]),
    "hssmf_factor_levels": (C.c_int, [vp, C.c_int, C.c_int, C.POINTER(Status)]),
    "hssmf_update_export": (C.c_int, [vp, C.c_int, vp, C.c_int, C.POINTER(Status)]),
    "hssmf_update_import": (C.c_int, [vp, C.c_int, vp, C.c_int, C.POINTER(Status)]),
    "hssmf_bupd_export": (C.c_int, [vp, C.c_int, vp, C.c_int, C.POINTER(Status)]),
    "hssmf_bupd_import": (C.c_int, [vp, C.c_int, vp, C.c_int, C.POINTER(Status)]),
    "hssmf_solve_levels": (C.c_int, [vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                     C.POINTER(Status)]),
    "hssmf_solve": (C.c_int, [vp, vp, C.c_int, C.c_int, C.c_int, C.POINTER(Status)]),
    "hssmf_factor_summary": (None, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                    C.POINTER(C.c_int), C.POINTER(C.c_int),
                                    C.POINTER(C.c_longlong)]),
    "hssmf_front_stats": (None, [vp, i32p, i32p, i32p, i32p, i64p, i32p]),
    "hssmf_front_hss": (C.c_int, [vp, C.c_int, vp, vp, C.POINTER(C.c_int),
                                  C.POINTER(C.c_int)]),
    "hssmf_timing": (None, [vp, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "hssmf_set_profile": (None, [vp, C.c_int]),
    "hssmf_kernel_stats": (C.c_int, [vp, C.c_int, C.c_char_p, i32p, f64c, f64c, f64c]),
    "hssmf_reset_kernel_stats": (None, [vp]),
    "hssmf_device_bytes": (C.c_longlong, [vp]),
    "hssmf_factors_free": (None, [vp]),
    "hssmf_hss_dense": (C.c_int, [C.c_int, vp, C.c_int, C.c_int, C.c_int, C.c_double,
                                  C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(vp),
                                  C.POINTER(Status)]),
    "hssmf_hss_dense_tree": (C.c_int, [C.c_int, vp, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp,
                                       C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.POINTER(vp), C.POINTER(Status)]),
    "hssmf_hss_matvec": (C.c_int, [vp, C.c_char, C.c_int, vp, C.c_int, C.c_int, C.c_int, vp,
                                   C.c_int, C.c_int, C.POINTER(Status)]),
    "hssmf_hss_extract": (C.c_int, [vp, vp, C.c_int, vp, C.c_int, vp, C.c_int,
                                    C.POINTER(C.c_longlong), C.POINTER(Status)]),
    "hssmf_mgpu_partition": (C.c_int, [vp, C.c_int, vp, C.POINTER(C.c_int), C.POINTER(Status)]),
    "hssmf_mgpu_factor": (C.c_int, [C.c_int, vp, vp, vp, C.c_int, C.c_int, vp, C.POINTER(vp),
                                    C.POINTER(Status)]),
    "hssmf_mgpu_solve": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.POINTER(Status)]),
    "hssmf_mgpu_local": (C.c_int, [C.c_int, vp, vp, vp, C.c_int, vp, C.c_int, C.POINTER(Status)]),
    "hssmf_hss_info": (C.c_int, [vp, vp, vp, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                 C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "hssmf_hss_solve": (C.c_int, [vp, vp, C.c_int, C.c_int, C.c_int, C.POINTER(Status)]),
    "hssmf_hss_free": (None, [vp]),
    "hssmf_dev_random_rows": (C.c_int, [C.c_int, C.c_int, i64p, C.c_int, C.c_int, vp,
                                        C.POINTER(Status)]),
    "hssmf_dev_gemm": (C.c_int, [C.c_int, C.c_char, C.c_char, C.c_int, C.c_int, C.c_int,
                                 C.c_double, vp, C.c_int, vp, C.c_int, C.c_double, vp,
                                 C.c_int, C.POINTER(Status)]),
    "hssmf_dev_id": (C.c_int, [C.c_int, vp, C.c_int, C.c_int, C.c_double, C.c_int,
                               C.c_double, i32p, C.POINTER(C.c_int), C.POINTER(C.c_int), vp,
                               C.POINTER(Status)]),
    "hssmf_dev_gram_id": (C.c_int, [C.c_int, vp, C.c_int, C.c_int, C.c_double, C.c_int,
                                    C.c_double, i32p, C.POINTER(C.c_int), C.POINTER(C.c_int), vp,
                                    C.POINTER(Status)]),
    "hssmf_dev_lu": (C.c_int, [C.c_int, vp, C.c_int, C.c_int, i32p, C.POINTER(Status)]),
    "hssmf_probe_enable": (C.c_int, [C.c_int, C.POINTER(Status)]),
    "hssmf_probe_read": (C.c_int, [C.POINTER(ProbeStat), C.POINTER(Status)]),
    "hssmf_bench_gemm": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.POINTER(C.c_double), C.POINTER(Status)]),
    "hssmf_bench_gram": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(Status)]),
}


def exported_symbols():
    return list(_SIGS)


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"hssmf_b200 native library missing: {LIB_PATH}. Build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists).")
    L = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L
