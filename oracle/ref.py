"""ORACLE — test infrastructure only (never imported by the product path).

ctypes bindings to oracle/_ref/libhssmf_ref.so, the UNMODIFIED reference
(/root/reference/proj) compiled in place by oracle/Makefile plus the
extern "C" shim in oracle/ref_driver.cpp (one semantics-preserving
specialization of LowRankSchur<double>::extract, see that file's header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libhssmf_ref.so")

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="F_CONTIGUOUS")
_f64c = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

_lib = None

GRID_KINDS = {"p2d": 0, "p3d": 1, "c2d": 2, "c3d": 3}
FRONT_TYPES = {0: "dense", 1: "hss", 2: "hss_dense"}


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not available():
        raise RuntimeError(f"oracle library missing: {LIB_PATH} (run make -C oracle)")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    sig = {
        "ref_last_error": (C.c_char_p, []),
        "ref_set_threads": (None, [C.c_int]),
        "ref_num_threads": (C.c_int, []),
        "ref_flops": (C.c_longlong, []),
        "ref_reset_counters": (None, []),
        "ref_sampler_value": (C.c_double, [C.c_longlong, C.c_longlong]),
        "ref_random_rows": (None, [C.c_int, _i64p, C.c_int, C.c_int, _f64p]),
        "ref_grid": (vp, [C.c_int, C.c_int, C.c_double]),
        "ref_grid_free": (None, [vp]),
        "ref_grid_n": (C.c_int, [vp]),
        "ref_grid_nnz": (C.c_longlong, [vp]),
        "ref_grid_csr": (None, [vp, _i32p, _i32p, _f64c]),
        "ref_ordered_grid": (vp, [C.c_int, C.c_int, C.c_double, C.c_int]),
        "ref_ordered_csr_geom": (vp, [C.c_int, _i32p, _i32p, _f64c, C.c_int, C.c_int,
                                      C.c_int, C.c_int, C.c_int]),
        "ref_ordered_from_arrays": (vp, [C.c_int, _i32p, _i32p, _f64c, C.c_int, _i32p,
                                         _i32p, _i32p, _i32p, _i32p, _i32p, _i32p]),
        "ref_ordered_graph": (vp, [C.c_int, _i32p, _i32p, _f64c, C.c_int, C.c_int, vp]),
        "ref_ordered_sep_clusters": (C.c_int, [vp, C.c_int, vp, vp, vp, vp, vp]),
        "ref_equilibrate": (C.c_int, [C.c_int, _i32p, _i32p, _f64c, _i32p, _f64c, _f64c, _f64c,
                                      _i32p, C.POINTER(C.c_int)]),
        "ref_read_mm": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_longlong), vp,
                                  vp, vp]),
        "ref_ordered_free": (None, [vp]),
        "ref_ordered_n": (C.c_int, [vp]),
        "ref_ordered_nnz": (C.c_longlong, [vp]),
        "ref_ordered_csr": (None, [vp, _i32p, _i32p, _f64c]),
        "ref_ordered_perm": (None, [vp, _i32p]),
        "ref_ordered_nnodes": (C.c_int, [vp]),
        "ref_ordered_upd_total": (C.c_longlong, [vp]),
        "ref_ordered_tree": (None, [vp, _i32p, _i32p, _i32p, _i32p, _i32p, _i32p, _i32p,
                                    _i32p]),
        "ref_factor": (vp, [vp, _i32p, C.c_double, C.POINTER(C.c_int),
                            C.POINTER(C.c_int), C.POINTER(C.c_int)]),
        "ref_factor_free": (None, [vp]),
        "ref_factor_seconds": (C.c_double, [vp]),
        "ref_factor_summary": (None, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                      C.POINTER(C.c_int), C.POINTER(C.c_longlong)]),
        "ref_front_stats": (None, [vp, _i32p, _i32p, _i32p, _i32p, _i64p, _i32p]),
        "ref_front_hss": (C.c_int, [vp, C.c_int, C.c_void_p, C.c_void_p,
                                    C.POINTER(C.c_int), C.POINTER(C.c_int)]),
        "ref_solve": (C.c_double, [vp, _f64p, C.c_int]),
        "ref_hss_dense": (vp, [_f64p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int,
                               C.c_int, C.c_int, C.POINTER(C.c_int)]),
        "ref_hss_free": (None, [vp]),
        "ref_hss_info": (C.c_int, [vp, C.c_void_p, C.c_void_p, C.POINTER(C.c_int),
                                   C.POINTER(C.c_int), C.POINTER(C.c_double),
                                   C.POINTER(C.c_double)]),
        "ref_hss_solve": (C.c_double, [vp, _f64p, C.c_int]),
        "ref_hss_matvec": (None, [vp, _f64p, _f64p, C.c_int]),
        "ref_lu": (C.c_int, [_f64p, C.c_int, C.c_int, _i32p]),
        "ref_id": (None, [_f64p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_double,
                          _i32p, C.POINTER(C.c_int), C.POINTER(C.c_int), _f64p]),
        "ref_cluster_front": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.c_void_p]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def set_threads(t: int) -> None:
    lib().ref_set_threads(int(t))


def sampler_value(row: int, col: int) -> float:
    return lib().ref_sampler_value(row, col)


def random_rows(grow, c0: int, c1: int) -> np.ndarray:
    g = np.ascontiguousarray(grow, dtype=np.int64)
    out = np.zeros((len(g), c1 - c0), dtype=np.float64, order="F")
    lib().ref_random_rows(len(g), g, c0, c1, out)
    return out


def grid_csr(kind: str, k: int, nu: float = 1e-4):
    L = lib()
    h = L.ref_grid(GRID_KINDS[kind], k, nu)
    n, nnz = L.ref_grid_n(h), L.ref_grid_nnz(h)
    ptr = np.zeros(n + 1, np.int32)
    ind = np.zeros(nnz, np.int32)
    val = np.zeros(nnz, np.float64)
    L.ref_grid_csr(h, ptr, ind, val)
    L.ref_grid_free(h)
    return ptr, ind, val


class Ordered:
    """permuted matrix + elimination tree with symbolic structure"""

    def __init__(self, handle):
        self.h = handle
        L = lib()
        self.n = L.ref_ordered_n(handle)
        nnz = L.ref_ordered_nnz(handle)
        self.ptr = np.zeros(self.n + 1, np.int32)
        self.ind = np.zeros(nnz, np.int32)
        self.val = np.zeros(nnz, np.float64)
        L.ref_ordered_csr(handle, self.ptr, self.ind, self.val)
        self.perm = np.zeros(self.n, np.int32)
        L.ref_ordered_perm(handle, self.perm)
        nn = L.ref_ordered_nnodes(handle)
        tot = L.ref_ordered_upd_total(handle)
        z = lambda k: np.zeros(k, np.int32)  # noqa: E731
        self.sep_begin, self.sep_end, self.child0, self.child1 = z(nn), z(nn), z(nn), z(nn)
        self.parent, self.level, self.upd_ptr, self.upd_ind = z(nn), z(nn), z(nn + 1), z(tot)
        L.ref_ordered_tree(handle, self.sep_begin, self.sep_end, self.child0, self.child1,
                           self.parent, self.level, self.upd_ptr, self.upd_ind)

    @property
    def nnodes(self):
        return len(self.sep_begin)

    def sep_clusters(self, i):
        L = lib()
        nn = L.ref_ordered_sep_clusters(self.h, int(i), None, None, None, None, None)
        arr = [np.zeros(nn, np.int32) for _ in range(5)]
        L.ref_ordered_sep_clusters(self.h, int(i), *[x.ctypes.data_as(C.c_void_p) for x in arr])
        return arr

    def __del__(self):
        try:
            if self.h:
                lib().ref_ordered_free(self.h)
                self.h = None
        except Exception:
            pass


def ordered_grid(kind: str, k: int, nd_leaf: int, nu: float = 1e-4) -> Ordered:
    return Ordered(lib().ref_ordered_grid(GRID_KINDS[kind], k, nu, nd_leaf))


def ordered_csr_geom(ptr, ind, val, dims, ndims, nd_leaf) -> Ordered:
    n = len(ptr) - 1
    return Ordered(lib().ref_ordered_csr_geom(
        n, np.ascontiguousarray(ptr, np.int32), np.ascontiguousarray(ind, np.int32),
        np.ascontiguousarray(val, np.float64), dims[0], dims[1], dims[2], ndims, nd_leaf))


def equilibrate(ptr, ind, val):
    """reference equilibrate_and_permute: (ind, val, dr, dc, qc, sweeps) or
    raises RefError(9) when structurally singular"""
    n = len(ptr) - 1
    ptr = np.ascontiguousarray(ptr, np.int32)
    oi = np.zeros(len(ind), np.int32)
    ov = np.zeros(len(ind), np.float64)
    dr, dc = np.zeros(n), np.zeros(n)
    qc = np.zeros(n, np.int32)
    sw = C.c_int()
    rc = lib().ref_equilibrate(n, ptr, np.ascontiguousarray(ind, np.int32),
                               np.ascontiguousarray(val, np.float64), oi, ov, dr, dc, qc,
                               C.byref(sw))
    if rc:
        raise RefError(rc, -1, -1, lib().ref_last_error().decode())
    return oi, ov, dr, dc, qc, sw.value


def read_mm(path):
    """reference read_matrix_market: (ptr, ind, val) or raises RefError(1)"""
    L = lib()
    n, nnz = C.c_int(), C.c_longlong()
    rc = L.ref_read_mm(os.fsencode(path), C.byref(n), C.byref(nnz), None, None, None)
    if rc:
        raise RefError(rc, -1, -1, L.ref_last_error().decode())
    ptr = np.zeros(n.value + 1, np.int32)
    ind = np.zeros(nnz.value, np.int32)
    val = np.zeros(nnz.value, np.float64)
    L.ref_read_mm(os.fsencode(path), C.byref(n), C.byref(nnz), ptr.ctypes.data_as(C.c_void_p),
                  ind.ctypes.data_as(C.c_void_p), val.ctypes.data_as(C.c_void_p))
    return ptr, ind, val


def ordered_graph(ptr, ind, val, nd_leaf, reorder_b=0, selected=None) -> Ordered:
    """graph ND pipeline of the reference (+ separator reordering)"""
    n = len(ptr) - 1
    sel = None
    if selected is not None:
        sel = np.ascontiguousarray(np.asarray(selected, bool).astype(np.int8))
    o = Ordered(lib().ref_ordered_graph(
        n, np.ascontiguousarray(ptr, np.int32), np.ascontiguousarray(ind, np.int32),
        np.ascontiguousarray(val, np.float64), int(nd_leaf), int(reorder_b),
        sel.ctypes.data_as(C.c_void_p) if sel is not None else None))
    o._keep = sel
    return o


def ordered_from_arrays(n, ptr, ind, val, sep_begin, sep_end, child0, child1, parent,
                        upd_ptr, upd_ind) -> Ordered:
    a = lambda x: np.ascontiguousarray(x, np.int32)  # noqa: E731
    return Ordered(lib().ref_ordered_from_arrays(
        n, a(ptr), a(ind), np.ascontiguousarray(val, np.float64), len(sep_begin),
        a(sep_begin), a(sep_end), a(child0), a(child1), a(parent), a(upd_ptr), a(upd_ind)))


class RefError(RuntimeError):
    def __init__(self, status, front, col, msg):
        super().__init__(msg)
        self.status, self.front, self.column = status, front, col


def options_array(ls=0, leaf=128, d0=128, dd=128, p=10, min_hss=512, max_rank=0, mode=0):
    return np.array([ls, leaf, d0, dd, p, min_hss, max_rank, mode], np.int32)


class Factors:
    def __init__(self, ordered: Ordered, eps=1e-8, **kw):
        L = lib()
        self.ordered = ordered
        st, fr, col = C.c_int(0), C.c_int(0), C.c_int(0)
        self.h = L.ref_factor(ordered.h, options_array(**kw), eps, C.byref(st), C.byref(fr),
                              C.byref(col))
        if not self.h:
            raise RefError(st.value, fr.value, col.value, L.ref_last_error().decode())
        self.factor_seconds = L.ref_factor_seconds(self.h)
        hf, fb, mr, nz = C.c_int(), C.c_int(), C.c_int(), C.c_longlong()
        L.ref_factor_summary(self.h, C.byref(hf), C.byref(fb), C.byref(mr), C.byref(nz))
        self.hss_fronts, self.fallbacks, self.max_front_rank = hf.value, fb.value, mr.value
        self.factor_nnz = nz.value
        nn = ordered.nnodes
        z = lambda: np.zeros(nn, np.int32)  # noqa: E731
        self.level, self.dim, self.sep, self.rank, self.type = z(), z(), z(), z(), z()
        self.flops = np.zeros(nn, np.int64)
        L.ref_front_stats(self.h, self.level, self.dim, self.sep, self.rank, self.flops,
                          self.type)

    def front_hss(self, front):
        """per HSS node (u_rank, v_rank), rounds, d_final; None for dense fronts"""
        L = lib()
        nn = L.ref_front_hss(self.h, front, None, None, None, None)
        if nn == 0:
            return None
        u = np.zeros(nn, np.int32)
        v = np.zeros(nn, np.int32)
        r, d = C.c_int(), C.c_int()
        L.ref_front_hss(self.h, front, u.ctypes.data, v.ctypes.data, C.byref(r), C.byref(d))
        return u, v, r.value, d.value

    def solve(self, b: np.ndarray):
        x = np.asfortranarray(np.array(b, dtype=np.float64, copy=True))
        if x.ndim == 1:
            x = x.reshape(-1, 1, order="F")
        t = lib().ref_solve(self.h, x, x.shape[1])
        self.solve_seconds = t
        return x

    def __del__(self):
        try:
            if self.h:
                lib().ref_factor_free(self.h)
                self.h = None
        except Exception:
            pass


class DenseHss:
    def __init__(self, a: np.ndarray, leaf=128, eps=1e-8, d0=128, dd=128, p=10,
                 max_rank=5000):
        L = lib()
        A = np.asfortranarray(a, dtype=np.float64)
        st = C.c_int(0)
        self.n = A.shape[0]
        self.h = L.ref_hss_dense(A, self.n, leaf, eps, d0, dd, p, max_rank, C.byref(st))
        if not self.h:
            raise RefError(st.value, -1, -1, L.ref_last_error().decode())
        r, d, tc, tu = C.c_int(), C.c_int(), C.c_double(), C.c_double()
        nn = L.ref_hss_info(self.h, None, None, C.byref(r), C.byref(d), C.byref(tc),
                            C.byref(tu))
        self.u_rank = np.zeros(nn, np.int32)
        self.v_rank = np.zeros(nn, np.int32)
        L.ref_hss_info(self.h, self.u_rank.ctypes.data, self.v_rank.ctypes.data,
                       C.byref(r), C.byref(d), C.byref(tc), C.byref(tu))
        self.rounds, self.d_final = r.value, d.value
        self.t_compress, self.t_ulv = tc.value, tu.value

    def solve(self, b):
        x = np.asfortranarray(np.array(b, dtype=np.float64, copy=True))
        if x.ndim == 1:
            x = x.reshape(-1, 1, order="F")
        self.solve_seconds = lib().ref_hss_solve(self.h, x, x.shape[1])
        return x

    def matvec(self, x):
        X = np.asfortranarray(np.array(x, dtype=np.float64))
        if X.ndim == 1:
            X = X.reshape(-1, 1, order="F")
        Y = np.zeros_like(X, order="F")
        lib().ref_hss_matvec(self.h, X, Y, X.shape[1])
        return Y

    def __del__(self):
        try:
            if self.h:
                lib().ref_hss_free(self.h)
                self.h = None
        except Exception:
            pass


def lu(a: np.ndarray):
    A = np.asfortranarray(np.array(a, dtype=np.float64, copy=True))
    m, n = A.shape
    piv = np.zeros(min(m, n), np.int32)
    col = lib().ref_lu(A, m, n, piv)
    return A, piv, col


def interpolative_decomposition(y, eps, max_rank=-1, abs_tol=0.0):
    Y = np.asfortranarray(y, dtype=np.float64)
    m, n = Y.shape
    perm = np.zeros(n, np.int32)
    rank, cert = C.c_int(), C.c_int()
    coeffs = np.zeros((min(m, n), n), np.float64, order="F")
    lib().ref_id(Y, m, n, eps, max_rank, abs_tol, perm, C.byref(rank), C.byref(cert),
                 coeffs)
    k = rank.value
    flat = coeffs.reshape(-1, order="F")[: k * (n - k)]
    return perm, k, bool(cert.value), flat.reshape((k, n - k), order="F")


def cluster_front(ns, nu, leaf):
    L = lib()
    nn = L.ref_cluster_front(ns, nu, leaf, None, None, None, None, None)
    arr = [np.zeros(nn, np.int32) for _ in range(5)]
    L.ref_cluster_front(ns, nu, leaf, *[a.ctypes.data for a in arr])
    return arr


def stats_strings(s, include_per_front=True):
    """the reference's stats_to_json / stats_csv_header / stats_csv_row
    (src/stats.cpp:37-123) for a RunStats-like object (fields of
    paper_1502_07405_b200.stats.RunStats; its rank_guard is passed as the
    options' max_rank, which resolves to itself)"""
    L = lib()
    ints = np.array([s.n, s.nnz, s.ls, s.leaf, s.d0, s.dd, s.p, s.min_hss, s.rank_guard,
                     s.threads, s.restart, s.maxit, s.nd_leaf, s.factor_flops, s.solve_flops,
                     s.factor_nnz, s.factor_nnz_bytes, s.peak_bytes, s.max_rank, s.fronts,
                     s.hss_fronts, s.hss_fallbacks, s.tree_depth, s.iterations,
                     1 if s.converged else 0], np.int64)
    reals = np.array([s.eps, s.rtol, s.atol, s.t_analysis, s.t_factor, s.t_solve, s.t_total,
                      s.relres, s.absres], np.float64)
    pf = np.array([[f["id"], f["level"], f["dim"], f["sep"], f["rank"], f["flops"]]
                   for f in s.per_front], np.int64).reshape(-1, 6)
    types = (C.c_char_p * max(1, len(s.per_front)))(*[f["type"].encode() for f in s.per_front])
    fn = L.ref_stats
    fn.restype = C.c_longlong
    fn.argtypes = [C.c_char_p, C.c_int, C.c_char_p, C.c_void_p, C.c_void_p, C.c_char_p,
                   C.c_char_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_char_p,
                   C.c_longlong]
    args = [s.source.encode(), 1 if s.strategy == "graph" else 0, s.mode.encode(),
            ints.ctypes.data, reals.ctypes.data, s.method.encode(), s.error.encode(),
            len(s.per_front), pf.ctypes.data if len(pf) else None, types,
            1 if include_per_front else 0]
    need = fn(*args, None, 0)
    buf = C.create_string_buffer(int(need))
    fn(*args, buf, need)
    parts = buf.raw[:need].split(b"\0")
    return parts[0].decode(), parts[1].decode(), parts[2].decode()
