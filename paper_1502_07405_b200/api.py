"""Python mirror of the reference's public interface for the hot path.

Same names, argument meaning and error behaviour as proj/include/hssmf
(SparseMatrix, generate_grid_problem, nested_dissection_geometric,
EliminationTree, symbolic_factorization, SolverOptions, HssOptions,
mf_factor, mf_solve, mf_solve_new, hss_compress, ulv_factor), implemented on
top of the C-ABI (include/hssmf_b200.h). Host analysis is native C++; all
numerics run in sm_100a kernels. There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _native as N

GRID_KINDS = {"p2d": 0, "p3d": 1, "c2d": 2, "c3d": 3}
FRONT_TYPES = {0: "dense", 1: "hss", 2: "hss_dense"}


# ---- exceptions (errors.hpp:10-54) -----------------------------------------
class SolverError(RuntimeError):
    pass


class IoError(SolverError):
    pass


class SingularMatrixError(SolverError):
    def __init__(self, msg, column):
        super().__init__(msg)
        self._column = column

    def column(self):
        return self._column


class HssRankExceeded(SolverError):
    pass


class StructuralSingularError(SolverError):
    """errors.hpp:32-35"""


class KrylovDivergenceError(SolverError):
    pass


class CudaError(SolverError):
    pass


def _check(rc, st: N.Status):
    if rc == 0:
        return
    msg = st.msg.decode(errors="replace")
    if rc == 1:
        raise IoError(msg)
    if rc == 2:
        raise SolverError(msg)
    if rc == 3:
        raise SingularMatrixError(msg, st.column)
    if rc == 4:
        raise CudaError(msg)
    if rc == 6:
        raise HssRankExceeded(msg)
    if rc == 8:
        raise KrylovDivergenceError(msg)
    if rc == 9:
        raise StructuralSingularError(msg)
    raise SolverError(msg)


def _call(fname, *args):
    st = N.Status()
    rc = getattr(N.lib(), fname)(*args, C.byref(st))
    _check(rc, st)


# ---- sparse matrix (sparse_matrix.hpp) --------------------------------------
class SparseMatrix:
    """square CSR with sorted, duplicate-free rows (owns a native handle)"""

    def __init__(self, handle):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle
        n, nnz = C.c_int(), C.c_longlong()
        N.lib().hssmf_csr_info(self._h, C.byref(n), C.byref(nnz))
        self.n = n.value
        self._nnz = nnz.value
        self._arrays = None

    @classmethod
    def from_csr(cls, n, ptr, ind, val):
        h = C.c_void_p()
        _call("hssmf_csr_create", int(n), np.ascontiguousarray(ptr, np.int32),
              np.ascontiguousarray(ind, np.int32), np.ascontiguousarray(val, np.float64),
              C.byref(h))
        return cls(h)

    def size(self):
        return self.n

    def nnz(self):
        return self._nnz

    def arrays(self):
        if self._arrays is None:
            ptr = np.zeros(self.n + 1, np.int32)
            ind = np.zeros(self._nnz, np.int32)
            val = np.zeros(self._nnz, np.float64)
            N.lib().hssmf_csr_get(self._h, ptr, ind, val)
            self._arrays = (ptr, ind, val)
        return self._arrays

    def permuted(self, perm):
        h = C.c_void_p()
        _call("hssmf_csr_permuted", self._h, np.ascontiguousarray(perm, np.int32), C.byref(h))
        return SparseMatrix(h)

    def matvec(self, x):
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(self.n, np.float64)
        N.lib().hssmf_csr_matvec(self._h, x, y)
        return y

    def __del__(self):
        try:
            if self._h:
                N.lib().hssmf_csr_free(self._h)
                self._h = None
        except Exception:
            pass


@dataclass
class GridGeometry:
    dims: tuple = (1, 1, 1)
    ndims: int = 0


@dataclass
class GridProblem:
    A: SparseMatrix
    geom: GridGeometry
    kind: str
    k: int
    nu: float


def generate_grid_problem(kind: str, k: int, nu: float = 1e-4) -> GridProblem:
    """grid_problems.hpp:65-117"""
    h = C.c_void_p()
    dims = np.zeros(3, np.int32)
    nd = C.c_int()
    _call("hssmf_csr_grid", GRID_KINDS[kind], int(k), float(nu), C.byref(h), dims,
          C.byref(nd))
    return GridProblem(SparseMatrix(h), GridGeometry(tuple(int(d) for d in dims), nd.value),
                       kind, k, nu)


def generate_convdiff3d(k: int, scale: float = 0.1) -> GridProblem:
    """BASELINE config 4 operator (constant beta, upwind); not a reference generator"""
    h = C.c_void_p()
    _call("hssmf_csr_convdiff3d", int(k), float(scale), C.byref(h))
    return GridProblem(SparseMatrix(h), GridGeometry((k, k, k), 3), "cd3d", k, scale)


# ---- Matrix Market I/O and equilibration (matrix_market.cpp, scaling.hpp) ----
def read_matrix_market(path) -> SparseMatrix:
    """matrix_market.cpp:10-65"""
    h = C.c_void_p()
    _call("hssmf_csr_read_mm", os.fsencode(path), C.byref(h))
    return SparseMatrix(h)


def write_matrix_market(a: SparseMatrix, path):
    """matrix_market.cpp:67-77"""
    _call("hssmf_csr_write_mm", a._h, os.fsencode(path))


@dataclass
class ScalingState:
    """scaling.hpp:15-32: As = Dr A Dc Qc"""
    dr: np.ndarray
    dc: np.ndarray
    qc: np.ndarray
    sweeps: int

    def apply_scaling(self, b):
        """b -> Dr b"""
        b = np.asarray(b, np.float64)
        return b * (self.dr if b.ndim == 1 else self.dr[:, None])

    def undo_scaling(self, xs):
        """xs -> x with x[qc[j]] = dc[qc[j]] xs[j]"""
        xs = np.asarray(xs, np.float64)
        x = np.empty_like(xs)
        x[self.qc] = (self.dc[self.qc] * xs) if xs.ndim == 1 else self.dc[self.qc][:, None] * xs
        return x


def equilibrate_and_permute(a: SparseMatrix):
    """scaling.hpp:40-139; returns (As, ScalingState)"""
    n = a.size()
    dr, dc = np.zeros(n), np.zeros(n)
    qc = np.zeros(n, np.int32)
    sw = C.c_int()
    h = C.c_void_p()
    _call("hssmf_equilibrate", a._h, C.byref(h), dr.ctypes.data_as(C.c_void_p),
          dc.ctypes.data_as(C.c_void_p), qc.ctypes.data_as(C.c_void_p), C.byref(sw))
    return SparseMatrix(h), ScalingState(dr, dc, qc, sw.value)


# ---- elimination tree (elimination_tree.hpp) --------------------------------
class EliminationTree:
    def __init__(self, handle):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle
        self.refresh()

    def refresh(self):
        n, nn, tot = C.c_int(), C.c_int(), C.c_longlong()
        N.lib().hssmf_tree_info(self._h, C.byref(n), C.byref(nn), C.byref(tot))
        self.n = n.value
        z = lambda k: np.zeros(k, np.int32)  # noqa: E731
        nn = nn.value
        self.sep_begin, self.sep_end, self.child0, self.child1 = z(nn), z(nn), z(nn), z(nn)
        self.parent, self.level, self.upd_ptr, self.upd_ind = z(nn), z(nn), z(nn + 1), \
            z(tot.value)
        N.lib().hssmf_tree_get(self._h, self.sep_begin, self.sep_end, self.child0,
                               self.child1, self.parent, self.level, self.upd_ptr,
                               self.upd_ind)

    @classmethod
    def from_arrays(cls, n, sep_begin, sep_end, child0, child1, parent, upd=None):
        a = lambda x: np.ascontiguousarray(x, np.int32)  # noqa: E731
        h = C.c_void_p()
        if upd is not None:
            up = np.zeros(len(sep_begin) + 1, np.int32)
            for i, u in enumerate(upd):
                up[i + 1] = up[i] + len(u)
            ui = a(np.concatenate([np.asarray(u, np.int32) for u in upd]) if len(upd) else [])
            upp, uip = up.ctypes.data_as(C.c_void_p), ui.ctypes.data_as(C.c_void_p)
            keep = (up, ui)
        else:
            upp = uip = None
            keep = None
        _call("hssmf_tree_create", int(n), len(sep_begin), a(sep_begin), a(sep_end),
              a(child0), a(child1), a(parent), upp, uip, C.byref(h))
        del keep
        return cls(h)

    def size(self):
        return len(self.sep_begin)

    def sep_clusters(self, i):
        """FrontNode::sep_clusters of front i as (begin, end, child0, child1,
        parent) arrays (empty when the separator was not reordered)"""
        L = N.lib()
        nn = L.hssmf_tree_sep_clusters(self._h, int(i), None, None, None, None, None)
        if nn < 0:
            raise IoError("sep_clusters: front out of range")
        arr = [np.zeros(nn, np.int32) for _ in range(5)]
        L.hssmf_tree_sep_clusters(self._h, int(i), *[x.ctypes.data_as(C.c_void_p) for x in arr])
        return arr

    def set_sep_clusters(self, i, begin, end, child0, child1):
        a = lambda x: np.ascontiguousarray(x, np.int32)  # noqa: E731
        b, e, c0, c1 = a(begin), a(end), a(child0), a(child1)
        _call("hssmf_tree_set_sep_clusters", self._h, int(i), len(b),
              *[x.ctypes.data_as(C.c_void_p) for x in (b, e, c0, c1)])

    def root_id(self):
        return self.size() - 1

    def upd(self, i):
        return self.upd_ind[self.upd_ptr[i]:self.upd_ptr[i + 1]]

    def __del__(self):
        try:
            if self._h:
                N.lib().hssmf_tree_free(self._h)
                self._h = None
        except Exception:
            pass


def nested_dissection_geometric(geom: GridGeometry, leaf: int):
    """ordering.cpp:213-222 + EliminationTree::from_separators; returns
    (tree without upd sets, perm with perm[old] = new)"""
    n = int(np.prod(geom.dims))
    perm = np.zeros(n, np.int32)
    h = C.c_void_p()
    _call("hssmf_nd_geometric", np.ascontiguousarray(geom.dims, np.int32), geom.ndims,
          int(leaf), perm, C.byref(h))
    return EliminationTree(h), perm


def nested_dissection_graph(a: SparseMatrix, leaf: int):
    """ordering.cpp:224-236 on a.symmetric_graph() + from_separators; returns
    (tree without upd sets, perm with perm[old] = new)"""
    perm = np.zeros(a.size(), np.int32)
    h = C.c_void_p()
    _call("hssmf_nd_graph", a._h, int(leaf), perm, C.byref(h))
    return EliminationTree(h), perm


def reorder_tree_separators(t: EliminationTree, a: SparseMatrix, selected, b: int):
    """separator_reorder.cpp:119-135: selected fronts get separator clusters
    of at most b vertices; returns perm[old] = new (identity elsewhere). The
    caller permutes a and re-runs symbolic_factorization."""
    sel = np.ascontiguousarray(np.asarray(selected, bool).astype(np.int8))
    if len(sel) != t.size():
        raise IoError("reorder: one selection flag per front")
    perm = np.zeros(t.n, np.int32)
    _call("hssmf_reorder_separators", t._h, a._h, sel.ctypes.data_as(C.c_void_p), int(b), perm)
    return perm


def ordered_graph(a: SparseMatrix, nd_leaf: int, reorder_b: int = 0, selected=None):
    """graph-ordering pipeline: ND + symbolic, then (reorder_b > 0) separator
    reordering of the selected fronts (default: every front with a
    separator) and the symbolic analysis of the relabeled matrix"""
    t, perm = nested_dissection_graph(a, nd_leaf)
    ap = a.permuted(perm)
    symbolic_factorization(ap, t)
    if reorder_b > 0:
        if selected is None:
            selected = (t.sep_end - t.sep_begin) > 0
        r = reorder_tree_separators(t, ap, selected, reorder_b)
        ap = ap.permuted(r)
        perm = r[perm]
        symbolic_factorization(ap, t)
    return OrderedProblem(ap, t, perm, None)


def symbolic_factorization(a: SparseMatrix, t: EliminationTree):
    """elimination_tree.hpp:67-73"""
    _call("hssmf_symbolic", a._h, t._h)
    t.refresh()


def front_cluster_tree(ns, nu, leaf):
    L = N.lib()
    nn = L.hssmf_front_cluster_tree(ns, nu, leaf, None, None, None, None, None)
    arr = [np.zeros(nn, np.int32) for _ in range(5)]
    L.hssmf_front_cluster_tree(ns, nu, leaf, *[x.ctypes.data_as(C.c_void_p) for x in arr])
    return arr


@dataclass
class OrderedProblem:
    a: SparseMatrix
    t: EliminationTree
    perm: np.ndarray
    geom: GridGeometry


def ordered_problem(g: GridProblem, nd_leaf: int) -> OrderedProblem:
    """the canonical pipeline of tests/support/problems.hpp:20-30"""
    t, perm = nested_dissection_geometric(g.geom, nd_leaf)
    a = g.A.permuted(perm)
    symbolic_factorization(a, t)
    return OrderedProblem(a, t, perm, g.geom)


def ordered_grid(kind: str, k: int, nd_leaf: int, nu: float = 1e-4) -> OrderedProblem:  # noqa: E302
    return ordered_problem(generate_grid_problem(kind, k, nu), nd_leaf)


# ---- options (solver_options.hpp:28-59, hss_compress.hpp:26-32) ------------
@dataclass
class SolverOptions:
    nd_leaf: int = 32
    ls: int = 0
    eps: float = 1e-8
    leaf: int = 128
    d0: int = 128
    dd: int = 128
    p: int = 10
    min_hss: int = 512
    max_rank: int = 0
    mode: str = "auto"  # auto | mf | mf-hss

    def validate(self):
        if self.eps < 0 or self.eps >= 1:
            raise IoError("eps must be in [0,1)")
        if self.ls < 0:
            raise IoError("ls must be >= 0")
        if self.leaf < 16:
            raise IoError("leaf size b must be >= 16")
        if self.d0 < 1 or self.dd < 1 or self.p < 0 or self.p >= self.d0:
            raise IoError("need d0 >= 1, dd >= 1, 0 <= p < d0")
        if self.nd_leaf < 1:
            raise IoError("dissection leaf must be >= 1")

    def native(self) -> N.Options:
        mode = {"auto": 0, "mf": 1, "mf-hss": 2}[self.mode]
        return N.Options(self.ls, self.eps, self.leaf, self.d0, self.dd, self.p, self.min_hss,
                         self.max_rank, mode)


@dataclass
class HssOptions:
    eps: float = 1e-8
    d0: int = 128
    dd: int = 128
    p: int = 10
    max_rank: int = 5000


@dataclass
class FrontStat:
    id: int
    level: int
    dim: int
    sep: int
    rank: int
    flops: int
    type: str


# ---- factorization (multifrontal.hpp:454-631) --------------------------------
class MfFactors:
    def __init__(self, handle, n):
        self._h = handle
        self.n = n
        self.refresh()
        self.factored = True

    def refresh(self):
        """re-read the summary and per-front stats (after factor phases)"""
        L = N.lib()
        nn, hf, fb, mr, nz = C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_longlong()
        L.hssmf_factor_summary(self._h, C.byref(nn), C.byref(hf), C.byref(fb), C.byref(mr),
                               C.byref(nz))
        self.hss_fronts, self.fallbacks, self.max_front_rank = hf.value, fb.value, mr.value
        self._factor_nnz = nz.value
        nn = nn.value
        z = lambda: np.zeros(nn, np.int32)  # noqa: E731
        self.level, self.dim, self.sep, self.rank, self.type = z(), z(), z(), z(), z()
        self.flops = np.zeros(nn, np.int64)
        L.hssmf_front_stats(self._h, self.level, self.dim, self.sep, self.rank, self.flops,
                            self.type)

    @property
    def front_stats(self):
        return [FrontStat(i, int(self.level[i]), int(self.dim[i]), int(self.sep[i]),
                          int(self.rank[i]), int(self.flops[i]), FRONT_TYPES[int(self.type[i])])
                for i in range(len(self.level))]

    def factor_nnz(self):
        return self._factor_nnz

    def front_hss(self, front):
        L = N.lib()
        nn = L.hssmf_front_hss(self._h, front, None, None, None, None)
        if nn == 0:
            return None
        u = np.zeros(nn, np.int32)
        v = np.zeros(nn, np.int32)
        r, d = C.c_int(), C.c_int()
        L.hssmf_front_hss(self._h, front, u.ctypes.data_as(C.c_void_p),
                          v.ctypes.data_as(C.c_void_p), C.byref(r), C.byref(d))
        return u, v, r.value, d.value

    def timing(self):
        f, s = C.c_double(), C.c_double()
        N.lib().hssmf_timing(self._h, C.byref(f), C.byref(s))
        return f.value, s.value

    def set_profile(self, on=True):
        N.lib().hssmf_set_profile(self._h, 1 if on else 0)

    def kernel_stats(self):
        k = 32
        names = C.create_string_buffer(32 * k)
        la = np.zeros(k, np.int32)
        ms, fl, by = np.zeros(k), np.zeros(k), np.zeros(k)
        n = N.lib().hssmf_kernel_stats(self._h, k, names, la, ms, fl, by)
        out = []
        for i in range(n):
            nm = names.raw[32 * i:32 * (i + 1)].split(b"\0")[0].decode()
            out.append(dict(name=nm, launches=int(la[i]), ms=float(ms[i]), flops=float(fl[i]),
                            bytes=float(by[i])))
        return out

    def reset_kernel_stats(self):
        N.lib().hssmf_reset_kernel_stats(self._h)

    def device_bytes(self):
        return N.lib().hssmf_device_bytes(self._h)

    def refactor(self, val=None, device_ptr=None):
        if device_ptr is not None:
            _call("hssmf_refactor", self._h, C.c_void_p(device_ptr), 1)
        elif val is not None:
            v = np.ascontiguousarray(val, np.float64)
            _call("hssmf_refactor", self._h, v.ctypes.data_as(C.c_void_p), 0)
        else:
            _call("hssmf_refactor", self._h, None, 0)

    def solve_device(self, ptr, ldb, nrhs):
        _call("hssmf_solve", self._h, C.c_void_p(ptr), int(ldb), int(nrhs), 1)

    def __del__(self):
        try:
            if self._h:
                N.lib().hssmf_factors_free(self._h)
                self._h = None
        except Exception:
            pass


def mf_factor(a: SparseMatrix, t: EliminationTree, opts: SolverOptions, device: int = 0):
    """multifrontal.hpp:473-503: raises IoError on size mismatch and
    SingularMatrixError('front <i>...', column) on an exact zero pivot"""
    if a.size() != t.n:
        raise IoError("mf factor: matrix and tree sizes differ")
    h = C.c_void_p()
    o = opts.native()
    _call("hssmf_factor", int(device), a._h, t._h, C.byref(o), C.byref(h))
    return MfFactors(h, a.size())


def mf_solve(m: MfFactors, b: np.ndarray):
    """multifrontal.hpp:612-622: solves in place (b is n x nrhs, column-major)"""
    if m is None or not getattr(m, "factored", False) or not m._h:
        raise SolverError("mf solve: not factored")
    if b.ndim == 1:
        b2 = b.reshape(-1, 1)
    else:
        b2 = b
    if b2.shape[0] != m.n:
        raise IoError("mf solve: rhs rows mismatch")
    if not (b2.flags.f_contiguous and b2.dtype == np.float64):
        raise IoError("mf solve: b must be a Fortran-ordered float64 array")
    _call("hssmf_solve", m._h, b2.ctypes.data_as(C.c_void_p), m.n, b2.shape[1], 0)
    return b


def mf_solve_new(m: MfFactors, b: np.ndarray) -> np.ndarray:
    x = np.array(b, dtype=np.float64, order="F", copy=True)
    mf_solve(m, x)
    return x


# ---- preconditioned iterative solves (krylov.hpp:18-232) ---------------------
@dataclass
class SolveReport:
    """krylov.hpp:22-29: residuals are the left-preconditioned ones"""
    iterations: int = 0
    rel_resid: float = 0.0
    abs_resid: float = 0.0
    converged: bool = False
    stagnated: bool = False
    history: list = field(default_factory=list)


class _KrylovReport(C.Structure):
    _fields_ = [("iterations", C.c_int), ("rel_resid", C.c_double), ("abs_resid", C.c_double),
                ("converged", C.c_int), ("stagnated", C.c_int), ("history_len", C.c_int)]


def _krylov(fn, a, m, b, extra, maxit):
    bb = np.ascontiguousarray(b, np.float64).reshape(-1)
    if bb.shape[0] != a.size():
        raise IoError("krylov: rhs size mismatch")
    x = np.zeros_like(bb)
    rep = _KrylovReport()
    hist = np.zeros(maxit + 2, np.float64)
    _call(fn, a._h, m._h if m is not None else None, bb.ctypes.data_as(C.c_void_p),
          x.ctypes.data_as(C.c_void_p), *extra, C.byref(rep), hist.ctypes.data_as(C.c_void_p),
          len(hist))
    r = SolveReport(rep.iterations, rep.rel_resid, rep.abs_resid, bool(rep.converged),
                    bool(rep.stagnated), hist[:rep.history_len].tolist())
    return x, r


def gmres(a: SparseMatrix, m, b, restart=30, rtol=1e-6, atol=1e-10, maxit=500):
    """krylov.hpp:93-184 with A = a (CSR SpMV on the device) and M^-1 =
    mf_solve(m) (m None: identity); returns (x, SolveReport)"""
    if restart < 1:
        raise IoError("gmres: restart must be >= 1")
    return _krylov("hssmf_gmres", a, m, b, (int(restart), float(rtol), float(atol), int(maxit)),
                   maxit)


def iterative_refinement(a: SparseMatrix, m, b, rtol=1e-6, atol=1e-10, maxit=500):
    """krylov.hpp:189-229"""
    return _krylov("hssmf_refine", a, m, b, (float(rtol), float(atol), int(maxit)), maxit)


# ---- standalone dense HSS (hss_compress.hpp:373-383, hss_ulv.hpp) ----------
class HssFactors:
    """hss_compress(A, ClusterTree::balanced(n, leaf), opts) + ulv_factor"""

    def __init__(self, a: np.ndarray, leaf: int, opts: HssOptions, device: int = 0,
                 device_ptr=None, n=None):
        h = C.c_void_p()
        if device_ptr is not None:
            self.n = int(n)
            _call("hssmf_hss_dense", int(device), C.c_void_p(device_ptr), self.n, self.n,
                  int(leaf), opts.eps, opts.d0, opts.dd, opts.p, opts.max_rank, 1, C.byref(h))
        else:
            A = np.asfortranarray(a, dtype=np.float64)
            if A.shape[0] != A.shape[1]:
                raise IoError("hss compress: matrix and cluster tree sizes disagree")
            self.n = A.shape[0]
            _call("hssmf_hss_dense", int(device), A.ctypes.data_as(C.c_void_p), self.n,
                  self.n, int(leaf), opts.eps, opts.d0, opts.dd, opts.p, opts.max_rank, 0,
                  C.byref(h))
        self._h = h
        L = N.lib()
        r, d, tc, tu = C.c_int(), C.c_int(), C.c_double(), C.c_double()
        nn = L.hssmf_hss_info(self._h, None, None, C.byref(r), C.byref(d), C.byref(tc),
                              C.byref(tu))
        self.u_rank = np.zeros(nn, np.int32)
        self.v_rank = np.zeros(nn, np.int32)
        L.hssmf_hss_info(self._h, self.u_rank.ctypes.data_as(C.c_void_p),
                         self.v_rank.ctypes.data_as(C.c_void_p), C.byref(r), C.byref(d),
                         C.byref(tc), C.byref(tu))
        self.rounds, self.d_final = r.value, d.value
        self.compress_ms, self.ulv_ms = tc.value, tu.value

    def hss_rank(self):
        return int(max(self.u_rank[:-1].max(initial=0), self.v_rank[:-1].max(initial=0)))

    def solve(self, b):
        x = np.array(b, dtype=np.float64, order="F", copy=True)
        x2 = x.reshape(-1, 1) if x.ndim == 1 else x
        if x2.shape[0] != self.n:
            raise IoError("ulv solve: rhs rows mismatch")
        _call("hssmf_hss_solve", self._h, x2.ctypes.data_as(C.c_void_p), self.n, x2.shape[1],
              0)
        return x

    def solve_device(self, ptr, ldb, nrhs):
        _call("hssmf_hss_solve", self._h, C.c_void_p(ptr), int(ldb), int(nrhs), 1)

    def matvec(self, op, x, root=-1):
        """HssMatrix::matvec_new (hss_matrix.hpp:234-249): op(A_hss) x on the
        subtree of cluster node `root` (-1: the whole matrix); op 'N', 'T' or
        'C'. Raises IoError when x's rows do not match the node."""
        X = np.array(x, dtype=np.float64, order="F", copy=True)
        X2 = X.reshape(-1, 1) if X.ndim == 1 else X
        Y = np.zeros_like(X2, order="F")
        _call("hssmf_hss_matvec", self._h, op.encode()[:1], int(root),
              X2.ctypes.data_as(C.c_void_p), max(1, X2.shape[0]), X2.shape[0], X2.shape[1],
              Y.ctypes.data_as(C.c_void_p), max(1, X2.shape[0]), 0)
        return Y.reshape(X.shape)

    def extract(self, rows, cols):
        """HssMatrix::extract (hss_matrix.hpp:261-280): A_hss(rows, cols) for
        index lists in any order; returns (block, leaves visited)"""
        ri = np.ascontiguousarray(rows, np.int32)
        ci = np.ascontiguousarray(cols, np.int32)
        out = np.zeros((len(ri), len(ci)), order="F")
        v = C.c_longlong()
        _call("hssmf_hss_extract", self._h, ri.ctypes.data_as(C.c_void_p), len(ri),
              ci.ctypes.data_as(C.c_void_p), len(ci), out.ctypes.data_as(C.c_void_p), 0,
              C.byref(v))
        self.leaf_visits = v.value
        return out

    def __del__(self):
        try:
            if self._h:
                N.lib().hssmf_hss_free(self._h)
                self._h = None
        except Exception:
            pass


def hss_compress(a: np.ndarray, leaf: int, opts: HssOptions, device: int = 0) -> HssFactors:
    return HssFactors(a, leaf, opts, device)


# ---- kernel-level parity hooks -------------------------------------------------
def dev_random_rows(grow, c0, c1, device=0):
    g = np.ascontiguousarray(grow, np.int64)
    out = np.zeros((len(g), c1 - c0), np.float64, order="F")
    _call("hssmf_dev_random_rows", device, len(g), g, c0, c1, out.ctypes.data_as(C.c_void_p))
    return out


def dev_gemm(ta, tb, alpha, a, b, beta, c, device=0):
    A = np.asfortranarray(a, np.float64)
    B = np.asfortranarray(b, np.float64)
    Cm = np.array(c, np.float64, order="F", copy=True)
    m, n = Cm.shape
    k = A.shape[1] if ta == "N" else A.shape[0]
    _call("hssmf_dev_gemm", device, ta.encode(), tb.encode(), m, n, k, alpha,
          A.ctypes.data_as(C.c_void_p), A.shape[0], B.ctypes.data_as(C.c_void_p), B.shape[0],
          beta, Cm.ctypes.data_as(C.c_void_p), m)
    return Cm


def dev_interpolative_decomposition(y, eps, max_rank=-1, abs_tol=0.0, device=0):
    Y = np.asfortranarray(y, np.float64)
    m, n = Y.shape
    perm = np.zeros(n, np.int32)
    rank, cert = C.c_int(), C.c_int()
    X = np.zeros(max(1, min(m, n) * n), np.float64)
    _call("hssmf_dev_id", device, Y.ctypes.data_as(C.c_void_p), m, n, eps, max_rank, abs_tol,
          perm, C.byref(rank), C.byref(cert), X.ctypes.data_as(C.c_void_p))
    k = rank.value
    return perm, k, bool(cert.value), X[: k * (n - k)].reshape((k, n - k), order="F")


def dev_gram_id(y, eps, max_rank=-1, abs_tol=0.0, device=0):
    """Gram-route ID of y (d x n): (perm, rank, certified, R = L^T in position order)."""
    Y = np.asfortranarray(y, np.float64)
    m, n = Y.shape
    perm = np.zeros(n, np.int32)
    rank, cert = C.c_int(), C.c_int()
    R = np.zeros(max(1, min(m, n) * n), np.float64)
    _call("hssmf_dev_gram_id", device, Y.ctypes.data_as(C.c_void_p), m, n, eps, max_rank, abs_tol,
          perm, C.byref(rank), C.byref(cert), R.ctypes.data_as(C.c_void_p))
    k = rank.value
    return perm, k, bool(cert.value), R[: k * n].reshape((k, n), order="F")


PROBE_KINDS = ("gemm_dmma", "gram_panel", "gram_syrk")


def probe_enable(on=True):
    """Per-kernel device-time probes (measurement only, see hssmf_probe_enable)."""
    _call("hssmf_probe_enable", 1 if on else 0)


def probe_read():
    out = (N.ProbeStat * len(PROBE_KINDS))()
    _call("hssmf_probe_read", out)
    return {k: {"launches": int(o.launches), "ms": o.ms, "flops": o.flops, "bytes": o.bytes}
            for k, o in zip(PROBE_KINDS, out)}


def dev_lu(a, device=0):
    A = np.array(a, np.float64, order="F", copy=True)
    m, n = A.shape
    piv = np.zeros(n, np.int32)
    _call("hssmf_dev_lu", device, A.ctypes.data_as(C.c_void_p), m, n, piv)
    return A, piv
