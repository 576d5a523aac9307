"""Subtree-to-GPU partition of the elimination tree.

With geometric nested dissection the 2^L subtrees rooted at tree level
L = log2(P) are independent: each is a contiguous range of postorder front
ids and of separator indices. Rank r owns the r-th such subtree (left to
right); a front above level L is owned by the owner of its child0 subtree
(subtree-to-subcube). The only exchanges are at ownership changes along tree
edges:

* factorization: a child's update operator (dense cb or the densified HSS
  update, nu_c x nu_c doubles) goes once to the parent's owner;
* forward solve: the child's bupd (nu_c x nrhs) goes up the same edge;
* backward solve: x(upd) of the child (nu_c x nrhs) comes back down.

These are point-to-point messages (NCCL send/recv over NVLink in production,
gloo on CPU in the tests). No all-reduce or all-gather is needed.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Partition:
    nranks: int
    level: int
    owner: np.ndarray                      # owner rank per front
    roots: list                            # subtree root front per rank
    edges: list = field(default_factory=list)  # (child, parent, src, dst, nu_child)

    def fronts_of(self, rank: int) -> np.ndarray:
        return np.nonzero(self.owner == rank)[0]

    def factor_bytes(self) -> int:
        return int(sum(8 * nu * nu for (_, _, _, _, nu) in self.edges))


def subtree_partition(t, nranks: int) -> Partition:
    """t: an EliminationTree-like object with child0/child1/level arrays and
    upd_ptr (postorder, root last)."""
    if nranks < 1 or nranks & (nranks - 1):
        raise ValueError("the subtree partition needs a power-of-two rank count")
    L = int(np.log2(nranks))
    nn = len(t.child0)
    level = np.asarray(t.level)
    child0 = np.asarray(t.child0)
    child1 = np.asarray(t.child1)
    # subtree roots at level L, left to right = increasing postorder id
    roots = [int(i) for i in np.nonzero(level == L)[0]]
    if len(roots) != nranks:
        raise ValueError(f"tree has {len(roots)} fronts at level {L}, need {nranks}")
    owner = np.full(nn, -1, np.int64)
    lo = np.arange(nn)
    for i in range(nn):  # postorder: children first
        for c in (child0[i], child1[i]):
            if c >= 0:
                lo[i] = min(lo[i], lo[c])
    for r, s in enumerate(roots):
        owner[lo[s]:s + 1] = r
    for i in range(nn):  # fronts above level L, bottom-up in postorder
        if owner[i] < 0:
            c = child0[i] if child0[i] >= 0 else child1[i]
            owner[i] = owner[c] if c >= 0 else 0
    nu = np.diff(np.asarray(t.upd_ptr))
    edges = []
    for i in range(nn):
        for c in (child0[i], child1[i]):
            if c >= 0 and owner[c] != owner[i]:
                edges.append((int(c), int(i), int(owner[c]), int(owner[i]), int(nu[c])))
    return Partition(nranks, L, owner, roots, edges)


def exchange_updates(part: Partition, rank: int, payload_of, send, recv):
    """Run the factorization-time exchange of one rank: for every cross-rank
    edge whose child this rank owns, send the child's update; for every edge
    whose parent it owns, receive it. payload_of(child) -> array; send(arr,
    dst); recv(shape, src) -> array. Returns {child: received array}."""
    got = {}
    # a fixed global order (by parent level, deepest first, then child id)
    # keeps every pair of ranks matched without deadlock
    order = sorted(part.edges, key=lambda e: (-e[1], e[0]))
    for (c, p, src, dst, nu) in order:
        if src == rank:
            send(payload_of(c), dst)
        elif dst == rank:
            got[c] = recv((nu, nu), src)
    return got


# ---- phased factorization / solve over a subtree partition ------------------
#
# Every rank runs the same sequence of phases; a phase touches only the fronts
# the rank owns. Exchanges happen between phases, edge by edge in one global
# order (deepest parent level first, then by child id), so every send meets
# its receive without a global barrier:
#
#   factor:  levels >= L (own subtree)  | for l = L-1..0: updates of the
#            children of level-l fronts cross over, then level l
#   solve:   forward levels >= L | for l = L-1..0: bupd of level-(l+1)
#            children cross over, forward level l | for l = 0..L-1: backward
#            level l, then x(upd) of the level-(l+1) children crosses back |
#            backward levels >= L
#
# `engine` objects expose factor_levels / export_update / import_update /
# export_bupd / import_bupd / solve_levels (PartFactors on a GPU; a recording
# fake in the CPU tests). `transport` moves arrays between ranks: send(obj,
# dst), recv(shape, src) -> obj (torch.distributed over NCCL on GPUs, a
# mailbox for several ranks in one process, gloo on CPU).


def _edges_into(part: Partition, t_level, l):
    return sorted([e for e in part.edges if t_level[e[1]] == l], key=lambda e: e[0])


def phased_factor(part: Partition, t_level, nlev, engines: dict, transport):
    """engines: {rank: engine} for the ranks living in this process"""
    L = part.level
    for e in engines.values():
        e.factor_levels(L, nlev - 1)
    for l in range(L - 1, -1, -1):
        for (c, p, src, dst, nu) in _edges_into(part, t_level, l):
            if src in engines:
                transport.send(engines[src].export_update(c), dst, src)
            if dst in engines:
                engines[dst].import_update(c, transport.recv((nu, nu), src, dst))
        for e in engines.values():
            e.factor_levels(l, l)


def phased_solve(part: Partition, t_level, nlev, upd_of, engines: dict, xs: dict, nrhs,
                 transport):
    """xs: {rank: device x (n x nrhs)} solved in place on every rank; each
    rank ends up with x correct on the separators of the fronts it owns"""
    L = part.level
    for r, e in engines.items():
        e.solve_levels(xs[r], L, nlev - 1, True)
    for l in range(L - 1, -1, -1):
        for (c, p, src, dst, nu) in _edges_into(part, t_level, l):
            if src in engines:
                transport.send(engines[src].export_bupd(c, nrhs), dst, src)
            if dst in engines:
                engines[dst].import_bupd(c, transport.recv((nu, nrhs), src, dst), nrhs)
        for r, e in engines.items():
            e.solve_levels(xs[r], l, l, True)
    for l in range(0, L):
        for r, e in engines.items():
            e.solve_levels(xs[r], l, l, False)
        # x at the update indices of the level-(l+1) children goes back down
        # (owner of the parent -> owner of the child)
        for (c, p, src, dst, nu) in _edges_into(part, t_level, l):
            if dst in engines:
                transport.send(engines[dst].gather_x(xs[dst], upd_of(c)), src, dst)
            if src in engines:
                engines[src].scatter_x(xs[src], upd_of(c), transport.recv((nu, nrhs), dst, src))
    for r, e in engines.items():
        e.solve_levels(xs[r], L, nlev - 1, False)


def separator_mask(t, owner, rank):
    """rows of x computed by `rank` (the separators of its fronts)"""
    m = np.zeros(int(t.sep_end.max(initial=0)), bool)
    for i in np.nonzero(np.asarray(owner) == rank)[0]:
        m[t.sep_begin[i]:t.sep_end[i]] = True
    return m


class Mailbox:
    """transport for several ranks in one process (one GPU): messages are
    copied into a queue keyed by (src, dst)"""

    def __init__(self):
        self.q = {}

    def send(self, obj, dst, src):
        self.q.setdefault((src, dst), []).append(obj.clone() if hasattr(obj, "clone") else obj.copy())

    def recv(self, shape, src, dst):
        return self.q[(src, dst)].pop(0)


class TorchTransport:
    """torch.distributed point-to-point (NCCL over NVLink on GPUs, gloo on
    CPU); tensors are device (NCCL) or host (gloo) float64"""

    def __init__(self, device=None):
        import torch
        self.torch = torch
        self.device = device

    def send(self, obj, dst, src):
        self.torch.distributed.send(obj.contiguous(), dst)

    def recv(self, shape, src, dst):
        buf = self.torch.empty(shape[::-1] if len(shape) == 2 else shape, dtype=self.torch.float64,
                               device=self.device)
        self.torch.distributed.recv(buf, src)
        # NCCL's recv only orders torch's current stream after the transfer;
        # the engine reads `buf` on its own stream, so the host waits here
        # until the data has landed (the import copies are host-ordered after)
        if buf.is_cuda:
            self.torch.cuda.current_stream(buf.device).synchronize()
        return buf


class PartFactors:
    """One rank's share of a subtree-partitioned factorization on a GPU
    (C-ABI hssmf_analyze_owned & co). Arrays crossing ranks are torch
    tensors on this rank's device; a (nu x k) column-major block is a torch
    (k, nu) row-major tensor."""

    def __init__(self, a, t, opts, part: Partition, rank: int, device: int = 0):
        import ctypes as C
        import torch
        from . import _native as N
        from .api import MfFactors, _call
        self.C, self.N, self.torch, self._call = C, N, torch, _call
        self.part, self.rank, self.device = part, rank, device
        self.dev = torch.device("cuda", device)
        owned = np.ascontiguousarray(np.asarray(part.owner) == rank, np.int8)
        h = C.c_void_p()
        o = opts.native()
        _call("hssmf_analyze_owned", int(device), a._h, t._h, C.byref(o),
              owned.ctypes.data_as(C.c_void_p), C.byref(h))
        self.m = MfFactors(h, a.size())
        self.m.factored = False
        self.nlev = N.lib().hssmf_nlevels(h)
        self.nu = np.diff(np.asarray(t.upd_ptr))
        self.n = a.size()

    @property
    def h(self):
        return self.m._h

    def factor_levels(self, lo, hi):
        self._call("hssmf_factor_levels", self.h, int(lo), int(hi))
        if lo == 0:
            self.m.refresh()
            self.m.factored = True

    def export_update(self, f):
        nu = int(self.nu[f])
        buf = self.torch.empty((nu, nu), dtype=self.torch.float64, device=self.dev)
        self._call("hssmf_update_export", self.h, int(f), self.C.c_void_p(buf.data_ptr()), 1)
        return buf

    def import_update(self, f, buf):
        self._call("hssmf_update_import", self.h, int(f), self.C.c_void_p(buf.data_ptr()), 1)

    def export_bupd(self, f, nrhs):
        nu = int(self.nu[f])
        buf = self.torch.empty((nrhs, nu), dtype=self.torch.float64, device=self.dev)
        self._call("hssmf_bupd_export", self.h, int(f), self.C.c_void_p(buf.data_ptr()), int(nrhs))
        return buf

    def import_bupd(self, f, buf, nrhs):
        self._call("hssmf_bupd_import", self.h, int(f), self.C.c_void_p(buf.data_ptr()), int(nrhs))

    def solve_levels(self, x, lo, hi, forward):
        nrhs = x.shape[0]
        self._call("hssmf_solve_levels", self.h, self.C.c_void_p(x.data_ptr()), self.n, int(nrhs),
                   int(lo), int(hi), 1 if forward else 0)

    def gather_x(self, x, rows):
        # solve_levels synchronised the engine stream before returning
        return x[:, rows].contiguous()

    def scatter_x(self, x, rows, vals):
        x[:, rows] = vals
        # the next solve_levels reads x on the engine's stream, not torch's
        self.torch.cuda.current_stream(self.dev).synchronize()


class ProtocolEngine:
    """Stand-in for PartFactors (CPU tests and `bench.py --dry-run`): 'factoring' front f gives val[f] = f + sum of
    the children's vals (a child's val must be local or imported), the forward
    sweep fwd[f] = val[f] + sum of the children's fwd, the backward sweep
    x[f] = fwd[f] + x[parent]. Checks that every phase finds its inputs."""

    def __init__(self, t, part, rank):
        import torch
        self.torch = torch
        self.t, self.part, self.rank = t, part, rank
        self.own = np.asarray(part.owner) == rank
        self.val, self.fwd = {}, {}

    def _kids(self, f):
        return [c for c in (self.t.child0[f], self.t.child1[f]) if c >= 0]

    def _at(self, lo, hi):
        return [f for f in range(len(self.own)) if self.own[f] and lo <= self.t.level[f] <= hi]

    def factor_levels(self, lo, hi):
        for f in sorted(self._at(lo, hi), key=lambda f: -self.t.level[f]):
            self.val[f] = float(f) + sum(self.val[c] for c in self._kids(f))

    def _nu(self, f):
        return int(self.t.upd_ptr[f + 1] - self.t.upd_ptr[f])

    def export_update(self, f):  # nu x nu, like the real update block
        nu = self._nu(f)
        return self.torch.full((nu, nu), self.val[f], dtype=self.torch.float64)

    def import_update(self, f, buf):
        self.val[f] = float(buf[0, 0])

    def export_bupd(self, f, nrhs):
        return self.torch.full((nrhs, self._nu(f)), self.fwd[f], dtype=self.torch.float64)

    def import_bupd(self, f, buf, nrhs):
        self.fwd[f] = float(buf[0, 0])

    def solve_levels(self, x, lo, hi, forward):
        fs = self._at(lo, hi)
        if forward:
            for f in sorted(fs, key=lambda f: -self.t.level[f]):
                self.fwd[f] = self.val[f] + sum(self.fwd[c] for c in self._kids(f))
        else:
            for f in sorted(fs, key=lambda f: self.t.level[f]):
                p = self.t.parent[f]
                x[0, f] = self.fwd[f] + (float(x[0, p]) if p >= 0 else 0.0)

    def gather_x(self, x, rows):
        return x[:, rows].clone()

    def scatter_x(self, x, rows, vals):
        x[:, rows] = vals


def protocol_expected(t):
    nn = len(t.child0)
    val, fwd, x = np.zeros(nn), np.zeros(nn), np.zeros(nn)
    for f in range(nn):  # postorder
        kids = [c for c in (t.child0[f], t.child1[f]) if c >= 0]
        val[f] = f + sum(val[c] for c in kids)
        fwd[f] = val[f] + sum(fwd[c] for c in kids)
    for f in range(nn - 1, -1, -1):
        p = t.parent[f]
        x[f] = fwd[f] + (x[p] if p >= 0 else 0.0)
    return val, x


def protocol_check(t, part, rank, transport):
    """Run the phased factor + solve protocol of `rank` with ProtocolEngine
    over `transport`; True when every owned front saw the inputs the
    sequential schedule would give it"""
    import torch
    eng = ProtocolEngine(t, part, rank)
    nlev = int(np.asarray(t.level).max()) + 1
    phased_factor(part, t.level, nlev, {rank: eng}, transport)
    x = torch.zeros((1, len(t.child0)), dtype=torch.float64)

    def upd_of(c):  # nu_c copies of the parent's slot in this stand-in x
        return torch.full((int(t.upd_ptr[c + 1] - t.upd_ptr[c]),), int(t.parent[c]),
                          dtype=torch.long)
    phased_solve(part, t.level, nlev, upd_of, {rank: eng}, {rank: x}, 1, transport)
    val, xe = protocol_expected(t)
    own = np.nonzero(eng.own)[0]
    return (all(abs(eng.val[f] - val[f]) < 1e-9 for f in own)
            and all(abs(float(x[0, f]) - xe[f]) < 1e-9 for f in own))


class DistributedMf:
    """Subtree-partitioned factorization + solve over nranks GPUs (SURVEY
    §8e). rank=None keeps every rank in this process on `device` (several
    engines on one GPU, messages through a Mailbox: the single-GPU check of
    the partitioned path); otherwise this process is `rank` and `transport`
    (TorchTransport over NCCL) reaches the others."""

    def __init__(self, a, t, opts, nranks, rank=None, transport=None, device=0):
        import torch
        self.torch = torch
        self.t = t
        self.part = subtree_partition(t, nranks)
        self.ranks = list(range(nranks)) if rank is None else [rank]
        self.transport = transport or Mailbox()
        self.dev = torch.device("cuda", device)
        self.engines = {r: PartFactors(a, t, opts, self.part, r, device) for r in self.ranks}
        self.nlev = next(iter(self.engines.values())).nlev
        self.masks = {r: torch.from_numpy(separator_mask(t, self.part.owner, r)).to(self.dev)
                      for r in self.ranks}
        self._upd = {}

    def upd_of(self, c):
        if c not in self._upd:
            self._upd[c] = self.torch.from_numpy(self.t.upd(c).astype(np.int64)).to(self.dev)
        return self._upd[c]

    def factor(self):
        phased_factor(self.part, self.t.level, self.nlev, self.engines, self.transport)

    def solve_device(self, xs: dict):
        """xs: {rank: (nrhs, n) float64 device tensor}, solved in place; each
        rank's x is correct on its own separators"""
        nrhs = next(iter(xs.values())).shape[0]
        # xs may have been written on torch's stream; the engines use their own
        self.torch.cuda.current_stream(self.dev).synchronize()
        phased_solve(self.part, self.t.level, self.nlev, self.upd_of, self.engines, xs, nrhs,
                     self.transport)

    def combine(self, xs: dict):
        """the solution rows of this process's ranks (other rows 0)"""
        out = None
        for r in self.ranks:
            v = self.torch.where(self.masks[r], xs[r], self.torch.zeros_like(xs[r]))
            out = v if out is None else out + v
        return out

    def solve(self, b):
        bb = np.asarray(b, np.float64)
        b2 = bb.reshape(-1, 1) if bb.ndim == 1 else bb
        xs = {r: self.torch.from_numpy(np.ascontiguousarray(b2.T)).to(self.dev) for r in self.ranks}
        self.solve_device(xs)
        x = self.combine(xs).cpu().numpy().T
        return x.reshape(bb.shape)


# ---- the native (C++) driver of the same protocol (csrc/mgpu.cu) ----------
def native_partition(t, nranks):
    """owner per front and the cross-rank edge count from the C++ partition
    (hssmf_mgpu_partition); equal to subtree_partition's"""
    import ctypes as C
    from . import _native as N
    from .api import _call
    owner = np.zeros(len(t.child0), np.int32)
    ne = C.c_int()
    _call("hssmf_mgpu_partition", t._h, int(nranks), owner.ctypes.data_as(C.c_void_p),
          C.byref(ne))
    del N
    return owner, ne.value


def native_local_solve(a, t, opts, nranks, b, device=0):
    """all nranks ranks of the C++ driver in this process on one GPU
    (hssmf_mgpu_local: in-process mailbox): partitioned factor + solve of b
    (n or n x nrhs), returns x"""
    import ctypes as C

    import torch

    from .api import _call
    bb = np.asarray(b, np.float64)
    b2 = bb.reshape(-1, 1) if bb.ndim == 1 else bb
    x = torch.from_numpy(np.ascontiguousarray(b2.T)).to(torch.device("cuda", device))
    torch.cuda.synchronize(device)
    o = opts.native()
    _call("hssmf_mgpu_local", int(device), a._h, t._h, C.byref(o), int(nranks),
          C.c_void_p(x.data_ptr()), int(b2.shape[1]))
    return x.cpu().numpy().T.reshape(bb.shape)
