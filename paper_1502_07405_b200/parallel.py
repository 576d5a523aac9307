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
