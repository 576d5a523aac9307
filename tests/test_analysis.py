"""Host analysis: integer outputs bit-exact with the reference (north star).

Compares the product's native C++ analysis (grid generators, geometric ND,
from_separators, symbolic, cluster trees) with the reference compiled in
oracle/_ref on the same inputs."""
import numpy as np
import pytest

import paper_1502_07405_b200 as P

TREE_FIELDS = ["sep_begin", "sep_end", "child0", "child1", "parent", "level", "upd_ptr",
               "upd_ind"]


@pytest.mark.parametrize("kind,k,nd_leaf", [("p2d", 7, 4), ("p2d", 31, 16), ("p2d", 256, 64),
                                             ("p3d", 16, 32), ("p3d", 33, 32), ("c2d", 40, 8),
                                             ("c3d", 12, 16), ("p2d", 1, 4), ("p3d", 2, 1)])
def test_pipeline_bit_exact(oracle, kind, k, nd_leaf):
    op = P.ordered_grid(kind, k, nd_leaf)
    o = oracle.ordered_grid(kind, k, nd_leaf)
    assert np.array_equal(op.perm, o.perm)
    for mine, theirs in zip(op.a.arrays(), (o.ptr, o.ind, o.val)):
        assert np.array_equal(mine, theirs)  # values too: bitwise
    for f in TREE_FIELDS:
        assert np.array_equal(getattr(op.t, f), getattr(o, f)), f


def test_c5_analysis_bit_exact(oracle):
    # the bench workload's integer structure (BASELINE config 5: P3D 128^3,
    # ND leaf 32): permutation, CSR, tree and upd sets identical to the
    # reference's
    op = P.ordered_grid("p3d", 128, 32)
    o = oracle.ordered_grid("p3d", 128, 32)
    assert np.array_equal(op.perm, o.perm)
    for mine, theirs in zip(op.a.arrays(), (o.ptr, o.ind, o.val)):
        assert np.array_equal(mine, theirs)
    for f in TREE_FIELDS:
        assert np.array_equal(getattr(op.t, f), getattr(o, f)), f


def test_grid_generator_values_bitwise(oracle):
    for kind in ["p2d", "p3d", "c2d", "c3d"]:
        g = P.generate_grid_problem(kind, 9, 1e-3)
        ptr, ind, val = oracle.grid_csr(kind, 9, 1e-3)
        a = g.A.arrays()
        assert np.array_equal(a[0], ptr) and np.array_equal(a[1], ind)
        assert a[2].tobytes() == val.tobytes()


def test_convdiff_operator_fed_to_oracle(oracle):
    # config 4's operator is ours; the oracle must order it identically
    g = P.generate_convdiff3d(12, 0.1)
    ptr, ind, val = g.A.arrays()
    op = P.ordered_problem(g, 32)
    o = oracle.ordered_csr_geom(ptr, ind, val, (12, 12, 12), 3, 32)
    assert np.array_equal(op.perm, o.perm)
    for f in TREE_FIELDS:
        assert np.array_equal(getattr(op.t, f), getattr(o, f)), f
    # upwind rule (grid_problems.hpp:57-61): diag 6.175, minus sides -1.1/-1.05/-1.025
    A = np.zeros((12 ** 3, 12 ** 3))
    for r in range(12 ** 3):
        A[r, ind[ptr[r]:ptr[r + 1]]] = val[ptr[r]:ptr[r + 1]]
    r = 5 + 12 * (5 + 12 * 5)
    assert A[r, r] == pytest.approx(6.175, abs=1e-12)
    assert A[r, r - 1] == pytest.approx(-1.1, abs=1e-12)
    assert A[r, r - 12] == pytest.approx(-1.05, abs=1e-12)
    assert A[r, r - 144] == pytest.approx(-1.025, abs=1e-12)
    assert A[r, r + 1] == A[r, r + 12] == A[r, r + 144] == -1.0


@pytest.mark.parametrize("ns,nu,leaf", [(128, 256, 64), (191, 319, 64), (4096, 0, 128),
                                        (2048, 4096, 128), (5, 7, 16), (0, 0, 8), (3, 0, 1)])
def test_front_cluster_tree_bit_exact(oracle, ns, nu, leaf):
    mine = P.front_cluster_tree(ns, nu, leaf)
    theirs = oracle.cluster_front(ns, nu, leaf)
    for a, b in zip(mine, theirs):
        assert np.array_equal(a, b)


def test_symbolic_kat():
    # reference test_ordering.cpp:253-287: a hand-built tree with known upd sets
    # path graph on 8 vertices plus the edges that create the documented fill
    import itertools
    trip = [(i, i, 4.0) for i in range(8)]
    for i, j in [(0, 4), (0, 5), (1, 4), (1, 5), (1, 7), (2, 5), (2, 6), (3, 6), (3, 7),
                 (2, 7)]:
        trip += [(i, j, -1.0), (j, i, -1.0)]
    trip.sort()
    n = 8
    ptr = np.zeros(n + 1, np.int32)
    for i, _, _ in trip:
        ptr[i + 1] += 1
    ptr = np.cumsum(ptr).astype(np.int32)
    ind = np.array([j for _, j, _ in trip], np.int32)
    val = np.array([v for _, _, v in trip])
    a = P.SparseMatrix.from_csr(n, ptr, ind, val)
    # leaves {0},{1} under sep {4}; leaves {2},{3} under sep {5}... build a
    # 7-node tree: 0,1 -> 2(sep 4); 3(2),4(3) -> 5(sep 5,6); root 6 (sep 7)
    t = P.EliminationTree.from_arrays(
        n, [0, 1, 4, 2, 3, 5, 7], [1, 2, 5, 3, 4, 7, 8], [-1, -1, 0, -1, -1, 3, 2],
        [-1, -1, 1, -1, -1, 4, 5], [2, 2, 6, 5, 5, 6, -1])
    P.symbolic_factorization(a, t)
    # brute-force elimination-graph oracle for the same supernodes
    adj = {i: set() for i in range(n)}
    for i, j, _ in trip:
        if i != j:
            adj[i].add(j)
            adj[j].add(i)
    def upd_of(node):
        lo, hi = t.sep_begin[node], t.sep_end[node]
        s = set()
        for c in range(lo, hi):
            s |= {x for x in adj[c] if x >= hi}
        for ch in (t.child0[node], t.child1[node]):
            if ch >= 0:
                s |= {x for x in upd_of(ch) if x >= hi}
        return s
    for i in range(t.size()):
        assert list(t.upd(i)) == sorted(upd_of(i))
    del itertools
