"""Graph nested dissection and separator reordering:
host-side integer outputs bit-exact with the reference (oracle/_ref), plus
the reference's own known-answer cases (test_ordering.cpp:145-186, 380-451)
restated."""
import numpy as np
import pytest

import paper_1502_07405_b200 as P

TREE_FIELDS = ["sep_begin", "sep_end", "child0", "child1", "parent", "level", "upd_ptr",
               "upd_ind"]


def csr_from_edges(n, edges, diag=2.0):
    rows = [[(i, diag)] for i in range(n)]
    for i, j in edges:
        rows[i].append((j, -1.0))
        rows[j].append((i, -1.0))
    ptr, ind, val = [0], [], []
    for r in rows:
        r = sorted(set(r))
        ind += [c for c, _ in r]
        val += [v for _, v in r]
        ptr.append(len(ind))
    return P.SparseMatrix.from_csr(n, np.array(ptr, np.int32), np.array(ind, np.int32),
                                   np.array(val, np.float64))


def random_graph(n, deg, seed):
    rng = np.random.default_rng(seed)
    e = set()
    for i in range(n):
        for j in rng.integers(0, n, deg):
            if i != j:
                e.add((min(i, j), max(i, j)))
    return csr_from_edges(n, sorted(e))


def compare(mine, o):
    assert np.array_equal(mine.perm, o.perm)
    for a, b in zip(mine.a.arrays(), (o.ptr, o.ind, o.val)):
        assert np.array_equal(a, b)
    for f in TREE_FIELDS:
        assert np.array_equal(getattr(mine.t, f), getattr(o, f)), f
    for i in range(o.nnodes):
        for x, y in zip(mine.t.sep_clusters(i), o.sep_clusters(i)):
            assert np.array_equal(x, y), i


def problems():
    yield "p2d9", P.generate_grid_problem("p2d", 9).A
    yield "p2d40", P.generate_grid_problem("p2d", 40).A
    yield "p3d12", P.generate_grid_problem("p3d", 12).A
    yield "c3d9", P.generate_grid_problem("c3d", 9, 1e-3).A
    yield "rand500", random_graph(500, 3, 1)
    yield "rand2000", random_graph(2000, 2, 7)
    # disconnected: two grids side by side plus isolated vertices
    g = P.generate_grid_problem("p2d", 6).A
    ptr, ind, val = g.arrays()
    n = g.size()
    e = [(i, j) for i in range(n) for j in ind[ptr[i]:ptr[i + 1]] if j > i]
    e += [(i + n, j + n) for i, j in e]
    yield "disconnected", csr_from_edges(2 * n + 3, e)


@pytest.mark.parametrize("nd_leaf", [1, 4, 16, 64])
def test_graph_nd_bit_exact(oracle, nd_leaf):
    for name, a in problems():
        mine = P.ordered_graph(a, nd_leaf)
        ptr, ind, val = a.arrays()
        compare(mine, oracle.ordered_graph(ptr, ind, val, nd_leaf))


@pytest.mark.parametrize("b", [1, 3, 8, 32])
def test_separator_reordering_bit_exact(oracle, b):
    for name, a in problems():
        ptr, ind, val = a.arrays()
        mine = P.ordered_graph(a, 16, reorder_b=b)
        compare(mine, oracle.ordered_graph(ptr, ind, val, 16, reorder_b=b))
        # an explicit selection (every other front)
        nn = mine.t.size()
        sel = np.arange(nn) % 2 == 0
        mine = P.ordered_graph(a, 16, reorder_b=b, selected=sel)
        compare(mine, oracle.ordered_graph(ptr, ind, val, 16, reorder_b=b, selected=sel))


def test_path_dissection_picks_the_middle_vertex():
    # test_ordering.cpp:145-166
    a = csr_from_edges(7, [(i, i + 1) for i in range(6)])
    t, perm = P.nested_dissection_graph(a, 3)
    assert sorted(perm) == list(range(7))
    r = t.root_id()
    assert t.sep_end[r] - t.sep_begin[r] == 1
    assert int(np.where(perm == t.sep_begin[r])[0][0]) == 3
    for c in (t.child0[r], t.child1[r]):
        assert c >= 0 and t.sep_end[c] - t.sep_begin[c] == 3


def test_disconnected_components_get_an_empty_separator():
    # test_ordering.cpp:168-186: two disjoint 4-paths
    a = csr_from_edges(8, [(b + i, b + i + 1) for b in (0, 4) for i in range(3)])
    t, perm = P.nested_dissection_graph(a, 4)
    assert sorted(perm) == list(range(8))
    assert t.sep_end[t.root_id()] == t.sep_begin[t.root_id()]


def test_reordering_keeps_the_symbolic_sizes():
    # test_ordering.cpp:405-451: relabeling inside separators changes neither
    # separator nor update sizes; clusters cover each selected separator with
    # leaves of at most b vertices
    a = P.generate_grid_problem("p2d", 9).A
    plain = P.ordered_graph(a, 16)
    t0 = plain.t
    sel = (t0.sep_end - t0.sep_begin) >= 4
    re = P.ordered_graph(a, 16, reorder_b=4, selected=sel)
    t1 = re.t
    assert np.array_equal(t0.sep_begin, t1.sep_begin) and np.array_equal(t0.sep_end, t1.sep_end)
    assert np.array_equal(np.diff(t0.upd_ptr), np.diff(t1.upd_ptr))
    for i in range(t1.size()):
        b, e, c0, c1, par = t1.sep_clusters(i)
        if not sel[i]:
            assert len(b) == 0
            continue
        assert e[-1] - b[-1] == t1.sep_end[i] - t1.sep_begin[i]
        leaves = c0 < 0
        assert np.all(e[leaves] - b[leaves] <= 4)
    # identity outside the selected separators
    r = re.perm[np.argsort(plain.perm)]
    for i in range(t0.size()):
        rng = np.arange(t0.sep_begin[i], t0.sep_end[i])
        assert np.all((r[rng] >= t0.sep_begin[i]) & (r[rng] < t0.sep_end[i]))
        if not sel[i]:
            assert np.array_equal(r[rng], rng)


def test_set_sep_clusters_roundtrip_and_validation():
    a = P.generate_grid_problem("p2d", 9).A
    op = P.ordered_graph(a, 16, reorder_b=4)
    t = op.t
    i = t.root_id()
    b, e, c0, c1, _ = t.sep_clusters(i)
    t2 = P.EliminationTree.from_arrays(t.n, t.sep_begin, t.sep_end, t.child0, t.child1,
                                       t.parent, [t.upd(k) for k in range(t.size())])
    t2.set_sep_clusters(i, b, e, c0, c1)
    for x, y in zip(t2.sep_clusters(i), t.sep_clusters(i)):
        assert np.array_equal(x, y)
    with pytest.raises(P.IoError):
        t2.set_sep_clusters(i, [0, 0], [1, 1], [1, -1], [-1, -1])
