"""Multifrontal factor + solve on the B200 vs the reference (oracle/_ref).

North-star gate with HSS disabled: solution within 1e-10 of the reference.
Restates the reference's multifrontal KATs (test_multifrontal.cpp)."""
import numpy as np
import pytest

import paper_1502_07405_b200 as P
from paper_1502_07405_b200.problems import csr_matvec, x_true

pytestmark = pytest.mark.gpu


def rhs(op, seed=1):
    ptr, ind, val = op.a.arrays()
    return csr_matvec(ptr, ind, val, x_true(op.a.size(), seed))


@pytest.mark.parametrize("kind,k,nd_leaf", [("p2d", 7, 4), ("p2d", 10, 8), ("p2d", 31, 16),
                                             ("p2d", 256, 64), ("p3d", 16, 32),
                                             ("c3d", 14, 16)])
def test_pure_mf_matches_reference(oracle, kind, k, nd_leaf):
    op = P.ordered_grid(kind, k, nd_leaf)
    b = rhs(op)
    m = P.mf_factor(op.a, op.t, P.SolverOptions(mode="mf"))
    x = P.mf_solve_new(m, b)
    o = oracle.ordered_grid(kind, k, nd_leaf)
    xr = oracle.Factors(o, mode=1).solve(b)[:, 0]
    assert np.linalg.norm(x - xr) / np.linalg.norm(xr) <= 1e-10
    assert m.hss_fronts == 0
    A = op.a
    r = A.matvec(x) - b
    assert np.linalg.norm(r) / np.linalg.norm(b) <= 1e-12


def test_multi_rhs_bitwise_equal_single():
    # test_multifrontal.cpp:340-346
    op = P.ordered_grid("p2d", 10, 8)
    m = P.mf_factor(op.a, op.t, P.SolverOptions())
    rng = np.random.default_rng(8)
    b3 = np.asfortranarray(rng.uniform(-1, 1, (op.a.size(), 3)))
    x3 = P.mf_solve_new(m, b3)
    for c in range(3):
        xc = P.mf_solve_new(m, np.asfortranarray(b3[:, c:c + 1]))
        assert xc.tobytes() == np.ascontiguousarray(x3[:, c:c + 1]).tobytes()


def test_known_solution_all_ones():
    op = P.ordered_grid("p2d", 10, 8)
    m = P.mf_factor(op.a, op.t, P.SolverOptions())
    ones = np.ones(op.a.size())
    x = P.mf_solve_new(m, op.a.matvec(ones))
    assert np.abs(x - 1).max() <= 1e-10


def _csr(n, trip):
    trip = sorted(trip)
    ptr = np.zeros(n + 1, np.int32)
    for i, _, _ in trip:
        ptr[i + 1] += 1
    return P.SparseMatrix.from_csr(n, np.cumsum(ptr).astype(np.int32),
                                   np.array([j for _, j, _ in trip], np.int32),
                                   np.array([v for _, _, v in trip]))


def test_identity_and_scalar_front():
    # test_multifrontal.cpp:289-318
    a = _csr(6, [(i, i, 1.0) for i in range(6)])
    t = P.EliminationTree.from_arrays(6, [0], [6], [-1], [-1], [-1], upd=[[]])
    m = P.mf_factor(a, t, P.SolverOptions())
    assert m.front_stats[0].type == "dense"
    b = np.asfortranarray(np.random.default_rng(91).uniform(-1, 1, (6, 2)))
    assert P.mf_solve_new(m, b).tobytes() == b.tobytes()
    a1 = _csr(1, [(0, 0, 2.0)])
    t1 = P.EliminationTree.from_arrays(1, [0], [1], [-1], [-1], [-1], upd=[[]])
    m1 = P.mf_factor(a1, t1, P.SolverOptions())
    assert P.mf_solve_new(m1, np.array([3.0]))[0] == 1.5


def test_empty_synthetic_root():
    # test_multifrontal.cpp:349-383: two decoupled blocks under an empty root
    h, n = 5, 10
    trip = []
    for blk in range(2):
        for i in range(h):
            trip.append((blk * h + i, blk * h + i, 4.0))
            if i + 1 < h:
                trip += [(blk * h + i, blk * h + i + 1, -1.0), (blk * h + i + 1, blk * h + i, -1.0)]
    a = _csr(n, trip)
    t = P.EliminationTree.from_arrays(n, [0, h, n], [h, n, n], [-1, -1, 0], [-1, -1, 1],
                                      [2, 2, -1], upd=[[], [], []])
    m = P.mf_factor(a, t, P.SolverOptions())
    b = np.random.default_rng(17).uniform(-1, 1, n)
    x = P.mf_solve_new(m, b)
    D = np.zeros((n, n))
    for i, j, v in trip:
        D[i, j] = v
    assert np.abs(x - np.linalg.solve(D, b)).max() <= 1e-12


def test_singular_front_names_front_and_column():
    # test_multifrontal.cpp:483-500
    a = _csr(3, [(0, 0, 1.0), (0, 1, 0.0), (1, 0, 0.0), (2, 2, 1.0)])
    t = P.EliminationTree.from_arrays(3, [0], [3], [-1], [-1], [-1], upd=[[]])
    with pytest.raises(P.SingularMatrixError) as e:
        P.mf_factor(a, t, P.SolverOptions())
    assert "front 0" in str(e.value)
    assert e.value.column() == 1


def test_argument_errors():
    # test_multifrontal.cpp:502-522
    a = _csr(2, [(0, 0, 1.0), (1, 1, 1.0)])
    a3 = _csr(3, [(0, 0, 1.0), (1, 1, 1.0), (2, 2, 1.0)])
    t = P.EliminationTree.from_arrays(2, [0], [2], [-1], [-1], [-1], upd=[[]])
    with pytest.raises(P.IoError):
        P.mf_factor(a3, t, P.SolverOptions())
    m = P.mf_factor(a, t, P.SolverOptions())
    with pytest.raises(P.IoError):
        P.mf_solve(m, np.zeros((5, 1), order="F"))
