"""The subtree-partitioned factorization and solve on one
GPU: every rank's engine lives in this process and the messages go through
an in-process mailbox. Each front is factored by the same kernels on the same
data as in the single-engine run, so the solution must be bitwise identical."""
import numpy as np
import pytest

import paper_1502_07405_b200 as P
from paper_1502_07405_b200.problems import csr_matvec, x_true

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,k,nd_leaf,so,nranks", [
    ("p2d", 64, 16, dict(mode="mf"), 2),
    ("p2d", 64, 16, dict(mode="mf"), 4),
    ("p3d", 24, 32, dict(min_hss=300, eps=1e-6, leaf=64, ls=64), 2),
    ("p3d", 24, 32, dict(min_hss=300, eps=1e-6, leaf=64, ls=64), 4),
])
def test_partitioned_equals_single(kind, k, nd_leaf, so, nranks):
    from paper_1502_07405_b200.parallel import DistributedMf
    op = P.ordered_grid(kind, k, nd_leaf)
    ptr, ind, val = op.a.arrays()
    b = csr_matvec(ptr, ind, val, x_true(op.a.size(), 1))
    opts = P.SolverOptions(nd_leaf=nd_leaf, **so)
    m = P.mf_factor(op.a, op.t, opts)
    x1 = P.mf_solve_new(m, b)
    d = DistributedMf(op.a, op.t, opts, nranks)
    d.factor()
    x2 = d.solve(b)
    assert np.array_equal(x1, x2)
    # every front factored once, by its owner, with the same outcome
    for r, e in d.engines.items():
        own = np.nonzero(d.part.owner == r)[0]
        assert np.array_equal(e.m.type[own], m.type[own])
        assert np.array_equal(e.m.rank[own], m.rank[own])
    if so.get("mode") != "mf":
        assert m.hss_fronts > 0
    # refactor + solve again (the phases restart from the deepest level)
    d.factor()
    assert np.array_equal(d.solve(b), x1)


@pytest.mark.parametrize("kind,k,nd_leaf,so,nranks", [
    ("p2d", 64, 16, dict(mode="mf"), 4),
    ("p3d", 24, 32, dict(min_hss=300, eps=1e-6, leaf=64, ls=64), 2),
    ("p3d", 24, 32, dict(min_hss=300, eps=1e-6, leaf=64, ls=64), 4),
])
def test_native_driver_equals_single(kind, k, nd_leaf, so, nranks):
    # the C++ driver of the phased protocol (csrc/mgpu.cu, the path the C++
    # drop-in uses over NCCL) with all ranks in this process: bitwise equal
    # to one engine, two right-hand sides
    from paper_1502_07405_b200.parallel import native_local_solve
    op = P.ordered_grid(kind, k, nd_leaf)
    ptr, ind, val = op.a.arrays()
    b = csr_matvec(ptr, ind, val, x_true(op.a.size(), 1))
    b2 = np.stack([b, 2.0 * b - 1.0], axis=1)
    opts = P.SolverOptions(nd_leaf=nd_leaf, **so)
    m = P.mf_factor(op.a, op.t, opts)
    x1 = P.mf_solve_new(m, b2)
    x2 = native_local_solve(op.a, op.t, opts, nranks, b2)
    assert np.array_equal(x1, x2)
