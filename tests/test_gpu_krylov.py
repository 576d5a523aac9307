"""GPU-resident GMRES / iterative refinement preconditioned by the
multifrontal solve: the reference's test_krylov.cpp cases restated
(tests/unit/test_krylov.cpp:126-293), plus the textbook-GMRES comparison
against a host restatement of the same algorithm."""
import numpy as np
import pytest

import paper_1502_07405_b200 as P

pytestmark = pytest.mark.gpu


def diag_csr(d):
    n = len(d)
    return P.SparseMatrix.from_csr(n, np.arange(n + 1), np.arange(n), np.asarray(d, float))


def identity(n):
    return diag_csr(np.ones(n))


def rel_residual(a, x, b):
    return np.linalg.norm(a.matvec(x) - b) / np.linalg.norm(b)


def test_identity_system_converges_in_one_iteration():  # test_krylov.cpp:126-138
    n = 40
    b = np.random.default_rng(3).standard_normal(n)
    x, rep = P.gmres(identity(n), None, b)
    assert rep.iterations == 1 and rep.converged
    assert np.linalg.norm(x - b) / np.linalg.norm(b) <= 1e-14
    assert len(rep.history) == 2 and rep.abs_resid <= 1e-12


def test_happy_breakdown_returns_the_exact_solution():  # :140-154
    n = 12
    b = np.random.default_rng(11).standard_normal(n)
    x, rep = P.gmres(diag_csr(np.full(n, 2.0)), None, b, 30, 1e-10, 1e-14, 50)
    assert rep.iterations == 1 and rep.converged
    assert np.all(np.abs(x - b / 2) <= 1e-15 * np.abs(b) + 1e-300)


def test_exact_factorization_preconditioner_converges_immediately():  # :156-172
    op = P.ordered_grid("p2d", 10, 8)
    m = P.mf_factor(op.a, op.t, P.SolverOptions())
    b = np.random.default_rng(5).standard_normal(op.a.size())
    x, rep = P.gmres(op.a, m, b, 30, 1e-6, 1e-10, 50)
    assert rep.converged and rep.iterations <= 2
    assert rel_residual(op.a, x, b) <= 1e-8
    xr, repr_ = P.iterative_refinement(op.a, m, b)
    assert repr_.converged and repr_.iterations == 1


def test_crude_compression_still_preconditions():  # :174-191
    op = P.ordered_grid("p3d", 16, 16)
    so = P.SolverOptions(nd_leaf=16, ls=3, min_hss=64, leaf=16, eps=0.9, d0=32, dd=32, p=8)
    m = P.mf_factor(op.a, op.t, so)
    assert m.hss_fronts >= 1
    b = np.random.default_rng(9).standard_normal(op.a.size())
    x, rep = P.gmres(op.a, m, b, 30, 1e-6, 1e-10, 150)
    assert rep.converged and rep.iterations <= 100


def naive_gmres(a, b, restart, maxit):
    """the reference test's textbook restarted GMRES on a dense matrix
    (test_krylov.cpp:44-118), restated with numpy"""
    n = len(b)
    x = np.zeros(n)
    r = b.copy()
    hist = [np.linalg.norm(r)]
    it = 0
    while it < maxit:
        beta = np.linalg.norm(r)
        v = [r / beta]
        h = np.zeros((restart + 1, restart))
        c, s, g = np.zeros(restart), np.zeros(restart), np.zeros(restart + 1)
        g[0] = beta
        j = 0
        while j < restart and it < maxit:
            w = a @ v[j]
            for i in range(j + 1):
                h[i, j] = v[i] @ w
                w = w - h[i, j] * v[i]
            h[j + 1, j] = np.linalg.norm(w)
            for i in range(j):
                t = c[i] * h[i, j] + s[i] * h[i + 1, j]
                h[i + 1, j] = -s[i] * h[i, j] + c[i] * h[i + 1, j]
                h[i, j] = t
            den = np.hypot(h[j, j], h[j + 1, j])
            c[j], s[j] = h[j, j] / den, h[j + 1, j] / den
            h[j, j] = den
            g[j + 1] = -s[j] * g[j]
            g[j] = c[j] * g[j]
            it += 1
            hist.append(abs(g[j + 1]))
            if h[j + 1, j] == 0.0:
                j += 1
                break
            v.append(w / h[j + 1, j])
            j += 1
        y = np.zeros(j)
        for i in range(j - 1, -1, -1):
            y[i] = (g[i] - h[i, i + 1:j] @ y[i + 1:j]) / h[i, i]
        for i in range(j):
            x = x + y[i] * v[i]
        r = b - a @ x
    return x, hist


def test_gmres_matches_a_naive_dense_reference():  # :213-233
    op = P.ordered_grid("p2d", 12, 8)
    n = op.a.size()
    ptr, ind, val = op.a.arrays()
    dense = np.zeros((n, n))
    for i in range(n):
        dense[i, ind[ptr[i]:ptr[i + 1]]] = val[ptr[i]:ptr[i + 1]]
    b = np.random.default_rng(21).standard_normal(n)
    restart, maxit = 8, 24
    x, rep = P.gmres(op.a, None, b, restart, 1e-14, 0.0, maxit)
    xr, hist = naive_gmres(dense, b, restart, maxit)
    assert len(rep.history) == len(hist)
    assert np.all(np.abs(np.array(rep.history) - np.array(hist)) <= 1e-10)
    assert np.all(np.abs(x - xr) <= 1e-10)
    for i in range(2, len(rep.history)):  # nonincreasing within a restart cycle
        if (i - 1) % restart != 0:
            assert rep.history[i] <= rep.history[i - 1] * (1 + 1e-12)


def test_non_finite_arnoldi_entries_raise_a_divergence_error():  # :235-248
    n = 8
    b = np.random.default_rng(2).standard_normal(n)
    d = np.ones(n)
    d[0] = np.nan
    bad = diag_csr(d)
    with pytest.raises(P.KrylovDivergenceError):
        P.gmres(bad, None, b)
    with pytest.raises(P.KrylovDivergenceError):
        P.iterative_refinement(bad, None, b)


def test_refinement_solves_trivial_cases_exactly():  # :250-260
    n = 9
    x, rep = P.iterative_refinement(identity(n), None, np.zeros(n))
    assert rep.converged and rep.iterations == 0 and np.all(x == 0.0)


def test_refinement_against_a_loosely_compressed_factorization():  # :262-279
    op = P.ordered_grid("p2d", 31, 16)
    so = P.SolverOptions(nd_leaf=16, ls=3, min_hss=24, leaf=16, eps=1e-6, d0=32, dd=32, p=8)
    m = P.mf_factor(op.a, op.t, so)
    assert m.hss_fronts >= 1
    b = np.random.default_rng(29).standard_normal(op.a.size())
    x, rep = P.iterative_refinement(op.a, m, b)
    assert rep.converged and rep.iterations <= 10 and not rep.stagnated


def test_refinement_stagnation_is_reported_not_fatal():  # :281-293
    op = P.ordered_grid("p2d", 10, 8)
    b = np.random.default_rng(31).standard_normal(op.a.size())
    x, rep = P.iterative_refinement(op.a, None, b, 1e-6, 1e-10, 8)
    assert not rep.converged and rep.stagnated and rep.iterations == 8


def test_gmres_on_c3_reaches_tight_residual():
    # the paper's use: HSS-compressed factorization (eps 1e-4, relres ~7.5e-4
    # as a direct solve) as a GMRES preconditioner on BASELINE config 3
    from paper_1502_07405_b200.problems import CONFIGS, csr_matvec, x_true
    cfg = CONFIGS["c3"]
    op = P.ordered_grid(cfg.kind, cfg.k, cfg.nd_leaf)
    ptr, ind, val = op.a.arrays()
    b = csr_matvec(ptr, ind, val, x_true(op.a.size(), 1))
    m = P.mf_factor(op.a, op.t, cfg.solver_options())
    x, rep = P.gmres(op.a, m, b, 30, 1e-10, 0.0, 60)
    assert rep.converged
    assert rel_residual(op.a, x, b) <= 1e-9


def test_run_stats_of_a_device_factorization():
    import json
    from paper_1502_07405_b200.stats import run_stats, stats_csv_row, stats_to_json
    op = P.ordered_grid("p2d", 31, 16)
    so = P.SolverOptions(nd_leaf=16, ls=3, min_hss=24, leaf=16, eps=1e-6, d0=32, dd=32, p=8)
    m = P.mf_factor(op.a, op.t, so)
    b = np.random.default_rng(29).standard_normal(op.a.size())
    x, rep = P.iterative_refinement(op.a, m, b)
    s = run_stats(m, so, op.a, source="p2d 31", method="refinement", iterations=rep.iterations,
                  relres=rel_residual(op.a, x, b), converged=rep.converged)
    j = json.loads(stats_to_json(s))
    assert j["factor"]["hss_fronts"] == m.hss_fronts >= 1
    assert j["factor"]["fronts"] == len(j["per_front"]) == len(m.level)
    assert sum(f["type"] == "hss" for f in j["per_front"]) == m.hss_fronts
    assert j["solve"]["converged"] and j["config"]["eps"] == 1e-6
    assert len(stats_csv_row(s).split(",")) >= 39
