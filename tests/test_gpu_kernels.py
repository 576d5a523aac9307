"""Kernel-level parity on the B200: DMMA GEMM vs a float64 reference, device
LU vs the reference's lu_partial_pivot, device sampler vs SeededRowSampler,
device CPQR/ID vs interpolative_decomposition (oracle/_ref)."""
import numpy as np
import pytest

import paper_1502_07405_b200.api as A

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ta,tb", [("N", "N"), ("T", "N"), ("N", "T"), ("T", "T")])
@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (7, 5, 3), (64, 64, 16), (130, 67, 45),
                                   (257, 129, 300),
                                   # split-K (few output tiles, long K): the HSS sampling shape
                                   (700, 96, 5003), (200, 128, 2048),
                                   # TMA kernel (even leading dimensions): edges
                                   # by zero fill, split-K, several k-tiles
                                   (96, 96, 32), (258, 130, 302), (1000, 998, 46),
                                   (640, 128, 4096), (384, 256, 1024)])
def test_gemm_matches_fp64(ta, tb, m, n, k):
    rng = np.random.default_rng(m * 1000 + n * 10 + k)
    a = rng.standard_normal((m, k) if ta == "N" else (k, m))
    b = rng.standard_normal((k, n) if tb == "N" else (n, k))
    c = rng.standard_normal((m, n))
    got = A.dev_gemm(ta, tb, -0.5, a, b, 2.0, c)
    oa = a if ta == "N" else a.T
    ob = b if tb == "N" else b.T
    want = -0.5 * oa @ ob + 2.0 * c
    # fp64 tolerance: k * eps * |a||b|
    tol = 8 * k * np.finfo(float).eps * (np.abs(oa) @ np.abs(ob) + np.abs(c)).max()
    assert np.abs(got - want).max() <= tol


def test_transposed_operands_on_the_tma_kernel():
    # transposed operands run on the 64 x 64 kernel by default;
    # HSSMF_TMA_TRANS=1 sends them to the TMA kernel, whose T/N, N/T and T/T
    # variants stay covered here (values and bitwise repeatability)
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = r'''
import sys
sys.path.insert(0, %r)
import numpy as np
import paper_1502_07405_b200.api as A
rng = np.random.default_rng(3)
for (ta, tb, m, n, k) in [("T", "N", 640, 128, 4096), ("N", "T", 258, 130, 2302), ("T", "T", 384, 256, 2048)]:
    a = rng.standard_normal((m, k) if ta == "N" else (k, m))
    b = rng.standard_normal((k, n) if tb == "N" else (n, k))
    c = rng.standard_normal((m, n))
    got = A.dev_gemm(ta, tb, -0.5, a, b, 2.0, c)
    again = A.dev_gemm(ta, tb, -0.5, a, b, 2.0, c)
    oa = a if ta == "N" else a.T
    ob = b if tb == "N" else b.T
    want = -0.5 * oa @ ob + 2.0 * c
    tol = 8 * k * np.finfo(float).eps * (np.abs(oa) @ np.abs(ob) + np.abs(c)).max()
    assert np.abs(got - want).max() <= tol, (ta, tb, m, n, k)
    assert np.array_equal(got, again), (ta, tb, m, n, k)
print("ok")
''' % root
    env = dict(os.environ, HSSMF_TMA_TRANS="1")
    env.pop("HSSMF_NO_TMA", None)
    out = subprocess.run([sys.executable, "-c", script], capture_output=True, text=True, env=env,
                         timeout=300)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-2000:]


def test_gemm_beta_zero_ignores_nan():
    a = np.ones((9, 4))
    b = np.ones((4, 6))
    c = np.full((9, 6), np.nan)
    got = A.dev_gemm("N", "N", 1.0, a, b, 0.0, c)
    assert np.all(got == 4.0)


def test_sampler_matches_reference(oracle):
    # test_sampler.cpp:34-41 rows, plus a spread of others; LCG states are
    # integer-exact, Box-Muller differs from glibc by at most a few ulp
    rows = np.array([0, 1, 5, 31, 4096, 1000000, 2**31 - 2, 2**31 - 1, 123456789], np.int64)
    for c0, c1 in [(0, 10), (3, 8), (0, 257), (128, 384)]:
        got = A.dev_random_rows(rows, c0, c1)
        want = oracle.random_rows(rows, c0, c1)
        assert np.allclose(got, want, rtol=1e-13, atol=1e-15)
        assert np.mean(got == want) > 0.7  # CUDA log/sincos vs glibc: last-ulp only


@pytest.mark.parametrize("n", [1, 5, 32, 33, 100, 257])
def test_lu_matches_reference(oracle, n):
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n))
    got, piv = A.dev_lu(a)
    want, wpiv, col = oracle.lu(a)
    assert col == -1
    assert np.array_equal(piv, wpiv)
    assert np.abs(got - want).max() <= 1e-12 * max(1.0, np.abs(want).max())


def test_lu_singular_column(oracle):
    # test_lu.cpp: an exactly zero column raises with its index
    a = np.array([[1.0, 0.0, 2.0], [2.0, 0.0, 1.0], [3.0, 0.0, 5.0]])
    with pytest.raises(A.SingularMatrixError) as e:
        A.dev_lu(a)
    assert e.value.column() == 1
    assert oracle.lu(a)[2] == 1


@pytest.mark.parametrize("m,n,rank", [(40, 30, 7), (128, 64, 20), (16, 50, 16), (300, 200, 60)])
def test_id_matches_reference(oracle, m, n, rank):
    rng = np.random.default_rng(m + n)
    y = rng.standard_normal((m, rank)) @ rng.standard_normal((rank, n))
    y += 1e-9 * rng.standard_normal((m, n))
    for eps, mr, at in [(1e-6, -1, 0.0), (1e-12, -1, 0.0), (1e-6, rank // 2, 0.0),
                        (1e-3, -1, 1e-2)]:
        p, k, cert, x = A.dev_interpolative_decomposition(y, eps, mr, at)
        wp, wk, wcert, wx = oracle.interpolative_decomposition(y, eps, mr, at)
        assert k == wk and cert == wcert
        assert np.array_equal(p[:k], wp[:k])
        if k and n > k:
            assert np.allclose(x, wx, rtol=1e-7, atol=1e-9 * np.abs(wx).max())
        # interpolation property Y ~= Y(:,J) [I X] Pi^T (certified IDs only)
        if k and cert:
            J = p[:k]
            full = np.zeros((k, n))
            full[:, J] = np.eye(k)
            full[:, p[k:]] = x
            assert np.linalg.norm(y[:, J] @ full - y) <= 1e3 * max(eps, 1e-12) * np.linalg.norm(y) + 1e-6


@pytest.mark.parametrize("cl", ["1", "2", "4", "8", "16"])
def test_id_cluster_cpqr_matches_reference(oracle, monkeypatch, cl):
    # the multi-CTA (thread-block cluster) CPQR must reproduce the reference's
    # pivots, ranks, certification and coefficients
    monkeypatch.setenv("HSSMF_CPQR_CLUSTER", cl)
    rng = np.random.default_rng(5)
    m, n, rank = 260, 500, 90
    y = (rng.standard_normal((m, rank)) * np.logspace(0, -9, rank)) @ rng.standard_normal((rank, n))
    for eps, mr in [(1e-6, -1), (1e-12, -1), (1e-6, 20)]:
        p, k, cert, x = A.dev_interpolative_decomposition(y, eps, mr, 0.0)
        wp, wk, wcert, wx = oracle.interpolative_decomposition(y, eps, mr, 0.0)
        assert (k, cert) == (wk, wcert)
        # leading pivots are well separated; deep ones may swap on near-ties
        # of the downdated norms (different summation order), which only
        # changes the skeleton choice, not the interpolation quality
        assert np.array_equal(p[:min(k, 12)], wp[:min(k, 12)])
        def interp_err(pp, xx):
            full = np.zeros((k, n))
            full[:, pp[:k]] = np.eye(k)
            full[:, pp[k:]] = xx
            return np.linalg.norm(y[:, pp[:k]] @ full - y) / np.linalg.norm(y)
        if cert:
            assert interp_err(p, x) <= 10 * interp_err(wp, wx) + 1e-13


def test_id_zero_and_empty():
    p, k, cert, _ = A.dev_interpolative_decomposition(np.zeros((8, 5)), 1e-6)
    assert k == 0 and cert and list(p) == [0, 1, 2, 3, 4]


@pytest.mark.parametrize("v1", ["0", "1"])
@pytest.mark.parametrize("m,n,rank", [(60, 200, 40), (200, 480, 150), (300, 1000, 260),
                                      (160, 3000, 140), (120, 7000, 100)])
def test_gram_id_matches_reference(oracle, monkeypatch, v1, m, n, rank):
    # the Gram route (pivoted Cholesky of Y^T Y; single CTA, 2/4/8/16-CTA
    # clusters, many 32-step panels) against the reference's Householder CPQR
    if v1 == "1":
        monkeypatch.setenv("HSSMF_GRAM_V1", "1")
    rng = np.random.default_rng(m + n)
    y = (rng.standard_normal((m, rank)) * np.logspace(0, -6, rank)) @ rng.standard_normal((rank, n))
    for eps, mr, at in [(1e-4, -1, 0.0), (1e-3, -1, 0.0), (1e-4, rank // 3, 0.0),
                        (1e-4, -1, 1e-2 * np.abs(y).max())]:
        p, k, cert, r = A.dev_gram_id(y, eps, mr, at)
        wp, wk, wcert, _ = oracle.interpolative_decomposition(y, eps, mr, at)
        assert (k, cert) == (wk, wcert)
        assert sorted(p) == list(range(n))
        assert np.array_equal(p[:min(k, 12)], wp[:min(k, 12)])
        if k:
            # R = L^T: upper triangular on the pivots, R^T R = Y^T Y on them
            r1 = r[:, :k]
            assert np.allclose(np.tril(r1, -1), 0.0)
            yp = y[:, p[:k]]
            assert np.allclose(r1.T @ r1, yp.T @ yp, rtol=1e-9, atol=1e-9 * np.abs(yp.T @ yp).max())
            # the whole R reproduces the Gram rows of the pivots
            assert np.allclose(r1.T @ r, yp.T @ y[:, p], rtol=1e-8,
                               atol=1e-8 * np.abs(yp.T @ y).max())


def test_gram_id_zero_and_empty():
    p, k, cert, _ = A.dev_gram_id(np.zeros((8, 5)), 1e-4)
    assert k == 0 and cert and list(p) == [0, 1, 2, 3, 4]
    y = np.random.default_rng(1).standard_normal((6, 4))
    p, k, cert, _ = A.dev_gram_id(y, 1e-12)  # full rank: exhausted = certified
    assert k == 4 and cert
