"""The header-only C++ drop-in (include/hssmf_b200/hssmf.hpp) used from a
program written against the reference's own types (tests/cpp/wrapper_check.cpp,
built by `make -C oracle wrapper` in the build container)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "wrapper_check")


def _need():
    if not os.path.exists(BIN):
        pytest.skip("wrapper_check not built (make -C oracle wrapper)")


def test_wrapper_links_against_library():
    _need()
    out = subprocess.run([BIN, "--version"], capture_output=True, text=True, check=True)
    assert "sm_100a" in out.stdout


@pytest.mark.gpu
def test_wrapper_drop_in_factor_solve():
    _need()
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["relres"] < 1e-12 and d["singular_col"] == 1 and d["front0"] == 1
    assert d["gmres_converged"] == 1 and d["gmres_iterations"] <= 2
    # reordered separators forwarded through the drop-in: HSS ranks within
    # +-10% of the reference's own mf_factor on the same tree
    assert d["reorder_hss_fronts"] > 0 and d["reorder_ranks_close"] == 1


DROPIN = os.path.join(ROOT, "oracle", "_ref", "dropin_check")


@pytest.mark.gpu
def test_dropin_reference_names_and_signatures(oracle):
    # include/hssmf_b200/dropin.hpp replaces the reference's multifrontal /
    # hss_compress / hss_ulv headers: reference-named calls with reference
    # signatures, results checked against the oracle on the same inputs
    if not os.path.exists(DROPIN):
        pytest.skip("dropin_check not built (make -C oracle dropin)")
    import numpy as np
    from paper_1502_07405_b200.problems import dense_c2
    out = subprocess.run([DROPIN], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["mf_relres"] < 1e-12
    assert d["singular_col"] == 1 and d["front0"] == 1
    assert d["rank_guard"] == 1 and d["io"] == 1
    # HSS fronts of P3D 24^3 vs the reference's mf_factor on the same tree
    o = oracle.ordered_grid("p3d", 24, 16)
    F = oracle.Factors(o, eps=1e-6, ls=64, min_hss=250, leaf=32)
    ref_ids = [int(i) for i in np.nonzero(F.type == 1)[0]]
    assert d["hss_ids"] == ref_ids and d["hss_fronts"] == F.hss_fronts
    ref_ranks = np.array([int(F.rank[i]) for i in ref_ids])
    assert np.all(np.abs(np.array(d["hss_ranks"]) - ref_ranks) <= np.maximum(2, 0.1 * ref_ranks))
    # dense HSS (config 2's operator at N = 2048, balanced leaf 128)
    r = oracle.DenseHss(dense_c2(2048), leaf=128, eps=1e-8)
    ru = np.asarray(r.u_rank[:-1])
    assert np.all(np.abs(np.array(d["dense_u"][:-1]) - ru) <= np.maximum(2, 0.1 * ru))
    assert d["dense_rounds"] == r.rounds and d["dense_d_final"] == r.d_final
    assert d["dense_relres"] < 1e-7 and d["uneven_relres"] < 1e-7


MGPU = os.path.join(ROOT, "oracle", "_ref", "mgpu_check")


@pytest.mark.gpu
def test_nccl_dropin_runs():
    # include/hssmf_b200/mgpu_nccl.hpp: the C++ multi-GPU path over NCCL with
    # every visible GPU (one on a gpurun box) equals the single-GPU drop-in
    if not os.path.exists(MGPU):
        pytest.skip("mgpu_check not built (make -C oracle mgpu)")
    out = subprocess.run([MGPU], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["nranks"] >= 1 and d["max_diff"] == 0.0
