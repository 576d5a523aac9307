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
