"""Report formats (reference src/stats.cpp:37-123): schema-1 JSON keys and the
CSV header / quoting / %.17g reals."""
import json

from paper_1502_07405_b200.stats import RunStats, stats_csv_header, stats_csv_row, stats_to_json


def test_json_schema_v1_layout():
    s = RunStats(source="p3d 64", n=262144, nnz=1810432, eps=1e-4, hss_fronts=120, relres=7.5e-4,
                 per_front=[dict(id=0, level=3, dim=100, sep=10, rank=0, flops=5, type="dense")])
    j = json.loads(stats_to_json(s))
    assert j["schema_version"] == 1
    assert set(j) == {"schema_version", "config", "timings", "factor", "solve", "per_front"}
    assert set(j["timings"]) == {"analysis", "factor", "solve", "total"}
    assert set(j["solve"]) == {"method", "iterations", "relres", "absres", "converged"}
    assert {"factor_flops", "factor_nnz", "hss_fronts", "hss_fallbacks", "tree_depth",
            "max_rank", "peak_bytes"} <= set(j["factor"])
    assert j["per_front"][0]["type"] == "dense"
    assert "per_front" not in json.loads(stats_to_json(s, include_per_front=False))
    s.error = "front 3: singular"
    assert json.loads(stats_to_json(s))["error"] == s.error


def test_csv_row_matches_header_and_quotes():
    s = RunStats(source='a,"b"', eps=0.1, relres=1.0 / 3.0)
    h = stats_csv_header().split(",")
    row = stats_csv_row(s)
    assert h[0] == "source" and h[-1] == "error" and len(h) == 39
    assert row.startswith('"a,""b"""')
    assert "0.33333333333333331" in row and "0.10000000000000001" in row


def _cases():
    pf = [dict(id=0, level=3, dim=100, sep=10, rank=0, flops=5, type="dense"),
          dict(id=1, level=2, dim=4096, sep=1024, rank=1142, flops=27880000000, type="hss"),
          dict(id=2, level=0, dim=7, sep=7, rank=0, flops=228, type="hss_dense")]
    yield RunStats(source="p3d 64", n=262144, nnz=1810432, ls=64, eps=1e-4, leaf=128, d0=128,
                   dd=128, p=10, min_hss=1000, rank_guard=5000, threads=6, nd_leaf=32,
                   t_analysis=0.4, t_factor=133.5, t_solve=0.078, t_total=133.978,
                   factor_flops=2788250896197, factor_nnz=354000000, factor_nnz_bytes=2832000000,
                   peak_bytes=4900000000, max_rank=1142, fronts=9633, hss_fronts=120,
                   tree_depth=14, method="gmres", iterations=7, relres=7.540352765509328e-4,
                   absres=1.25e-10, converged=True, per_front=pf)
    yield RunStats(source='odd,"name"', strategy="graph", mode="mf", n=7, nnz=19, eps=0.1,
                   rank_guard=3,
                   rtol=1e-12, atol=0.0, relres=1.0 / 3.0, absres=2.5e-300, converged=False,
                   method="refinement", error="front 0: singular, column 1", per_front=[])


def test_json_and_csv_bytes_match_reference(oracle):
    # byte-identical to the reference's own src/stats.cpp (compiled into the
    # oracle with nlohmann json): schema-1 JSON with and without the per-front
    # list, the CSV header and row
    for s in _cases():
        for inc in (True, False):
            rj, rh, rr = oracle.stats_strings(s, inc)
            assert stats_to_json(s, inc) == rj
        assert stats_csv_header() == rh
        assert stats_csv_row(s) == rr
