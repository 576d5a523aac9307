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
