"""Benchmark report compatibility (src/bench.py) against the unmodified
reference's behaviour recorded in tests/golden/report.json
(tests/golden/make_report_golden.py): report.csv bytes (schema=1), the CSV
reader, the config round trip, and -- on the B200 -- a run_benchmark grid
with the reference's setup calls, iteration counts, per-cell details and
hierarchy summary."""

import hashlib
import json

import pytest

from conftest import GOLDEN

from paper_2201_01970_b200 import report as R

G = json.loads((GOLDEN / "report.json").read_text())


def test_report_csv_bytes_match_reference(tmp_path):
    fixed = R.RunReport(rows=[R.BenchRow(0.0, 0, 1, 3, 0.25, 17, 1.5, 1.0, 1.0),
                              R.BenchRow(0.1, 5, 2, 1, 1 / 3, 18, 0.1 + 0.2, None, 2.5)])
    p = tmp_path / "report.csv"
    R.write_report_csv(fixed, p)
    b = p.read_bytes()
    assert hashlib.sha256(b).hexdigest() == G["fixed_csv_sha"], b.decode()
    rows = R.read_report_csv(p)
    assert rows[1]["speedup"] is None and rows[1]["time_s"] == 0.1 + 0.2
    assert rows[0] == fixed.rows[0].as_record()


def test_report_schema_guard(tmp_path):
    p = tmp_path / "bad.csv"
    p.write_text("schema=2\n")
    with pytest.raises(ValueError, match="unsupported report schema"):
        R.read_report_csv(p)


def test_bench_config_round_trip():
    cfg = R.BenchConfig.from_dict(G["config"])
    assert cfg.to_dict() == G["config"]
    with pytest.raises(ValueError, match="unknown bench config keys"):
        R.BenchConfig.from_dict({"nx": 2, "bogus": 1})


@pytest.mark.gpu
def test_run_benchmark_grid_matches_reference(gpu, tmp_path):
    rep = R.run_benchmark(R.BenchConfig.from_dict(G["config"]))
    assert not rep.failures
    rows = [{k: v for k, v in r.as_record().items()
             if k not in ("time_s", "setup_ratio", "speedup", "speedup_star")} for r in rep.rows]
    assert rows == G["rows"]
    cells = [{k: v for k, v in c.items() if not k.endswith("_s")} for c in rep.details["cells"]]
    assert cells == G["cells"]
    assert rep.details["hierarchy"] == G["hierarchy"]
    assert rep.details["provenance"] == G["provenance"]
    R.write_report_csv(rep, tmp_path / "report.csv")
    R.write_report_json(rep, tmp_path / "report.json")
    assert len(R.read_report_csv(tmp_path / "report.csv")) == 4
    assert all(r.speedup is not None and r.speedup_star is not None for r in rep.rows)
