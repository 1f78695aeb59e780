"""Golden behaviour of the reference's benchmark report (cprkit.bench,
src/bench.py): a small run_benchmark grid (iteration counts, setup calls,
per-cell details and the hierarchy summary -- everything but wall times) and
the exact bytes of report.csv for a fixed row set.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_report_golden.py
"""
import hashlib
import json
import sys
import tempfile
from pathlib import Path

OUT = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
from cprkit.bench import BenchConfig, BenchRow, RunReport, run_benchmark, write_report_csv  # noqa: E402

cfg = BenchConfig.from_dict({"nx": 8, "ny": 8, "nz": 2, "nsteps": 3, "drift": 0.05, "seed": 1,
                             "thetas": [0.0], "mus": [0, 5], "workers": [1, 2],
                             "solver": {"cycle": "v", "theta_amg": 0.0}})
rep = run_benchmark(cfg)
rows = [{k: v for k, v in r.as_record().items() if k not in ("time_s", "setup_ratio", "speedup",
                                                             "speedup_star")} for r in rep.rows]
cells = [{k: v for k, v in c.items() if not k.endswith("_s")} for c in rep.details["cells"]]
fixed = RunReport(rows=[BenchRow(0.0, 0, 1, 3, 0.25, 17, 1.5, 1.0, 1.0),
                        BenchRow(0.1, 5, 2, 1, 1 / 3, 18, 0.1 + 0.2, None, 2.5)])
with tempfile.TemporaryDirectory() as td:
    p = Path(td) / "report.csv"
    write_report_csv(fixed, p)
    csv_bytes = p.read_bytes()
out = {"config": cfg.to_dict(), "rows": rows, "cells": cells,
       "hierarchy": rep.details["hierarchy"], "provenance": rep.details["provenance"],
       "fixed_csv": csv_bytes.decode(), "fixed_csv_sha": hashlib.sha256(csv_bytes).hexdigest()}
(OUT / "report.json").write_text(json.dumps(out, indent=1) + "\n")
print(json.dumps(out, indent=1)[:1500])
