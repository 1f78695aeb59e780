"""Rebuild-mix sequence on the device setup path (repro helper)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2201_01970_b200 as P

grid = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "20,30,10").split(","))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
mu = int(sys.argv[3]) if len(sys.argv) > 3 else 0
seq = P.generate_blackoil_like_sequence(*grid, n, 0.05, 0)
cfg = P.SolverConfig(theta=0.0, theta_amg=0.0, cycle="v")
out = P.ascpr_gmres_sequence(seq.systems, mu, cfg, keep_solutions=False)
print("calls", out.setup_calls, [(r.outer, r.inner, r.rebuilt) for r in out.records], flush=True)
