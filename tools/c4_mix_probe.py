"""Find an SPE10-shaped (C3 grid) Newton-sequence configuration whose ASCPR
run mixes reuse and rebuild (src/cpr.py:204-212, :349-382)."""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2201_01970_b200 as P

grid = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "60,220,85").split(","))
for drift, mu in ((0.05, 5), (0.1, 5), (0.2, 5), (0.3, 6)):
    t = time.perf_counter()
    seq = P.generate_blackoil_like_sequence(*grid, 6, drift, 0)
    cfg = P.SolverConfig(theta=0.0, theta_amg=0.0, cycle="v")
    out = P.ascpr_gmres_sequence(seq.systems, mu, cfg, keep_solutions=False)
    print(f"drift={drift} mu={mu} calls={out.setup_calls} "
          f"its={[(r.outer, r.inner) for r in out.records]} rebuilt={[int(r.rebuilt) for r in out.records]} "
          f"conv={out.all_converged} {time.perf_counter() - t:.1f}s", flush=True)
