"""compute-sanitizer target: C1 CPR-GMRES solves through every device path
(V-cycle with and without the persistent tail, device K-cycle with and
without its tail, device BILU factorization + stencil solves, device
generator).  Small enough to run under memcheck / racecheck / synccheck."""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2201_01970_b200 as P

for cycle, env in (("v", {}), ("v", {"CPRB_TAIL_ROWS": "100000"}), ("k", {}),
                   ("k", {"CPRB_KTAIL_ROWS": "100000"})):
    os.environ.pop("CPRB_TAIL_ROWS", None)
    os.environ.pop("CPRB_KTAIL_ROWS", None)
    os.environ.update(env)
    (A, b), = P.generate_blackoil_like_sequence(10, 10, 10, 1, 0.01, 0).systems
    cfg = P.SolverConfig(theta=0.0, theta_amg=0.0, cycle=cycle)
    B = P.build_cpr(A, cfg)
    res = P.gmres_solve(A, b, None, B, cfg.gmres_params())
    print(cycle, env, res.outer, res.inner, f"{res.rel_residual:.6e}", flush=True)
