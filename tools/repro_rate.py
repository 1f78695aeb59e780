"""Failure rate of repeated CPR-GMRES solves (stencil BILU) on one grid."""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2201_01970_b200 as P

grid = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "120,440,170").split(","))
(A, b), = P.generate_blackoil_like_sequence(*grid, 1, 0.01, 0).systems
cfg = P.SolverConfig(theta=0.0, theta_amg=0.0, cycle="v")
B = P.build_cpr(A, cfg)
bd = torch.from_numpy(b).cuda()
n = int(os.environ.get("REPS", "20"))
for rep in range(n):
    res = P.gmres_solve(A, bd, None, B, cfg.gmres_params())
    torch.cuda.synchronize()
print("OK", n, "solves", res.outer, res.inner, f"{res.rel_residual:.6e}", flush=True)
