"""C5 single-GPU solve with per-kernel error checks (no graphs) -- repro helper."""
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
Bd = B.device()
Bd.use_graphs = os.environ.get("GRAPHS", "0") == "1"
torch.cuda.synchronize()
print("setup ok", type(B.relaxation).__name__, flush=True)
for rep in range(int(os.environ.get("REPS", "3"))):
    res = P.gmres_solve(A, torch.from_numpy(b).cuda(), None, B, cfg.gmres_params())
    torch.cuda.synchronize()
    print(rep, res.outer, res.inner, f"{res.rel_residual:.6e}", flush=True)
