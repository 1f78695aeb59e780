"""Time the K-cycle CPR-GMRES solve on C3 (60x220x85) and compare with the
reference run's golden (outer 2, inner 5,
rel 2.131596607608327e-06)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2201_01970_b200 as P  # noqa: E402

nx, ny, nz = (int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "60,220,85").split(","))
(A, b), = P.generate_blackoil_like_sequence(nx, ny, nz, 1, 0.01, 0).systems
cfg = P.SolverConfig(theta=0.0, theta_amg=0.0, cycle="k")
t0 = time.perf_counter()
B = P.build_cpr(A, cfg)
B.device()
torch.cuda.synchronize()
print("setup s", round(time.perf_counter() - t0, 2))
bd = torch.from_numpy(b).cuda()
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = P.gmres_solve(A, bd, None, B, cfg.gmres_params())
    torch.cuda.synchronize()
    print(f"K-cycle solve {time.perf_counter() - t0:.3f} s outer={res.outer} inner={res.inner} "
          f"rel={res.rel_residual:.16e}")
