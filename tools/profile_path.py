"""Run pieces of the CPR-GMRES path on the C3 system for profiling under ncu.

    python tools/profile_path.py [--what apply|spmv|bilu|vcycle|solve] [--reps N] [--grid 60,220,85]
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2201_01970_b200 as P  # noqa: E402
from paper_2201_01970_b200 import device as D  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", default="apply")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--grid", default="60,220,85")
    ap.add_argument("--nograph", action="store_true")
    a = ap.parse_args()
    nx, ny, nz = map(int, a.grid.split(","))
    (A, b), = P.generate_blackoil_like_sequence(nx, ny, nz, 1, 0.01, 0).systems
    cfg = P.SolverConfig(theta=0.0, theta_amg=0.0, cycle="v")
    B = P.build_cpr(A, cfg)
    Bd = B.device()
    Bd.use_graphs = not a.nograph
    M = D.device_matrix(A)
    bd = torch.from_numpy(b).cuda()
    z = torch.empty_like(bd)
    zp = D.empty(A.nrows)
    ops = {
        "apply": lambda: Bd.apply(bd, z),
        "spmv": lambda: P.spmv(A, bd),
        "bilu": lambda: Bd.bilu.apply(bd, z),
        "vcycle": lambda: Bd.amg.vcycle(bd, zp),
        "solve": lambda: P.gmres_solve(A, bd, None, B, cfg.gmres_params()),
    }
    fn = ops[a.what]
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(a.reps):
        fn()
    torch.cuda.synchronize()
    print(f"{a.what}: {(time.perf_counter() - t0) / a.reps * 1e3:.3f} ms/rep (wall)")


if __name__ == "__main__":
    main()
