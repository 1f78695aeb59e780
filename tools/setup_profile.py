"""Where does SETUP time go on C3?  build_cpr (host) and the first device()
upload, each under cProfile; prints the top cumulative entries."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2201_01970_b200 as P  # noqa: E402

grid = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "60,220,85").split(","))
t = time.perf_counter()
(A, b), = P.generate_blackoil_like_sequence(*grid, 1, 0.01, 0).systems
print(f"generate {time.perf_counter() - t:.2f} s")
cfg = P.SolverConfig(theta=0.0, theta_amg=0.0, cycle="v")
for what in ("build_cpr", "device"):
    pr = cProfile.Profile()
    torch.cuda.synchronize()
    t = time.perf_counter()
    pr.enable()
    if what == "build_cpr":
        B = P.build_cpr(A, cfg)
    else:
        B.device()
        torch.cuda.synchronize()
    pr.disable()
    print(f"== {what} {time.perf_counter() - t:.2f} s")
    pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
