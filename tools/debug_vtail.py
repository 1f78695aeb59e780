"""Run one V-cycle with the persistent tail on C1 (compute-sanitizer target)."""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2201_01970_b200 as P

g = np.load(Path(__file__).resolve().parents[1] / "tests/golden/gen_c1.npz")
A = P.BlockCsrMatrix(3, 1000, 1000, g["ptr"], g["cols"], g["vals"])
cfg = P.SolverConfig(theta=0.0, theta_amg=0.0, cycle="v")
h = P.build_hierarchy(P.pressure_matrix(A), cfg.amg_params())
print("levels", [l.A.nrows for l in h.levels], "colours", [l.partition.c if l.partition else None for l in h.levels])
d = h.device().desc
print("tail_start", d.tail_start, "phases", d.tail_nphases, "chunks", d.tail_nchunks, "slot", d.tail_slot,
      "smem", d.tail_smem, "veclen", d.tail_vec_len, flush=True)
r = np.random.default_rng(11).standard_normal(A.nrows)
z = P.amg_cycle(h, r)
print("ok", float(np.linalg.norm(z)))
