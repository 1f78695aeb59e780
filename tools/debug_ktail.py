"""Which K-cycle variants agree for a snapshot-colour hierarchy (theta_amg > 0)?"""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2201_01970_b200 as P
from paper_2201_01970_b200 import device as D

(M, _), = P.generate_blackoil_like_sequence(24, 20, 12, 1, 0.01, 4).systems
r = np.random.default_rng(5).standard_normal(M.nrows)
for th in (0.0, 0.25):
    out = {}
    for tag, rows, thr in (("launched", 0, 1024), ("tail512", 100000, 512), ("tail1024", 100000, 1024),
                          ("tail512_300", 300, 512)):
        os.environ["CPRB_KTAIL_ROWS"] = str(rows)
        os.environ["CPRB_KTAIL_THREADS"] = str(thr)
        h = P.build_hierarchy(P.pressure_matrix(M), P.AmgParams(theta_amg=th, cycle="k", krylov="fcg"))
        dev = h.device(1)
        dev.kdesc()
        z = D.empty(M.nrows)
        dev.cycle(D.upload(r), z, "k")
        out[tag] = z.cpu().numpy()
        if tag == "launched":
            zh = D.empty(M.nrows)
            dev.hostcycle(D.upload(r), zh, "k")
            out["host"] = zh.cpu().numpy()
            print("theta", th, "levels", [l.A.nrows for l in h.levels],
                  "colours", [l.partition.c if l.partition else None for l in h.levels],
                  "snap", [int(dl.snapshot.any()) for dl in dev.levels])
    for k, v in out.items():
        print(f"  {k:12s} eq_launched={np.array_equal(v, out['launched'])} "
              f"maxdiff={np.max(np.abs(v - out['launched'])):.3e}")
