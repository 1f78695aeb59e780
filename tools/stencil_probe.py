"""Time the BILU apply of C3 (or --grid) with the stencil plan and the general
wavefront plan; print per-kernel times (CUDA events)."""
import argparse
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2201_01970_b200 as P
from paper_2201_01970_b200.ilu import DeviceBilu

ap = argparse.ArgumentParser()
ap.add_argument("--grid", default="60,220,85")
ap.add_argument("--general", action="store_true")
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
nx, ny, nz = (int(v) for v in a.grid.split(","))
(A, b), = P.generate_blackoil_like_sequence(nx, ny, nz, 1, 0.01, 0).systems
t = time.time()
F = P.bilu0_factorize(A)
print("factorize", round(time.time() - t, 2))
for mode in (["1", "0"] if a.general else ["1"]):
    os.environ["CPRB_STENCIL"] = mode
    t = time.time()
    dev = DeviceBilu(F)
    torch.cuda.synchronize()
    print("plan", mode, "stencil" if dev.stencil else "wave", round(time.time() - t, 2))
    r = torch.from_numpy(np.random.default_rng(0).standard_normal(3 * F.n)).cuda()
    z = torch.empty_like(r)
    for _ in range(3):
        dev.apply(r, z)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        dev.apply(r, z)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / a.reps * 1e3
    nb = F.n
    byt = (F.L.nnz - nb + F.U.nnz - nb) * 76 + nb * 72 + 2 * (nb + 1) * 4 + 4 * 3 * nb * 8
    print(f"bilu apply {us:.1f} us  {byt / us / 1e3:.1f} GB/s")
    if mode == "1":
        z1 = z.clone()
    else:
        print("bitwise equal to stencil:", bool(torch.equal(z, z1)))

if os.environ.get("STENCIL_LOG", "0") == "1":
    import ctypes as C
    from paper_2201_01970_b200 import _native as N
    os.environ["CPRB_STENCIL"] = "1"
    dev = DeviceBilu(F)
    log = torch.zeros(2 * 1024 * 8, dtype=torch.int64, device="cuda")
    N.lib().cprb_stencil_set_log(C.c_void_p(log.data_ptr()))
    dev.apply(r, z)
    torch.cuda.synchronize()
    N.lib().cprb_stencil_set_log(None)
    L = log.cpu().numpy().reshape(2, 1024, 8)
    for u, name in ((0, "L"), (1, "U")):
        e = L[u, :nz]
        t0 = e[:, 0].min()
        order = range(nz) if u == 0 else range(nz - 1, -1, -1)
        print(f"{name}: total {(e[:, 1].max() - t0) / 1e3:.1f} us")
        for zz in list(order)[:3] + list(order)[7:10] + list(order)[-2:]:
            s0, s1, cm, cz, ct, nd, cc, ci = e[zz, :8]
            print(f"  plane {zz:3d}: start {(s0 - t0) / 1e3:7.2f} us end {(s1 - t0) / 1e3:7.2f} us "
                  f"dur {(s1 - s0) / 1e3:6.2f} us  per-step {(s1 - s0) / nd:6.1f} ns  "
                  f"tma-wait {cm / ct * 100:4.1f}%  z-wait {cz / ct * 100:4.1f}%  "
                  f"compute {cc / ct * 100:4.1f}%  segbar {ci / ct * 100:4.1f}%  cyc/step {ct / nd:.0f}")
        st = np.diff(np.sort(e[:, 0]))
        print(f"  start lag per plane: median {np.median(st) / 1e3:.2f} us")
