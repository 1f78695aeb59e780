"""Per-plane timeline of the stencil BILU solves (TL variant): cycles spent
in the TMA-slot waits, the neighbouring-plane waits, the arithmetic and the
named barrier, per plane, for one apply at the given grid."""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
import torch
import paper_2201_01970_b200 as P
from paper_2201_01970_b200 import _native as N
from test_stencil import _grid

shape = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "60,220,85").split(","))
F = P.bilu0_factorize(_grid(*shape, seed=0))
dev = F.device()
r = torch.from_numpy(np.random.default_rng(0).standard_normal(3 * F.n)).cuda()
z = torch.empty_like(r)
for _ in range(3):
    dev.apply(r, z)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(20):
    dev.apply(r, z)
ev[1].record()
torch.cuda.synchronize()
print(f"{shape}: apply {ev[0].elapsed_time(ev[1]) / 20 * 1e3:.1f} us (no log)")
log = torch.zeros(2 * 1024 * 8, dtype=torch.int64, device="cuda")
N.lib().cprb_stencil_set_log(N.C.c_void_p(log.data_ptr()))
dev.apply(r, z)
torch.cuda.synchronize()
a = log.cpu().numpy().reshape(2, 1024, 8).astype(np.float64)
nz = shape[2]
for u in (0, 1):
    e = a[u, :nz]
    t0 = e[:, 0].min()
    print("LU"[u], f"span {(e[:, 1].max() - t0) / 1e3:.1f} us; per plane: start/end us, cycles: total, mbar, z, comp, bar")
    for p in list(range(0, 3)) + list(range(7, 10)) + list(range(nz - 3, nz)):
        zz = p if u == 0 else nz - 1 - p
        x = e[zz]
        D = x[5]
        print(f"  plane {zz:3d}: {(x[0]-t0)/1e3:7.1f} {(x[1]-t0)/1e3:7.1f}  tot {x[4]/D:6.0f}/diag  mbar {x[2]/D:5.0f}  z {x[3]/D:5.0f}  comp {x[6]/D:5.0f}  bar {x[7]/D:5.0f}")

if os.environ.get("ALL"):
    for u in (0, 1):
        e = a[u, :nz]
        t0 = e[:, 0].min()
        order = range(nz) if u == 0 else range(nz - 1, -1, -1)
        ends = [(e[z, 1] - t0) / 1e3 for z in order]
        starts = [(e[z, 0] - t0) / 1e3 for z in order]
        print("LU"[u], "end us by processing order:", " ".join(f"{v:.0f}" for v in ends))
        print("LU"[u], "start us:", " ".join(f"{v:.0f}" for v in starts))
        zc = [e[z, 3] / e[z, 5] for z in order]
        print("LU"[u], "z-wait cycles/diag:", " ".join(f"{v:.0f}" for v in zc))

