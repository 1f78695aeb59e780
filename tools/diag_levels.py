"""Per-level timing of the V-cycle pieces with CUDA events (warm caches)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_01970_b200 as P  # noqa: E402
from paper_2201_01970_b200 import _native as N  # noqa: E402
from paper_2201_01970_b200 import device as D  # noqa: E402


def tm(fn, reps=50):
    st = torch.cuda.current_stream()
    fn(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


grid = tuple(map(int, (sys.argv[1] if len(sys.argv) > 1 else "60,220,85").split(",")))
(A, b), = P.generate_blackoil_like_sequence(*grid, 1, 0.01, 0).systems
B = P.build_cpr(A, P.SolverConfig(theta=0.0, theta_amg=0.0, cycle="v"))
Bd = B.device()
lib = N.lib()
x1 = torch.zeros(1, device="cuda")
print(f"torch tiny op: {tm(lambda: x1.add_(1.0), 1000):.2f} us/launch")
amg = Bd.amg
for l, dl in enumerate(amg.levels):
    n = dl.split.n
    bvec = torch.rand(n, dtype=torch.float64, device="cuda")
    xvec = torch.zeros(n, dtype=torch.float64, device="cuda")
    f = tm(lambda: lib.cprb_pgs_scm_pass(C.byref(dl.desc), D.ptr(bvec), D.ptr(xvec), 0, 1, D.stream()))
    bk = tm(lambda: lib.cprb_pgs_scm_pass(C.byref(dl.desc), D.ptr(bvec), D.ptr(xvec), 1, 0, D.stream()))
    nc = amg.h.levels[l + 1].A.nrows
    bc = torch.empty(nc, dtype=torch.float64, device="cuda")
    rr = tm(lambda: lib.cprb_resid_restrict(C.byref(dl.desc), D.ptr(bvec), D.ptr(xvec), D.ptr(bc), D.stream()))
    pr = tm(lambda: lib.cprb_prolong(C.byref(dl.desc), D.ptr(bc), D.ptr(xvec), D.stream()))
    print(f"level {l:2d} n={n:8d} colors={dl.split.ncolors:2d}  fwd(zg) {f:8.1f} us ({f/dl.split.ncolors:5.1f}/color)"
          f"  bwd {bk:8.1f} us  resid+restrict {rr:7.1f}  prolong {pr:6.1f}")
r = torch.from_numpy(b).cuda()
zp = torch.empty(A.nrows, dtype=torch.float64, device="cuda")
print(f"vcycle direct: {tm(lambda: amg.vcycle(r, zp), 20):.1f} us")
print(f"vcycle graph : {tm(lambda: lib.cprb_amg_cycle_graph(Bd.graphs, C.byref(amg.desc), D.ptr(r), D.ptr(zp), D.stream()), 20):.1f} us")
z = torch.empty_like(r)
print(f"bilu wave    : {tm(lambda: Bd.bilu.apply(r, z), 20):.1f} us")
F = B.relaxation
dv = F.device(use_wave=False)
print(f"bilu sync-free level kernel: {tm(lambda: dv.apply(r, z), 10):.1f} us")
