"""Time the C3 V-cycle graph, the CPR application and the full solve on the
current library (CPRB_LIB selects a variant); save the cycle output so
variants can be compared bitwise."""
import ctypes as C
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_2201_01970_b200 as P
from paper_2201_01970_b200 import _native as N
from paper_2201_01970_b200 import device as D

tag = sys.argv[1]
(A, b), = P.generate_blackoil_like_sequence(60, 220, 85, 1, 0.01, 0).systems
cfg = P.SolverConfig(theta=0.0, theta_amg=0.0, cycle="v")
B = P.build_cpr(A, cfg)
Bd = B.device()
lib = N.lib()
bd = torch.from_numpy(b).cuda()
zp = D.empty(Bd.amg.levels[0].n if hasattr(Bd.amg.levels[0], "n") else A.nrows)
zp = D.empty(A.nrows)
z = D.empty(3 * A.nrows)


def ev_time(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


vc = lambda: N.check(lib.cprb_amg_cycle_graph(Bd.graphs, C.byref(Bd.amg.desc), D.ptr(bd), D.ptr(zp), D.stream()))  # noqa: E731
t_vc = ev_time(vc)
t_ap = ev_time(lambda: Bd.apply(bd, z))
params = cfg.gmres_params()
t_so = ev_time(lambda: P.gmres_solve(A, bd, None, B, params), reps=5)
vc()
torch.cuda.synchronize()
np.save(f"gpurun_out/vc_{tag}.npy", zp.cpu().numpy())
res = P.gmres_solve(A, bd, None, B, params)
print(f"{tag}: vcycle {t_vc:.1f} us  cpr_apply {t_ap:.1f} us  solve {t_so / 1e3:.3f} ms  "
      f"iters {res.outer}/{res.inner} rel {res.rel_residual:.6e}", flush=True)
