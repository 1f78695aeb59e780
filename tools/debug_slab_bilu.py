"""Sequential (one rank at a time) run of the slab-partitioned BILU solves:
checks that every mirror slot a rank polls was filled by its neighbour."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_01970_b200 as P  # noqa: E402
from paper_2201_01970_b200 import _native as N  # noqa: E402
from paper_2201_01970_b200 import device as D  # noqa: E402
from paper_2201_01970_b200.partition import SlabBilu, SlabMatrix, SlabPartition  # noqa: E402

SENT = 0x7FF4C0FFEE5EED01
(A, _), = P.generate_blackoil_like_sequence(12, 10, 14, 1, 0.01, 0).systems
F = P.bilu0_factorize(A)
nr = 2
part = SlabPartition(A.nrows, nr, 60)
rng = np.random.default_rng(7)
r = rng.standard_normal(3 * A.nrows)
zp = rng.standard_normal(A.nrows)
ranks, mats = [], []
for q in range(nr):
    ranks.append(SlabBilu(F, part, q, plan=ranks[0].plan if ranks else None))
    mats.append(SlabMatrix(A, part, q))
for q in range(nr):
    if q + 1 < nr:
        ranks[q].peer_l = D.ptr(ranks[q + 1].zl_step)
    if q > 0:
        ranks[q].peer_u = D.ptr(ranks[q - 1].y_step)
lib = N.lib()
st = D.stream()
zps = [D.upload(zp[m.w0:m.w1].copy()) for m in mats]
rs = [D.upload(r[3 * m.c0:3 * m.c1].copy()) for m in mats]
for q in range(nr):
    sb, m = ranks[q], mats[q]
    N.check(lib.cprb_stage2_residual_steps(m.desc_ref(), C.byref(sb.desc), sb.c0, D.ptr(zps[q]),
                                           D.ptr(rs[q]), D.ptr(sb.rhs_l), D.ptr(sb.zl_step),
                                           D.ptr(sb.y_step), st))
torch.cuda.synchronize()


def sentinels(t, idx, b):
    a = t.cpu().numpy().view(np.uint64)
    s = np.concatenate([idx + c for c in range(b)]) if idx.size else idx
    return int((a[s] == SENT).sum()), int(s.size)


hl, hu = ranks[0].plan["hl"], ranks[0].plan["hu"]
print("L chunk ranges", hl["chunk_range"].tolist(), "U", hu["chunk_range"].tolist())
print("L mirror r1 before", sentinels(ranks[1].zl_step, hl["mirror"][1], 3))
sb = ranks[0]
N.check(lib.cprb_wave_solve_part(C.byref(sb.desc), 0, sb.lr[0], sb.lr[1] - sb.lr[0], D.ptr(sb.rhs_l),
                                 D.ptr(sb.zl_step), sb.peer_l or None, D.ptr(sb.tickets), st))
torch.cuda.synchronize()
print("rank0 L done; L mirror r1 after", sentinels(ranks[1].zl_step, hl["mirror"][1], 3))
# which polled slots of rank 1 are still sentinel?
sb = ranks[1]
N.check(lib.cprb_wave_solve_part(C.byref(sb.desc), 0, sb.lr[0], sb.lr[1] - sb.lr[0], D.ptr(sb.rhs_l),
                                 D.ptr(sb.zl_step), None, D.ptr(sb.tickets), st))
torch.cuda.synchronize()
print("rank1 L done")
for q in range(nr):
    sb, m = ranks[q], mats[q]
    N.check(lib.cprb_l_to_u_rows(C.byref(sb.desc), sb.c0, m.n_own, D.ptr(sb.zl_step), D.ptr(sb.rhs_u), st))
sb = ranks[1]
N.check(lib.cprb_wave_solve_part(C.byref(sb.desc), 1, sb.ur[0], sb.ur[1] - sb.ur[0], D.ptr(sb.rhs_u),
                                 D.ptr(sb.y_step), sb.peer_u or None, D.ptr(sb.tickets) + 4, st))
torch.cuda.synchronize()
print("rank1 U done; U mirror r0 after", sentinels(ranks[0].y_step, hu["mirror"][0], 3))
sb = ranks[0]
N.check(lib.cprb_wave_solve_part(C.byref(sb.desc), 1, sb.ur[0], sb.ur[1] - sb.ur[0], D.ptr(sb.rhs_u),
                                 D.ptr(sb.y_step), None, D.ptr(sb.tickets) + 4, st))
torch.cuda.synchronize()
print("rank0 U done")

