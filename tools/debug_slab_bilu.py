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

# ---- concurrency probe: rank 1's L (needs rank 0) first, then rank 0's L
import time  # noqa: E402
for q in range(nr):
    sb, m = ranks[q], mats[q]
    N.check(lib.cprb_stage2_residual_steps(m.desc_ref(), C.byref(sb.desc), sb.c0, D.ptr(zps[q]),
                                           D.ptr(rs[q]), D.ptr(sb.rhs_l), D.ptr(sb.zl_step),
                                           D.ptr(sb.y_step), st))
for q in range(nr):
    ranks[q].rearm(st)
torch.cuda.synchronize()
s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
print("L mirror r1 armed", sentinels(ranks[1].zl_step, hl["mirror"][1], 3), flush=True)
sb = ranks[1]
N.check(lib.cprb_wave_solve_part(C.byref(sb.desc), 0, sb.lr[0], sb.lr[1] - sb.lr[0], D.ptr(sb.rhs_l),
                                 D.ptr(sb.zl_step), None, D.ptr(sb.tickets), s1.cuda_stream))
time.sleep(0.5)
print("after 0.5 s: s1 done?", s1.query(), flush=True)
sb = ranks[0]
N.check(lib.cprb_wave_solve_part(C.byref(sb.desc), 0, sb.lr[0], sb.lr[1] - sb.lr[0], D.ptr(sb.rhs_l),
                                 D.ptr(sb.zl_step), sb.peer_l or None, D.ptr(sb.tickets), s0.cuda_stream))
t0 = time.time()
while time.time() - t0 < 5 and not (s0.query() and s1.query()):
    time.sleep(0.2)
print("s0 done", s0.query(), "s1 done", s1.query(), flush=True)

# ---- full concurrent pipeline with per-stage events
for q in range(nr):
    sb, m = ranks[q], mats[q]
    N.check(lib.cprb_stage2_residual_steps(m.desc_ref(), C.byref(sb.desc), sb.c0, D.ptr(zps[q]),
                                           D.ptr(rs[q]), D.ptr(sb.rhs_l), D.ptr(sb.zl_step),
                                           D.ptr(sb.y_step), st))
for q in range(nr):
    ranks[q].rearm(st)
torch.cuda.synchronize()
streams = [torch.cuda.Stream() for _ in range(nr)]
ev = {}
zs = [D.zeros(3 * m.n_own) for m in mats]
for q in range(nr):
    sb, m = ranks[q], mats[q]
    s_ = streams[q].cuda_stream
    d = C.byref(sb.desc)
    N.check(lib.cprb_wave_solve_part(d, 0, sb.lr[0], sb.lr[1] - sb.lr[0], D.ptr(sb.rhs_l),
                                     D.ptr(sb.zl_step), sb.peer_l or None, D.ptr(sb.tickets), s_))
    e = torch.cuda.Event(); e.record(streams[q]); ev[(q, "L")] = e
    N.check(lib.cprb_l_to_u_rows(d, sb.c0, m.n_own, D.ptr(sb.zl_step), D.ptr(sb.rhs_u), s_))
    e = torch.cuda.Event(); e.record(streams[q]); ev[(q, "l2u")] = e
    N.check(lib.cprb_wave_solve_part(d, 1, sb.ur[0], sb.ur[1] - sb.ur[0], D.ptr(sb.rhs_u),
                                     D.ptr(sb.y_step), sb.peer_u or None, D.ptr(sb.tickets) + 4, s_))
    e = torch.cuda.Event(); e.record(streams[q]); ev[(q, "U")] = e
t0 = time.time()
while time.time() - t0 < 5 and not all(e.query() for e in ev.values()):
    time.sleep(0.2)
print({f"{k[0]}{k[1]}": e.query() for k, e in ev.items()}, flush=True)

# ---- bisect: full solve_steps per rank (L, l2u, U, combine, rearm)
for variant in ("combine", "solve_steps"):
    for q in range(nr):
        sb, m = ranks[q], mats[q]
        N.check(lib.cprb_stage2_residual_steps(m.desc_ref(), C.byref(sb.desc), sb.c0, D.ptr(zps[q]),
                                               D.ptr(rs[q]), D.ptr(sb.rhs_l), D.ptr(sb.zl_step),
                                               D.ptr(sb.y_step), st))
    for q in range(nr):
        ranks[q].rearm(st)
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(nr)]
    evs = []
    for q in range(nr):
        sb, m = ranks[q], mats[q]
        s_ = streams[q].cuda_stream
        zp_own = D.ptr(zps[q]) + (m.c0 - m.w0) * 8
        if variant == "solve_steps":
            sb.solve_steps(zs[q], zp_own, m.n_own, st=s_)
        else:
            d = C.byref(sb.desc)
            N.check(lib.cprb_wave_solve_part(d, 0, sb.lr[0], sb.lr[1] - sb.lr[0], D.ptr(sb.rhs_l),
                                             D.ptr(sb.zl_step), sb.peer_l or None, D.ptr(sb.tickets), s_))
            N.check(lib.cprb_l_to_u_rows(d, sb.c0, m.n_own, D.ptr(sb.zl_step), D.ptr(sb.rhs_u), s_))
            N.check(lib.cprb_wave_solve_part(d, 1, sb.ur[0], sb.ur[1] - sb.ur[0], D.ptr(sb.rhs_u),
                                             D.ptr(sb.y_step), sb.peer_u or None, D.ptr(sb.tickets) + 4, s_))
            N.check(lib.cprb_wave_combine_rows(d, sb.c0, m.n_own, D.ptr(sb.y_step), zp_own, D.ptr(zs[q]), s_))
        e = torch.cuda.Event(); e.record(streams[q]); evs.append(e)
    t0 = time.time()
    while time.time() - t0 < 5 and not all(e.query() for e in evs):
        time.sleep(0.2)
    print(variant, [e.query() for e in evs], flush=True)
    if not all(e.query() for e in evs):
        break
