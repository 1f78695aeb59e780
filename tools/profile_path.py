"""Run pieces of the CPR-GMRES path on the C3 system for profiling under ncu.

    python tools/profile_path.py [--what apply|spmv|bilu|vcycle|solve] [--reps N] [--grid 60,220,85]
"""
import argparse
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
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
        "finish": lambda: N.check(N.lib().cprb_cpr_finish(C.byref(Bd.desc), D.ptr(bd), D.ptr(z),
                                                          D.stream())),
        "applynog": lambda: N.check(N.lib().cprb_cpr_apply(C.byref(Bd.desc), D.ptr(bd), D.ptr(z),
                                                           D.stream())),
        "vcycleg": lambda: N.check(N.lib().cprb_amg_cycle_graph(Bd.graphs, C.byref(Bd.amg.desc),
                                                                D.ptr(bd), D.ptr(zp), D.stream())),
        "solve": lambda: P.gmres_solve(A, bd, None, B, cfg.gmres_params()),
    }
    import ctypes as C
    from paper_2201_01970_b200 import _native as N
    if a.what == "vtailtl":
        t = torch
        log = t.zeros(4096, dtype=t.int64, device="cuda")
        N.lib().cprb_vtail_set_log(D.ptr(log))
        for rep in range(3):
            log.zero_()
            N.check(N.lib().cprb_amg_cycle(C.byref(Bd.amg.desc), D.ptr(bd), D.ptr(zp), D.stream()))
            t.cuda.synchronize()
        N.lib().cprb_vtail_set_log(None)
        d = Bd.amg.desc
        L = log.cpu().numpy()[:2 + d.tail_nphases]
        ph = Bd.amg.tail_phase_host
        print("tail_start", d.tail_start, "phases", d.tail_nphases, "chunks", d.tail_nchunks,
              "slot", d.tail_slot, "stream bytes", Bd.amg.tail_bytes)
        print(f"pdl wait {(L[1] - L[0]) / 1e3:.2f} us, total after wait {(L[-1] - L[1]) / 1e3:.2f} us")
        prev = L[1]
        for i in range(d.tail_nphases):
            print(f"  {i:3d} {tuple(int(v) for v in ph[i])} {(L[2 + i] - prev) / 1e3:7.2f} us")
            prev = L[2 + i]
        C3 = log.cpu().numpy()[2 + d.tail_nphases:2 + d.tail_nphases + 3 * d.tail_nchunks].reshape(-1, 3)
        if C3[:, 0].all():
            w = (C3[:, 1] - C3[:, 0]) / 1e3
            cpt = (C3[:, 2] - C3[:, 1]) / 1e3
            gap = (C3[1:, 0] - C3[:-1, 2]) / 1e3
            print(f"chunks: wait total {w.sum():.1f} us, compute total {cpt.sum():.1f} us, "
                  f"between-chunk (arrive/barrier/loop) total {gap.sum():.1f} us")
            for c in range(min(40, len(w))):
                print(f"   chunk {c:3d} wait {w[c]:6.2f} compute {cpt[c]:6.2f}")
        return
    if a.what == "amgtl":
        t = torch
        log = t.zeros(4 * 4096, dtype=t.int64, device="cuda")
        for rep in range(4):
            log.zero_()
            N.lib().cprb_amg_set_log(D.ptr(log))
            if a.nograph:
                Bd.amg.vcycle(bd, zp)
            else:
                N.check(N.lib().cprb_amg_cycle_graph(Bd.graphs, C.byref(Bd.amg.desc), D.ptr(bd),
                                                     D.ptr(zp), D.stream()))
            t.cuda.synchronize()
        N.lib().cprb_amg_set_log(None)
        L = log.cpu().numpy().reshape(-1, 4)
        L = L[L[:, 1] > 0]
        L = L[np.argsort(L[:, 1])]
        t0 = L[0, 1]
        names = {1: "sweep", 2: "sweepZG", 3: "rr", 4: "prol"}
        tot = (L[-1, 3] - t0) / 1e3
        print("launches", len(L), "span us", tot)
        if os.environ.get("AMGTL_OUT"):
            np.save(os.environ["AMGTL_OUT"], L)
        gaps = (L[1:, 1] - L[:-1, 3]) / 1e3
        waits = (L[:, 2] - L[:, 1]) / 1e3
        work = (L[:, 3] - L[:, 2]) / 1e3
        print("median: start-gap(prev end->start)", np.median(gaps), "wait", np.median(waits), "work", np.median(work))
        for i in range(0, len(L)):
            if i < 60 or i % 20 == 0:
                print(f"{i:4d} {names.get(int(L[i,0]),'?'):8s} start {(L[i,1]-t0)/1e3:8.2f} wait {(L[i,2]-L[i,1])/1e3:6.2f} work {(L[i,3]-L[i,2])/1e3:6.2f}")
        return
    if a.what == "wavetl":
        t = torch
        log = t.zeros(2 * 256 * 512, dtype=t.int64, device="cuda")
        N.lib().cprb_wave_set_log(D.ptr(log))
        for rep in range(3):
            log.zero_()
            Bd.bilu.apply(bd, z)
            t.cuda.synchronize()
        N.lib().cprb_wave_set_log(None)
        L = log.cpu().numpy().reshape(2, 256, 512)
        t0 = L[L > 0].min()
        for u in range(2):
            nch = int((L[u, :200, 0] > 0).sum())
            print(("U" if u else "L"), "chunks", nch)
            for c in list(range(min(nch, 4))) + [nch // 2, nch - 1]:
                row = L[u, c]
                row = row[row > 0]
                d = np.diff(row)
                print(f" chunk {c}: start {(row[0]-t0)/1e3:.1f} end {(row[-1]-t0)/1e3:.1f} us, steps {row.size},"
                      f" median step {np.median(d)/1e3:.3f} us, max step {d.max()/1e3:.2f}")
            F = L[u, 200:205, :128].astype(np.float64) / 280.0   # chunk 0 (c % 4 == 0 slot), cycles/step
            nm = ["wait_full", "prefetch_next", "row(loads+spin+fp)", "publish+stores", "syncwarp+arrive"]
            iss = 0 * L[u, 206, :279].astype(np.float64)
            got = L[u, 207, :279].astype(np.float64)
            pw = L[u, 208, :279].astype(np.float64)
            if iss[5] > 0:
                lat = got - iss
                print("  TMA issue->landed-seen (cycles) median", np.median(lat[4:]), "p90", np.percentile(lat[4:], 90),
                      "| producer wait on empty median", np.median(pw[4:]),
                      "| issue interval median", np.median(np.diff(iss[4:])))
            print("  cycles/step tid0:", {nm[q]: round(F[q, 0]) for q in range(5)})
            print("  cycles/step mean over threads:", {nm[q]: round(F[q].mean()) for q in range(5)})
            # lag between consecutive chunks at equal local step 100
            lag = [(L[u, c, 100] - L[u, c - 1, 100]) / 1e3 for c in range(1, nch) if L[u, c, 100] > 0]
            print(" lag@step100 median", np.median(lag), "first", lag[:5])
        return
    if a.what in ("vcyclecold", "bilucold"):
        t = torch
        flush = t.empty(64 * 1024 * 1024, dtype=t.float64, device="cuda")   # 512 MB > L2
        g = ops["vcycleg"] if a.what == "vcyclecold" else ops["bilu"]
        e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
        tot = 0.0
        for rep in range(a.reps + 2):
            flush.fill_(1.0)
            e0.record()
            g()
            e1.record()
            t.cuda.synchronize()
            if rep >= 2:
                tot += e0.elapsed_time(e1)
        print(f"{a.what}: {tot / a.reps:.3f} ms/rep (device, L2 flushed before each rep)")
        return
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
