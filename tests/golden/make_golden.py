"""Generate golden fixtures from the UNMODIFIED reference (cprkit).

Run in the build container only (the reference tree is not present on the GPU
box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--big]

It imports cprkit from /root/reference/pkg/src, runs the reference's own
public functions on seeded inputs and stores small .npz/.json fixtures next
to this file.  Large arrays are stored as SHA-256 digests plus strided
samples.  ``--big`` additionally runs the SPE10-shaped 60x220x85 solve
(about 6 minutes of CPU).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest()


def _import_ref():
    sys.path.insert(0, REF)
    sys.path.insert(0, "/root/reference/pkg/tests")
    import cprkit  # noqa: F401
    return cprkit


def record_history(cpr_mod, A, b, B, params):
    """wrap cprkit.cpr.dot/norm2 (module-level names
    used only by gmres_solve) and replay the Givens recurrence."""
    log = []
    _d, _n = cpr_mod.dot, cpr_mod.norm2
    cpr_mod.dot = lambda x, y: (log.append(_d(x, y)), log[-1])[1]
    cpr_mod.norm2 = lambda x: (log.append(_n(x)), log[-1])[1]
    try:
        res = cpr_mod.gmres_solve(A, b, None, B, params)
    finally:
        cpr_mod.dot, cpr_mod.norm2 = _d, _n
    beta0, p, hist = log[0], 1, []
    m = params.m
    for _ in range(res.outer):
        H = np.zeros((m + 1, m))
        g = np.zeros(m + 1)
        cs = np.zeros(m)
        sn = np.zeros(m)
        g[0] = log[p]
        p += 1
        j = 0
        while True:
            H[:j + 1, j] = log[p:p + j + 1]
            p += j + 1
            H[j + 1, j] = log[p]
            p += 1
            brk = H[j + 1, j] == 0.0
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            d = float(np.hypot(H[j, j], H[j + 1, j]))
            cs[j], sn[j] = (1.0, 0.0) if d == 0.0 else (H[j, j] / d, H[j + 1, j] / d)
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            hist.append(abs(g[j + 1]) / beta0)
            j += 1
            if brk:
                m = j
                break
            if abs(g[j]) < params.tol * beta0 or j == m:
                break
        hist.append(-log[p] / beta0)   # negative marks the explicit residual
        p += 1
    return res, np.array(hist)


def hierarchy_arrays(h, prefix="h"):
    out = {}
    out[f"{prefix}_nlev"] = np.array(len(h.levels))
    out[f"{prefix}_sym"] = np.array(bool(h.symmetric))
    for li, lvl in enumerate(h.levels):
        out[f"{prefix}{li}_ptr"] = lvl.A.row_ptr
        out[f"{prefix}{li}_cols"] = lvl.A.col_idx
        out[f"{prefix}{li}_vals"] = lvl.A.values
        if lvl.aggregates is not None:
            out[f"{prefix}{li}_agg"] = lvl.aggregates
            out[f"{prefix}{li}_perm"] = lvl.partition.perm()
            out[f"{prefix}{li}_gsz"] = np.array([g.shape[0] for g in lvl.partition.groups])
    out[f"{prefix}_lu"] = h.coarsest_lu[0]
    out[f"{prefix}_piv"] = h.coarsest_lu[1]
    return out


def bilu_arrays(F, prefix="f"):
    ls, us = F._l_solve, F._u_solve
    return {
        f"{prefix}_lptr": ls.ptr, f"{prefix}_lcols": ls.cols, f"{prefix}_lvals": ls.vals,
        f"{prefix}_uptr": us.ptr, f"{prefix}_ucols": us.cols, f"{prefix}_uvals": us.vals,
        f"{prefix}_uinv": F.u_diag_inv,
        f"{prefix}_llev": np.concatenate(F.l_schedule.levels),
        f"{prefix}_llevsz": np.array([x.shape[0] for x in F.l_schedule.levels]),
        f"{prefix}_ulev": np.concatenate(F.u_schedule.levels),
        f"{prefix}_ulevsz": np.array([x.shape[0] for x in F.u_schedule.levels]),
    }


def make_small():
    cprkit = _import_ref()
    from cprkit import cpr as cpr_mod
    from cprkit.amg import AmgParams, amg_cycle, build_hierarchy
    from cprkit.coloring import strong_connections, vertices_grouping
    from cprkit.cpr import GmresParams, SolverConfig, ascpr_gmres_sequence, build_cpr
    from cprkit.ilu import bilu0_factorize, bilu_apply
    from cprkit.problems import generate_blackoil_like_sequence, poisson_2d
    from cprkit.smoothers import pgs_scm_sweep
    from cprkit.sparse import spmv
    from conftest import random_block, random_sparse

    # -- generator: C1 and a 3-step drifted sequence ---------------------------
    seq = generate_blackoil_like_sequence(10, 10, 10, 1, 0.01, 0)
    A, b = seq.systems[0]
    np.savez_compressed(OUT / "gen_c1.npz", ptr=A.row_ptr, cols=A.col_idx, vals=A.values, b=b)
    seq3 = generate_blackoil_like_sequence(6, 5, 4, 3, 0.05, 11)
    d = {}
    for k, (Ak, bk) in enumerate(seq3.systems):
        d[f"vals{k}"] = Ak.values
        d[f"b{k}"] = bk
    d["ptr"], d["cols"] = seq3.systems[0][0].row_ptr, seq3.systems[0][0].col_idx
    np.savez_compressed(OUT / "gen_seq3.npz", **d)

    # -- C1 hierarchy / BILU / solve, four configurations ---------------------
    rng = np.random.default_rng(5)
    r_test = rng.standard_normal(3000)
    rp_test = rng.standard_normal(1000)
    summary = {}
    for tag, th_amg, cyc in (("v0", 0.0, "v"), ("k0", 0.0, "k"),
                             ("vd", 0.08, "v"), ("kd", 0.08, "k")):
        cfg = SolverConfig(theta=0.0, theta_amg=th_amg, cycle=cyc)
        B = build_cpr(A, cfg)
        res, hist = record_history(cpr_mod, A, b, B, cfg.gmres_params())
        arrs = hierarchy_arrays(B.pressure_solver)
        arrs.update(bilu_arrays(B.relaxation))
        arrs["x"] = res.x
        arrs["hist"] = hist
        arrs["r_test"] = r_test
        arrs["z_apply"] = B.apply(r_test)
        arrs["rp_test"] = rp_test
        arrs["zp_cycle"] = amg_cycle(B.pressure_solver, rp_test)
        arrs["z_bilu"] = bilu_apply(B.relaxation, r_test)
        np.savez_compressed(OUT / f"c1_{tag}.npz", **arrs)
        summary[tag] = dict(outer=res.outer, inner=res.inner, converged=bool(res.converged),
                            rel=res.rel_residual,
                            sizes=[l.A.nrows for l in B.pressure_solver.levels],
                            colors=[l.partition.c if l.partition else None
                                    for l in B.pressure_solver.levels])

    # -- random smoother / colouring / aggregation cases (conftest generators) --
    rng = np.random.default_rng(20240817)
    cases = {}
    for ci in range(12):
        n = int(rng.integers(5, 300))
        theta = float(rng.choice([0.0, 0.0, 0.05, 0.3]))
        sym = bool(rng.integers(0, 2))
        M = random_sparse(rng, n, avg_nnz=int(rng.integers(3, 9)), symmetric=sym)
        part = vertices_grouping(strong_connections(M, theta))
        bb = rng.standard_normal(n)
        x0 = rng.standard_normal(n)
        from cprkit.amg import pairwise_aggregate
        agg = pairwise_aggregate(M, 0.05)
        cases[f"c{ci}_ptr"] = M.row_ptr
        cases[f"c{ci}_cols"] = M.col_idx
        cases[f"c{ci}_vals"] = M.values
        cases[f"c{ci}_theta"] = np.array(theta)
        cases[f"c{ci}_perm"] = part.perm()
        cases[f"c{ci}_gsz"] = np.array([g.shape[0] for g in part.groups])
        cases[f"c{ci}_b"] = bb
        cases[f"c{ci}_x0"] = x0
        cases[f"c{ci}_sweep"] = pgs_scm_sweep(M, bb, x0, part)
        cases[f"c{ci}_agg"] = agg.aggregate_of
        cases[f"c{ci}_spmv"] = spmv(M, x0)
    cases["ncases"] = np.array(12)
    np.savez_compressed(OUT / "random_scalar.npz", **cases)

    blk = {}
    for ci in range(6):
        n = int(rng.integers(3, 120))
        M = random_block(rng, n, b=3, avg_nnz=int(rng.integers(2, 7)))
        F = bilu0_factorize(M)
        x0 = rng.standard_normal(3 * n)
        blk[f"c{ci}_ptr"] = M.row_ptr
        blk[f"c{ci}_cols"] = M.col_idx
        blk[f"c{ci}_vals"] = M.values
        blk[f"c{ci}_x"] = x0
        blk[f"c{ci}_spmv"] = spmv(M, x0)
        blk[f"c{ci}_bilu"] = bilu_apply(F, x0)
        blk.update(bilu_arrays(F, prefix=f"c{ci}f"))
    blk["ncases"] = np.array(6)
    np.savez_compressed(OUT / "random_block.npz", **blk)

    # -- Poisson 32^2 V(1,1) (test_acceptance.py:190-208) ---------------------
    P = poisson_2d(32, 32)
    h = build_hierarchy(P, AmgParams(coarsest_size=256, cycle="v"))
    bb = np.ones(P.nrows)
    x = np.zeros(P.nrows)
    res_hist = []
    for _ in range(25):
        x = x + amg_cycle(h, bb - spmv(P, x))
        res_hist.append(float(np.linalg.norm(bb - spmv(P, x))))
    summary["poisson32"] = dict(sizes=[l.A.nrows for l in h.levels], res=res_hist)

    # -- pressure-only AMG on 16x16x16 (C2 shape, small), theta_amg = 0 --------
    from cprkit import problems
    from cprkit.cpr import pressure_matrix

    def pressure_op(nx, ny, nz, seed=0):
        r2 = np.random.default_rng(seed)
        nn = nx * ny * nz
        links = problems._neighbor_links(nx, ny, nz)
        logk = r2.normal(0.0, 1.0, nn)
        conv = r2.uniform(0.2, 0.5, nn)
        cpl = r2.standard_normal((nn, 6)) * 0.5
        return pressure_matrix(problems._assemble_step(nn, links, np.array([1.0, 1.0, 0.2]),
                                                       np.exp(logk), conv, cpl, 0.0))

    Pp = pressure_op(16, 16, 16)
    h = build_hierarchy(Pp, AmgParams(theta_amg=0.0, cycle="v"))
    bb = np.ones(Pp.nrows)
    x = np.zeros(Pp.nrows)
    cyc = []
    for _ in range(6):
        x = x + amg_cycle(h, bb - spmv(Pp, x))
        cyc.append(float(np.linalg.norm(bb - spmv(Pp, x)) / np.linalg.norm(bb)))
    summary["press16"] = dict(sizes=[l.A.nrows for l in h.levels],
                              nnz=[l.A.nnz for l in h.levels],
                              colors=[l.partition.c if l.partition else None for l in h.levels],
                              rel=cyc,
                              digests=[digest(l.aggregates) if l.aggregates is not None else None
                                       for l in h.levels],
                              perm_digests=[digest(l.partition.perm()) if l.partition else None
                                            for l in h.levels],
                              vals_digests=[digest(l.A.values) for l in h.levels])

    # -- acceptance sequence (test_output.txt:203): 32x32x4x10, mu=15 ---------
    t0 = time.time()
    seqa = generate_blackoil_like_sequence(32, 32, 4, 10, 0.01, seed=20240817)
    cfga = SolverConfig(theta=0.0, mu=15, m=28, tol=1e-5, cycle="v", coarsest_size=200)
    outa = ascpr_gmres_sequence(seqa.systems, 15, cfga)
    summary["accept_seq"] = dict(total_inner=outa.total_inner, setup_calls=outa.setup_calls,
                                 inner=[r.inner for r in outa.records],
                                 outer=[r.outer for r in outa.records],
                                 rel=[r.rel_residual for r in outa.records],
                                 rebuilt=[r.rebuilt for r in outa.records],
                                 seconds=time.time() - t0)
    (OUT / "summary.json").write_text(json.dumps(summary, indent=1) + "\n")


def make_big_k():
    """SPE10-shaped 60x220x85 (C3), theta_amg = 0, K-cycle (the reference's
    default cycle, src/cpr.py:72): iteration counts, the Givens history of both
    restarts and solution samples (about 12 minutes of CPU)."""
    _import_ref()
    from cprkit import cpr as cpr_mod
    from cprkit.cpr import SolverConfig, build_cpr
    from cprkit.problems import generate_blackoil_like_sequence
    t0 = time.time()
    seq = generate_blackoil_like_sequence(60, 220, 85, 1, 0.01, 0)
    A, b = seq.systems[0]
    tg = time.time() - t0
    cfg = SolverConfig(theta=0.0, theta_amg=0.0, cycle="k")
    t0 = time.time()
    B = build_cpr(A, cfg)
    ts = time.time() - t0
    t0 = time.time()
    res, hist = record_history(cpr_mod, A, b, B, cfg.gmres_params())
    tsol = time.time() - t0
    out = dict(outer=res.outer, inner=res.inner, rel=res.rel_residual, hist=hist.tolist(),
               x_norm=float(np.linalg.norm(res.x)), x_sample_stride=97,
               x_sample=res.x[::97].tolist(), b_digest=digest(b),
               seconds=dict(generate=tg, setup=ts, solve=tsol))
    (OUT / "c3_k0.json").write_text(json.dumps(out) + "\n")


def make_big():
    """SPE10-shaped 60x220x85 (C3), theta_amg = 0, V-cycle: iteration counts,
    Givens history, solution samples, hierarchy digests."""
    _import_ref()
    from cprkit import cpr as cpr_mod
    from cprkit.cpr import SolverConfig, build_cpr
    from cprkit.problems import generate_blackoil_like_sequence
    t0 = time.time()
    seq = generate_blackoil_like_sequence(60, 220, 85, 1, 0.01, 0)
    A, b = seq.systems[0]
    tg = time.time() - t0
    cfg = SolverConfig(theta=0.0, theta_amg=0.0, cycle="v")
    t0 = time.time()
    B = build_cpr(A, cfg)
    ts = time.time() - t0
    t0 = time.time()
    res, hist = record_history(cpr_mod, A, b, B, cfg.gmres_params())
    tsol = time.time() - t0
    h = B.pressure_solver
    out = dict(
        outer=res.outer, inner=res.inner, rel=res.rel_residual, hist=hist.tolist(),
        x_norm=float(np.linalg.norm(res.x)), x_sample_stride=97,
        x_sample=res.x[::97].tolist(),
        b_digest=digest(b), vals_digest=digest(A.values),
        sizes=[l.A.nrows for l in h.levels], nnz=[l.A.nnz for l in h.levels],
        colors=[l.partition.c if l.partition else None for l in h.levels],
        agg_digests=[digest(l.aggregates) if l.aggregates is not None else None for l in h.levels],
        perm_digests=[digest(l.partition.perm()) if l.partition else None for l in h.levels],
        lvl_vals_digests=[digest(l.A.values) for l in h.levels],
        lvl_cols_digests=[digest(l.A.col_idx) for l in h.levels],
        bilu_llev=len(B.relaxation.l_schedule.levels),
        bilu_ulev=len(B.relaxation.u_schedule.levels),
        seconds=dict(generate=tg, setup=ts, solve=tsol),
    )
    (OUT / "c3_v0.json").write_text(json.dumps(out) + "\n")


def make_c4_mix():
    """Config 4 with a reuse/rebuild MIX (src/cpr.py:204-212, :349-382): ten
    SPE10-shaped (C3 grid) Newton systems with drift 0.05 and mu = 5, where
    the aging preconditioner crosses mu and forces rebuilds mid-sequence
    (about 30 minutes of CPU)."""
    _import_ref()
    from cprkit.cpr import SolverConfig, ascpr_gmres_sequence
    from cprkit.problems import generate_blackoil_like_sequence
    t0 = time.time()
    seq = generate_blackoil_like_sequence(60, 220, 85, 10, 0.05, 0)
    tg = time.time() - t0
    cfg = SolverConfig(theta=0.0, theta_amg=0.0, cycle="v")
    t0 = time.time()
    out = ascpr_gmres_sequence(seq.systems, 5, cfg, keep_solutions=True)
    tsol = time.time() - t0
    rec = dict(grid=[60, 220, 85], nsteps=10, drift=0.05, seed=0, mu=5,
               setup_calls=out.setup_calls, rebuilt=[bool(r.rebuilt) for r in out.records],
               its=[[r.outer, r.inner] for r in out.records],
               rel=[r.rel_residual for r in out.records],
               x_norm=[float(np.linalg.norm(r.x)) for r in out.records],
               x_sample_stride=997, x_sample=[r.x[::997].tolist() for r in out.records],
               b_digests=[digest(b) for _, b in seq.systems],
               seconds=dict(generate=tg, sequence=tsol, setup=out.setup_time, solve=out.solve_time))
    (OUT / "c4_mix.json").write_text(json.dumps(rec) + "\n")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--bigk", action="store_true")
    ap.add_argument("--c4mix", action="store_true")
    ap.add_argument("--skip-small", action="store_true")
    a = ap.parse_args()
    if not a.skip_small:
        make_small()
    if a.big:
        make_big()
    if a.bigk:
        make_big_k()
    if a.c4mix:
        make_c4_mix()
