"""CPR-GMRES SOLVE benchmark (BASELINE.json metric) on the SPE10-shaped system.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--grid 60,220,85] [--cycle v|k]

One step = one complete CPR-GMRES solve (build_cpr done beforehand, as the
reference times SETUP and SOLVE separately, src/cpr.py:369-376) of the
synthetic 60x220x85 three-phase black-oil Jacobian (3,366,000 DOF, 3x3 BSR,
seed 0, drift 0.01) with SolverConfig(theta=0, theta_amg=0, cycle='v').
`value` is the device time-to-solution in ms (inputs resident in HBM; the
working set, > 1 GB, exceeds the 126 MB L2 so no flush is needed).  `e2e`
is the same solve through the public API from pinned host buffers.
`--impl reference` times complete solves of the CPU oracle
(oracle/cprkit_oracle.py, a numpy restatement of the reference) on the host
cores, with the same config dict.  `--gpus N` (N > 1) relaunches itself as N
torchrun ranks when WORLD_SIZE is unset; at N > 1 the default is ONE system
row-partitioned over the N GPUs (strong scaling: NCCL halos, GPU-count-
invariant reductions, the BILU wavefront over peer memory; DESIGN.md
section 7) plus a config-5 (26.9M DOF) sub-record; `--replicas` solves N
independent systems instead (weak scaling, no data-path collective).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "CPR-GMRES solve time & iters, SPE10-shape 3.28M DOF; smoother/SpMV HBM GB/s"


def _peaks():
    """HBM roofline denominator: the driver-measured copy bandwidth when
    MEASURED_PEAKS.json is present, else the profiling guide's fallback."""
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            v = float(json.loads(p.read_text())["hbm_gbs"])
            if v > 0:
                return v, "measured"
        except (ValueError, KeyError, TypeError):
            pass
    return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler for the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", os.environ.get("CPRB_SMI_MS", "20")],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self, start: bool):
        """Bracket the timed region (samples outside it are not reported)."""
        if start:
            self.t0 = time.time()
        else:
            self.t1 = time.time()
            time.sleep(0.05)        # let the sample covering the end arrive

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0, t1 = getattr(self, "t0", None), getattr(self, "t1", None)
        lines = [ln for t, ln in self.lines
                 if t0 is None or t1 is None or (t0 <= t <= t1 + 0.025)]
        for ln in lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)),
                "reasons": sorted(reasons), "samples": len(sm)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def max_over_ranks(value: float, dist, torch, device: str) -> float:
    """Whole-job time of a step = the slowest rank's (the contract's max over
    ranks); collective on any backend (NCCL on the GPU box, gloo in tests)."""
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.barrier()
    return float(t.item())


def _config_name(grid) -> str:
    return {(60, 220, 85): "config 3", (120, 440, 170): "config 5 on one GPU",
            (10, 10, 10): "config 1"}.get(tuple(grid), "custom grid")


def _config(grid, cycle, ws, dof, nnzb, levels):
    """The `config` dict of BOTH arms (identical for the same --gpus/--grid/--cycle)."""
    nx, ny, nz = grid
    return {"workload": f"SPE10-shaped {nx}x{ny}x{nz} three-phase BSR3 CPR-GMRES solve "
                        f"({_config_name(grid)}), SolverConfig(theta=0, theta_amg=0, cycle='{cycle}')",
            "dof": int(dof), "nnz_blocks": int(nnzb), "levels": int(levels),
            "parallelism": (f"one system row-partitioned into {ws} z-slabs, one GPU each (NCCL halos, "
                            "GPU-count-invariant reductions, global BILU wavefront over peer memory)")
            if ws > 1 else "single-gpu",
            "l2": "working set > 1 GB exceeds the 126 MB L2 (no flush between solves); per-kernel "
                  "figures flush the L2 before every launch"}


def _grid(s):
    return tuple(int(v) for v in s.split(","))


def _bytes_spmv(nb, nnzb):
    return nnzb * (72 + 4) + (nb + 1) * 4 + 2 * (3 * nb) * 8


def _bytes_sweep(n, nnz):
    return (nnz - n) * 12 + n * 36


def _bytes_bilu(nb, n_off_l, n_off_u):
    return (n_off_l + n_off_u) * 76 + nb * 72 + 2 * (nb + 1) * 4 + 4 * 3 * nb * 8


def _time_op(fn, reps, torch):
    st = torch.cuda.current_stream()
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3   # microseconds


def _time_cold(fn, reps, torch, flush):
    """Per-launch device time with the L2 flushed before every launch (a
    write of a buffer larger than the 126 MB L2 between launches, outside the
    events): the median over `reps` of cold single launches, microseconds."""
    st = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(reps)]
    for e0, e1 in ev:
        flush.fill_(1.0)
        e0.record(st)
        fn()
        e1.record(st)
    torch.cuda.synchronize()
    return float(np.median([e0.elapsed_time(e1) for e0, e1 in ev])) * 1e3


def run_ours(args):
    import ctypes as C

    import torch
    import torch.distributed as dist

    import paper_2201_01970_b200 as P
    from paper_2201_01970_b200 import _native as N
    from paper_2201_01970_b200 import device as D

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    nx, ny, nz = args.grid
    t0 = time.perf_counter()
    # N > 1: weak scaling over independent units -- rank r solves its own
    # system (generator seed r; rank 0 is the reference's seed-0 system)
    (A, b), = P.generate_blackoil_like_sequence(nx, ny, nz, 1, 0.01, rank).systems
    t_gen = time.perf_counter() - t0
    cfg = P.SolverConfig(theta=0.0, theta_amg=0.0, cycle=args.cycle)
    t0 = time.perf_counter()
    B = P.build_cpr(A, cfg)
    Bd = B.device()
    M = D.device_matrix(A)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    n = b.shape[0]
    bd = torch.from_numpy(b).cuda()
    params = cfg.gmres_params()
    lib = N.lib()
    launches = {"n": 0}

    def solve():
        return P.gmres_solve(A, bd, None, B, params)

    clk = Clocks(local).__enter__()     # sampler up before the timed region
    for _ in range(args.warmup):
        res = solve()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    st = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    clk.mark(True)
    e0.record(st)
    for _ in range(args.steps):
        res = solve()
    e1.record(st)
    torch.cuda.synchronize()
    clk.mark(False)
    clk.__exit__()
    ms = e0.elapsed_time(e1) / args.steps
    if ws > 1:
        ms = max_over_ranks(ms, dist, torch, "cuda")
    x_dev = res.x
    xs = P.problems.manufactured_solution(nx * ny * nz)
    x_err = float(np.linalg.norm(x_dev.cpu().numpy() - xs) / np.linalg.norm(xs))

    # e2e: public API from pinned host buffers (H2D of b, D2H of x inside)
    b_pin = torch.from_numpy(b).pin_memory()
    P.gmres_solve(A, b_pin, None, B, params)
    torch.cuda.synchronize()
    te = []
    for _ in range(max(1, min(args.steps, 3))):
        t0 = time.perf_counter()
        r2 = P.gmres_solve(A, b_pin, None, B, params)
        _ = r2.x.numpy()
        te.append(time.perf_counter() - t0)
    e2e_ms = float(np.median(te) * 1e3)
    if ws > 1:
        e2e_ms = max_over_ranks(e2e_ms, dist, torch, "cuda")
    small = sum((j + 2) * 8 + 16 for j in range(res.inner)) + 8 * (3 + 2 * res.outer)

    # per-kernel timing on the launching stream (CUDA events), algorithmic bytes
    peak, peak_kind = _peaks()
    nb, nnzb = A.nrows, A.nnz
    w = D.empty(n)
    z = D.empty(n)
    lvl0 = Bd.amg.levels[0]
    A0 = B.pressure_solver.levels[0].A
    kern = {}
    warm = {}
    reps = 20
    flush = torch.empty(64 << 20, dtype=torch.float64, device="cuda")     # 512 MB > L2

    def both(name, fn, byt):
        kern[name] = (_time_cold(fn, reps, torch, flush), byt)
        warm[name] = _time_op(fn, reps, torch)

    both("bsr_spmv", lambda: lib.cprb_spmv(M.desc_ref(), 3, D.ptr(bd), D.ptr(w), None, D.stream()),
         _bytes_spmv(nb, nnzb))
    bp = D.empty(A0.nrows)
    xp = D.zeros(A0.nrows)
    bp.copy_(torch.from_numpy(np.ascontiguousarray(b[0::3])).cuda())
    both("pgs_scm_sweep_l0", lambda: lib.cprb_pgs_scm_pass(C.byref(lvl0.desc), D.ptr(bp), D.ptr(xp),
                                                           1, 0, D.stream()),
         _bytes_sweep(A0.nrows, A0.nnz))
    bc = Bd.amg.levels[1].b if len(Bd.amg.levels) > 1 else D.empty(A0.nrows)
    both("resid_restrict_l0", lambda: lib.cprb_resid_restrict(C.byref(lvl0.desc), D.ptr(bp), D.ptr(xp),
                                                              D.ptr(bc), D.stream()),
         A0.nnz * 12 + A0.nrows * 28)
    Fl = B.relaxation
    n_off_l = Fl.L.nnz - nb
    n_off_u = Fl.U.nnz - nb
    both("bilu_apply", lambda: Bd.bilu.apply(bd, z), _bytes_bilu(nb, n_off_l, n_off_u))
    zp = D.empty(nb)
    lv = B.pressure_solver.levels
    vbytes = sum(2 * _bytes_sweep(l.A.nrows, l.A.nnz) + l.A.nnz * 12 + l.A.nrows * 28
                 for l in lv[:-1])
    both("amg_vcycle", lambda: N.check(lib.cprb_amg_cycle_graph(Bd.graphs, C.byref(Bd.amg.desc),
                                                                D.ptr(bd), D.ptr(zp), D.stream())),
         vbytes)
    both("cpr_apply", lambda: Bd.apply(bd, z), None)
    del flush
    kernels = {}
    for k, (us_, byt) in kern.items():
        d = {"us": round(us_, 2), "us_warm_l2": round(warm[k], 2)}
        if byt:
            gbs = byt / (us_ * 1e-6) / 1e9
            d.update({"bytes": int(byt), "GB/s": round(gbs, 1), "frac": round(gbs / peak, 4)})
        kernels[k] = d
    # dominant kernel over one solve: count per-solve invocations
    napply = res.inner + res.outer
    share = {"bilu_apply": kern["bilu_apply"][0] * napply,
             "amg_vcycle": kern["amg_vcycle"][0] * napply,
             "bsr_spmv": kern["bsr_spmv"][0] * (2 * res.inner + 2 * res.outer + napply)}
    dom = max(share, key=share.get)
    dus, dbytes = kern[dom]
    achieved = dbytes / (dus * 1e-6) / 1e9
    traffic, traffic_src = _ncu_traffic(dom, tuple(args.grid))
    roofline = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 4),
                "traffic": traffic, "traffic_source": traffic_src,
                "algorithmic_bytes": int(dbytes),
                "share_of_step": round(share[dom] * 1e-3 / ms, 3)}

    launches_per_solve, kernel_names = _count_launches(solve, torch)
    out = {
        "metric": METRIC, "value": round(ms, 4), "unit": "ms", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator restated bitwise: seed 0, drift 0.01)",
        "config": _config(args.grid, args.cycle, ws, n, nnzb, len(lv)),
        "iters": {"outer": res.outer, "inner": res.inner, "rel_residual": res.rel_residual,
                  "x_err_vs_manufactured": x_err},
        "e2e": {"value": round(e2e_ms, 4), "unit": "ms", "h2d_bytes_per_step": int(8 * n),
                "d2h_bytes_per_step": int(8 * n + small)},
        "roofline": roofline, "kernels": kernels,
        "setup_s": round(t_setup, 2), "generate_s": round(t_gen, 2),
        "gpu_launches": launches_per_solve * args.steps,
        "gpu_launches_per_solve": launches_per_solve, "kernel_families": kernel_names,
        "clocks": clk.summary(),
    }
    if ws > 1:
        out["scaling"] = "weak"
        out["config"]["parallelism"] = (f"--replicas: {ws} independent systems, one per GPU "
                                        "(seed = rank), no data-path collective")
    if rank == 0 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(A, b, args, sample=True)
    if rank == 0:
        print(json.dumps(out))
    if ws > 1:
        dist.destroy_process_group()


def _partitioned_record(grid, cycle, steps, warmup, ws, rank, local, torch, dist, clocks=True):
    """One system row-partitioned over the ws ranks (
    paper_2201_01970_b200/partition.py): timed solves (max over ranks) and the
    e2e solve from pinned host buffers.  Returns rank 0's record."""
    import paper_2201_01970_b200 as P
    from paper_2201_01970_b200 import partition as S

    nx, ny, nz = grid
    t0 = time.perf_counter()
    (A, b), = P.generate_blackoil_like_sequence(nx, ny, nz, 1, 0.01, 0).systems
    t_gen = time.perf_counter() - t0
    cfg = P.SolverConfig(theta=0.0, theta_amg=0.0, cycle=cycle)
    t0 = time.perf_counter()
    B = P.build_cpr(A, cfg)
    comm = S.SlabComm()
    part = S.SlabPartition(A.nrows, ws)
    cpr = S.SlabCpr(B, part, comm)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    a, e = part.rows(rank)
    b_loc = np.ascontiguousarray(b[3 * a:3 * e])
    bd = torch.from_numpy(b_loc).cuda()
    params = cfg.gmres_params()

    def solve(rhs):
        return S.gmres_solve_slab(A, rhs, None, B, params, comm=comm, part=part, cpr=cpr)

    clk = Clocks(local).__enter__() if clocks else None
    for _ in range(warmup):
        res = solve(bd)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    st = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if clk:
        clk.mark(True)
    e0.record(st)
    for _ in range(steps):
        res = solve(bd)
    e1.record(st)
    torch.cuda.synchronize()
    if clk:
        clk.mark(False)
        clk.__exit__()
    ms = e0.elapsed_time(e1) / steps
    if ws > 1:
        ms = max_over_ranks(ms, dist, torch, "cuda")
    x = S.gather_rows(res.x, part, comm, 3).cpu().numpy()
    xs = P.problems.manufactured_solution(nx * ny * nz)
    x_err = float(np.linalg.norm(x - xs) / np.linalg.norm(xs))
    b_pin = torch.from_numpy(b_loc).pin_memory()
    solve(b_pin)                 # warm the pinned result buffers (as run_ours does)
    torch.cuda.synchronize()
    te = []
    for _ in range(max(1, min(steps, 3))):
        if ws > 1:
            dist.barrier()
        t0 = time.perf_counter()
        r2 = solve(b_pin)
        _ = r2.x.numpy()
        te.append(time.perf_counter() - t0)
    e2e_ms = float(np.median(te) * 1e3)
    if ws > 1:
        e2e_ms = max_over_ranks(e2e_ms, dist, torch, "cuda")
    launches_per_solve, kernel_names = _count_launches(lambda: solve(bd), torch)
    out = {
        "metric": METRIC, "value": round(ms, 4), "unit": "ms", "n_gpus": ws,
        "steps": steps, "warmup": warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator restated bitwise: seed 0, drift 0.01)",
        "config": _config(grid, cycle, ws, b.shape[0], A.nnz, len(B.pressure_solver.levels)),
        "partition": {"ranks": ws, "seg_cells": part.seg_cells, "bilu": cpr.bilu_mode,
                      "rows_per_rank": [int(part.rows(q)[1] - part.rows(q)[0]) for q in range(ws)],
                      "coarse_levels": "levels >= 1 agglomerated on rank 0"},
        "iters": {"outer": res.outer, "inner": res.inner, "rel_residual": res.rel_residual,
                  "x_err_vs_manufactured": x_err},
        "e2e": {"value": round(e2e_ms, 4), "unit": "ms", "h2d_bytes_per_step": int(8 * b_loc.size),
                "d2h_bytes_per_step": int(8 * b_loc.size)},
        "setup_s": round(t_setup, 2), "generate_s": round(t_gen, 2),
        "gpu_launches": launches_per_solve * steps,
        "gpu_launches_per_solve": launches_per_solve, "kernel_families": kernel_names,
    }
    if clk:
        out["clocks"] = clk.summary()
    del cpr, B, A
    return out


def run_partitioned(args):
    """N > 1 default (and --partition at N = 1): the C3 system row-partitioned
    over the N ranks (strong scaling anchored on the N = 1 BENCH line), plus
    a config-5 (26.9M DOF) sub-record at the same N (the north star's scaling
    system; --no-c5 skips it)."""
    import torch
    import torch.distributed as dist

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    out = _partitioned_record(tuple(args.grid), args.cycle, args.steps, args.warmup, ws, rank,
                              local, torch, dist)
    if ws > 1 and not args.no_c5 and tuple(args.grid) == (60, 220, 85):
        try:
            torch.cuda.empty_cache()
            c5 = _partitioned_record((120, 440, 170), args.cycle, max(1, min(args.steps, 5)),
                                     3, ws, rank, local, torch, dist, clocks=False)
            out["c5"] = {k: c5[k] for k in ("value", "unit", "steps", "warmup", "config", "partition",
                                            "iters", "e2e", "setup_s", "gpu_launches_per_solve")}
        except Exception as exc:  # reported, not fatal: the C3 line above is the bench line
            out["c5"] = {"error": repr(exc)[:300]}
    if rank == 0:
        print(json.dumps(out))
    if ws > 1:
        dist.destroy_process_group()


def run_c2(args):
    """Config 2: one AMG V(1,1) cycle on the 128^3 variable-coefficient
    pressure system (AMG stage alone, 1 GPU; src/amg.py:228-267)."""
    import ctypes as C

    import torch

    import paper_2201_01970_b200 as P
    from paper_2201_01970_b200 import _native as N
    from paper_2201_01970_b200 import device as D

    torch.cuda.set_device(0)
    t0 = time.perf_counter()
    A = P.problems.pressure_operator(128, 128, 128)
    h = P.build_hierarchy(A, P.AmgParams(theta_amg=0.0, cycle="v"))
    dev = h.device(1)
    t_setup = time.perf_counter() - t0
    n = A.nrows
    r = D.upload(np.ones(n))
    z = D.empty(n)
    cache = C.c_void_p()
    N.check(N.lib().cprb_graph_cache_create(C.byref(cache)))
    cyc = lambda: N.check(N.lib().cprb_amg_cycle_graph(cache, C.byref(dev.desc), D.ptr(r), D.ptr(z),
                                                       D.stream()))
    for _ in range(max(args.warmup, 3)):
        cyc()
    us = _time_op(cyc, max(args.steps, 10), torch)
    peak, peak_kind = _peaks()
    lv = h.levels
    vbytes = sum(2 * _bytes_sweep(l.A.nrows, l.A.nnz) + l.A.nnz * 12 + l.A.nrows * 28
                 for l in lv[:-1])
    lvl0 = dev.levels[0]
    xp = D.zeros(n)
    us0 = _time_op(lambda: N.lib().cprb_pgs_scm_pass(C.byref(lvl0.desc), D.ptr(r), D.ptr(xp), 1, 0,
                                                     D.stream()), 20, torch)
    b0 = _bytes_sweep(n, A.nnz)
    r_pin = torch.ones(n, dtype=torch.float64).pin_memory()
    te = []
    for _ in range(5):
        t1 = time.perf_counter()
        _ = P.amg_cycle(h, r_pin).numpy()
        te.append(time.perf_counter() - t1)
    ach = vbytes / (us * 1e-6) / 1e9
    out = {"metric": "AMG V(1,1)-cycle time, 128^3 pressure system (config 2)", "value": round(us / 1e3, 4),
           "unit": "ms", "n_gpus": 1, "steps": max(args.steps, 10), "warmup": max(args.warmup, 3),
           "higher_is_better": False, "dtype": "f64", "data": "synthetic (reference generator, seed 0)",
           "config": {"workload": "128^3 pressure operator, AmgParams(theta_amg=0, cycle='v'), b = ones",
                      "rows": n, "nnz": int(A.nnz), "levels": len(lv),
                      "colors": [l.partition.c for l in lv[:-1]]},
           "e2e": {"value": round(float(np.median(te)) * 1e3, 4), "unit": "ms",
                   "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n},
           "roofline": {"bound": "hbm", "kernel": "amg_vcycle (all levels)", "achieved": round(ach, 1),
                        "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                        "frac": round(ach / peak, 4), "algorithmic_bytes": int(vbytes)},
           "kernels": {"pgs_scm_sweep_l0": {"us": round(us0, 2), "bytes": int(b0),
                                            "GB/s": round(b0 / (us0 * 1e-6) / 1e9, 1),
                                            "frac": round(b0 / (us0 * 1e-6) / 1e9 / peak, 4)}},
           "setup_s": round(t_setup, 2)}
    N.lib().cprb_graph_cache_destroy(cache)
    print(json.dumps(out))


def run_c4(args):
    """Config 4: 10 Newton Jacobians of the SPE10-shaped model through the
    adaptive-setup sequence solver (src/cpr.py:349-382), mu = 5."""
    import torch

    import paper_2201_01970_b200 as P

    torch.cuda.set_device(0)
    nx, ny, nz = args.grid
    t0 = time.perf_counter()
    seq = P.generate_blackoil_like_sequence(nx, ny, nz, 10, 0.01, 0)
    systems = [(A, torch.from_numpy(b).cuda()) for A, b in seq.systems]
    t_gen = time.perf_counter() - t0
    cfg = P.SolverConfig(theta=0.0, theta_amg=0.0, cycle=args.cycle)
    P.ascpr_gmres_sequence(systems[:1], 5, cfg, keep_solutions=False)   # warm-up (module init)
    res = P.ascpr_gmres_sequence(systems, 5, cfg, keep_solutions=False)
    recs = res.records
    out = {"metric": "ASCPR sequence: SOLVE and SETUP time over 10 Newton Jacobians (config 4)",
           "value": round(res.solve_time * 1e3, 3), "unit": "ms", "n_gpus": 1, "steps": 1,
           "warmup": 1, "higher_is_better": False, "dtype": "f64",
           "data": "synthetic (reference generator restated bitwise: seed 0, drift 0.01)",
           "config": {"workload": f"10 SPE10-shaped {nx}x{ny}x{nz} systems, mu = 5, "
                                  f"SolverConfig(theta=0, theta_amg=0, cycle='{args.cycle}')"},
           "setup_calls": res.setup_calls, "setup_s": round(res.setup_time, 3),
           "solve_ms_per_system": round(res.solve_time * 1e3 / len(recs), 3),
           "inner": [r.inner for r in recs], "outer": [r.outer for r in recs],
           "rebuilt": [bool(r.rebuilt) for r in recs],
           "converged": all(r.converged for r in recs), "generate_s": round(t_gen, 2),
           "note": ("each Jacobian is assembled in HBM by the device generator (csrc/gen.cu, "
                    "bitwise the reference's values; its host copy is downloaded for the API), so "
                    "no upload lies inside the solve; generate_s covers the random draws, the "
                    "device assembly and the host copies of all 10 systems")}
    print(json.dumps(out))


def _ncu_traffic(kernel: str, grid):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`
    (a bench kernel family) from the committed ncu --set full capture
    summarised in profiles/ (tools/ncu_summary.py); None if absent."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None, None
    d = json.loads(p.read_text())
    if tuple(d.get("grid", (60, 220, 85))) != tuple(grid):
        return None, None                    # captured on another workload
    e = d.get("kernels", {}).get(kernel)
    if not e:
        return None, None
    return int(e["dram_bytes"]), e.get("source") or d.get("source")


def _count_launches(solve, torch):
    """Kernels of libcprb200 launched by one solve, counted from CUPTI kernel
    records (torch.profiler), graph-replayed kernels included."""
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        solve()
        torch.cuda.synchronize()
    names = {}
    n = 0
    for ev in prof.events():
        if getattr(ev, "device_type", None) is None or str(ev.device_type).endswith("CPU"):
            continue
        nm = ev.name
        if "cprb" in nm or nm.startswith(("k_", "void k_")):
            n += 1
            fam = nm.split("(")[0].split("<")[0].replace("void ", "").replace("cprb::", "")
            names[fam] = names.get(fam, 0) + 1
    return n, names


def cpu_baseline(A, b, args, sample=True):
    """The oracle's CPR-GMRES solve on the host (1 thread: the reference's
    GIL-bound path), on the same system and config.  Setup comes from the
    oracle's own restatement of the reference's setup."""
    from oracle import cprkit_oracle as orc
    Ao = orc.Bsr(3, A.nrows, A.ncols, A.row_ptr, A.col_idx, A.values)
    cfg = orc.SolverConfig(theta=0.0, theta_amg=0.0, cycle=args.cycle)
    t0 = time.perf_counter()
    B = orc.build_cpr(Ao, cfg)
    t_setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    res = orc.gmres_solve(Ao, b, None, B, cfg.m, cfg.max_restarts, cfg.tol)
    t_solve = time.perf_counter() - t0
    return {"value": round(t_solve * 1e3, 1), "unit": "ms", "cores": 1, "kind": "port",
            "sample": f"one full CPR-GMRES solve of the same {A.nrows * 3}-DOF system "
                      f"(outer={res.outer}, inner={res.inner}); oracle setup {t_setup:.1f} s "
                      "untimed; numpy/OpenBLAS single thread",
            "host_cpus": os.cpu_count()}


def run_reference(args):
    """Reference arm: the reference's CPU algorithm (the oracle port; the
    reference is pure Python and compiles nothing) on the
    host cores, for the same workload and config dict as our arm.  Every step
    (warm-up and timed) is one COMPLETE CPR-GMRES solve of the same system
    (src/cpr.py:231-316, preconditioner built beforehand as the reference
    times SETUP and SOLVE separately, src/cpr.py:369-376).  Under torchrun only
    rank 0 runs; the other ranks exit without work."""
    ws, rank, _ = _dist()
    if rank != 0:
        return
    sys.path.insert(0, str(ROOT))
    from oracle import cprkit_oracle as orc
    nx, ny, nz = args.grid
    (A, b), = orc.generate_blackoil_like_sequence(nx, ny, nz, 1, 0.01, 0)
    cfg = orc.SolverConfig(theta=0.0, theta_amg=0.0, cycle=args.cycle)
    t0 = time.perf_counter()
    B = orc.build_cpr(A, cfg)
    t_setup = time.perf_counter() - t0
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        res = orc.gmres_solve(A, b, None, B, cfg.m, cfg.max_restarts, cfg.tol)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    ms = float(np.mean(times) * 1e3)
    nlev = len(B.hierarchy.levels)
    sample = (f"each step = one complete CPR-GMRES solve of the same {b.shape[0]}-DOF system on the "
              f"oracle port (numpy restatement of cprkit, ~4x faster than the unmodified cprkit "
              f"package: SURVEY.md 0.3 measured 53.7 s per C3 V solve for cprkit itself); "
              f"outer={res.outer}, inner={res.inner}, rel={res.rel_residual:.6e}; oracle setup "
              f"{t_setup:.1f} s untimed; numpy single thread (the reference's path is GIL-bound, "
              f"pkg/README.md:114-124)")
    out = {"impl": "reference", "metric": METRIC, "value": round(ms, 2), "unit": "ms",
           "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 2),
           "higher_is_better": False, "scaling": "strong" if ws > 1 else "weak",
           "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (reference generator restated bitwise: seed 0, drift 0.01)",
           "config": _config(args.grid, args.cycle, ws, b.shape[0], A.nnz, nlev),
           "iters": {"outer": res.outer, "inner": res.inner, "rel_residual": res.rel_residual},
           "cpu_baseline": {"value": round(ms, 2), "unit": "ms", "cores": 1, "kind": "port",
                            "sample": sample, "host_cpus": os.cpu_count()},
           "e2e": {"value": round(ms, 2), "unit": "ms", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def _spawn(args) -> int:
    """--gpus N without torchrun: relaunch this command as N ranks on this
    node (torch.distributed.run, rendezvous on 127.0.0.1)."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--grid", type=_grid, default=(60, 220, 85))
    ap.add_argument("--cycle", default="v", choices=["v", "k"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--config", default="c3", choices=["c3", "c2", "c4"],
                    help="c2: AMG V-cycle on 128^3 pressure; c4: ASCPR 10-system sequence")
    ap.add_argument("--partition", action="store_true",
                    help="N = 1: run the row-slab partitioned path (the N > 1 default)")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent systems per GPU (weak scaling) instead of the partition")
    ap.add_argument("--no-c5", action="store_true", help="N > 1: skip the config-5 sub-record")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(_spawn(args))
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
    if args.impl == "reference":
        run_reference(args)
    elif args.config == "c2":
        run_c2(args)
    elif args.config == "c4":
        run_c4(args)
    elif (ws > 1 and not args.replicas) or args.partition:
        run_partitioned(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
