"""Structured-grid BILU(0) solves (csrc/stencil.cu, ilu.stencil_plan).

CPU: the plan's detection rules and a numpy emulation of the kernel's
diagonal sweep over the plan's records, bitwise against the oracle's
level-scheduled solve (src/ilu.py:196-223).  GPU: the kernel itself, bitwise
against the oracle and against the general chunked-wavefront kernel, for
every lane-segment count S = ceil(nx / 32) = 1..4."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import orc, random_block

import paper_2201_01970_b200 as P
from paper_2201_01970_b200.ilu import _strict, stencil_plan


def _oracle_bilu(F):
    lp, lc, lv = _strict(F.L)
    up, uc, uv = _strict(F.U)
    return orc.Bilu(F.n, F.block_size, lp, lc, lv, up, uc, uv, F.u_diag_inv,
                    F.l_schedule.levels, F.u_schedule.levels)


def _grid(nx, ny, nz, seed=0, drift=0.01):
    (A, b), = P.generate_blackoil_like_sequence(nx, ny, nz, 1, drift, seed).systems
    return A


def _emulate(pl, r):
    """The kernel's arithmetic on the plan's records (numpy, one plane and
    one anti-diagonal at a time; all lanes of a diagonal at once)."""
    nx, ny, nz, Dn, P_ = pl["nx"], pl["ny"], pl["nz"], pl["D"], pl["P"]
    doff, slot = pl["doff"].astype(np.int64), pl["slot"].astype(np.int64)
    rhs = np.zeros(pl["len"])
    for c in range(3):
        rhs[slot + c] = r[c::3]
    out = {}
    for upper in (False, True):
        nf = 37 if upper else 27
        rec = (pl["urec"] if upper else pl["lrec"]).reshape(-1, nf)
        res = np.zeros(pl["len"])
        planes = range(nz - 1, -1, -1) if upper else range(nz)
        for z in planes:
            has_z = z + 1 < nz if upper else z > 0
            zb = (z + 1) * P_ if upper else (z - 1) * P_
            for t in range(Dn):
                d = Dn - 1 - t if upper else t
                lo, hi = max(0, d - (ny - 1)), min(nx - 1, d)
                o, wp = int(doff[d]), int(doff[d + 1] - doff[d])
                ix = np.arange(lo, hi + 1)
                j = ix - lo
                iy = d - ix
                pos = z * P_ + o + j
                blk = rec[pos].T
                rh = rhs[3 * pos[:, None] + np.arange(3)]
                # neighbour values (ascending column order)
                if upper:
                    nb = [(ix + 1 < nx, z * P_ + doff[d + 1] + (ix + 1 - max(0, d + 1 - (ny - 1))) if d + 1 < Dn else pos),
                          (iy + 1 < ny, z * P_ + doff[d + 1] + (ix - max(0, d + 1 - (ny - 1))) if d + 1 < Dn else pos),
                          (np.full(ix.shape, has_z), zb + o + j)]
                else:
                    nb = [(np.full(ix.shape, has_z), zb + o + j),
                          (iy > 0, z * P_ + doff[d - 1] + (ix - max(0, d - 1 - (ny - 1))) if d > 0 else pos),
                          (ix > 0, z * P_ + doff[d - 1] + (ix - 1 - max(0, d - 1 - (ny - 1))) if d > 0 else pos)]
                prods = []
                for m, (h, p) in enumerate(nb):
                    p = np.where(h, p, 0)
                    v = res[3 * p[:, None] + np.arange(3)]
                    pr = np.empty((ix.shape[0], 3))
                    for rr in range(3):
                        mm = blk[m * 9 + rr * 3:m * 9 + rr * 3 + 3].T
                        pr[:, rr] = (mm[:, 0] * v[:, 0] + mm[:, 2] * v[:, 2]) + mm[:, 1] * v[:, 1]
                    prods.append(np.where(h[:, None], pr, -0.0))
                anyh = nb[0][0] | nb[1][0] | nb[2][0]
                s = np.where(anyh[:, None], prods[0] + (prods[1] + prods[2]), 0.0)
                dd = rh - s
                if upper:
                    ui = blk[27:36].T.reshape(-1, 3, 3)
                    y = np.empty_like(dd)
                    for rr in range(3):
                        y[:, rr] = (ui[:, rr, 0] * dd[:, 0] + ui[:, rr, 2] * dd[:, 2]) + ui[:, rr, 1] * dd[:, 1]
                    dd = y
                res[3 * pos[:, None] + np.arange(3)] = dd
        out[upper] = res
        rhs = res
    y = out[True]
    return np.stack([y[slot + c] for c in range(3)], axis=1).reshape(-1)


def test_stencil_plan_detection():
    rng = np.random.default_rng(1)
    assert stencil_plan(P.bilu0_factorize(_grid(10, 10, 10))) is not None
    pl = stencil_plan(P.bilu0_factorize(_grid(40, 7, 5)))
    assert (pl["nx"], pl["ny"], pl["nz"], pl["S"], pl["D"]) == (40, 7, 5, 2, 46)
    assert np.all(np.diff(pl["doff"]) % 2 == 0)
    # every row has its own stencil position
    assert np.unique(pl["slot"]).shape[0] == 40 * 7 * 5
    # not a 7-point grid: general path
    M = random_block(rng, 60, 3, 4)
    assert stencil_plan(P.bilu0_factorize(P.BlockCsrMatrix(3, M.nrows, M.ncols, M.ptr, M.cols,
                                                             M.vals))) is None
    # too wide for 4 lane segments, and degenerate grids
    assert stencil_plan(P.bilu0_factorize(_grid(129, 2, 2))) is None
    assert stencil_plan(P.bilu0_factorize(_grid(6, 1, 4))) is None
    assert stencil_plan(P.bilu0_factorize(_grid(6, 5, 1))) is None


@pytest.mark.parametrize("shape", [(10, 10, 10), (40, 7, 5), (33, 3, 4), (2, 2, 2), (5, 9, 3)])
def test_stencil_emulation_bitwise_oracle(shape):
    F = P.bilu0_factorize(_grid(*shape, seed=sum(shape)))
    pl = stencil_plan(F)
    assert pl is not None
    r = np.random.default_rng(7).standard_normal(3 * F.n)
    r[::17] = 0.0
    assert np.array_equal(_emulate(pl, r), orc.bilu_apply(_oracle_bilu(F), r))


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(10, 10, 10), (40, 7, 5), (70, 9, 6), (100, 5, 4), (128, 3, 3),
                                   (2, 2, 2), (33, 40, 3)])
def test_stencil_kernel_bitwise_oracle_and_wave(gpu, shape, monkeypatch):
    import torch
    F = P.bilu0_factorize(_grid(*shape, seed=len(shape) + shape[0]))
    dev = F.device()
    assert dev.stencil
    Fo = _oracle_bilu(F)
    rng = np.random.default_rng(3)
    for _ in range(3):                        # re-armed tickets / sentinels every call
        r = rng.standard_normal(3 * F.n)
        rd = torch.from_numpy(r).cuda()
        z = torch.empty_like(rd)
        dev.apply(rd, z)
        assert np.array_equal(z.cpu().numpy(), orc.bilu_apply(Fo, r))
    # the general chunked-wavefront plan of the same factors agrees bitwise
    monkeypatch.setenv("CPRB_STENCIL", "0")
    from paper_2201_01970_b200.ilu import DeviceBilu
    gen = DeviceBilu(F)
    assert not gen.stencil
    z2 = torch.empty_like(rd)
    gen.apply(rd, z2)
    assert torch.equal(z, z2)


@pytest.mark.gpu
@pytest.mark.parametrize("shape,clusters", [((40, 7, 33), 1), ((70, 9, 20), 1), ((100, 5, 30), 1),
                                            ((128, 3, 25), 1), ((70, 9, 40), 2), ((33, 6, 17), 3)])
def test_stencil_persistent_rounds_bitwise(gpu, shape, clusters, monkeypatch):
    """Persistent clusters taking several rounds of 8 planes each (the grid is
    capped below nz / 8 clusters), S = 2..4 lane segments.  Exercises the
    DSMEM hand-off across rounds, where a warp whose segment is empty on a
    diagonal used to run a barrier phase ahead of its sender and hang."""
    import torch
    monkeypatch.setenv("CPRB_STENCIL_MAXCLUS", str(clusters))
    F = P.bilu0_factorize(_grid(*shape, seed=1))
    dev = F.device()
    assert dev.stencil
    Fo = _oracle_bilu(F)
    rng = np.random.default_rng(11)
    for _ in range(3):
        r = rng.standard_normal(3 * F.n)
        rd = torch.from_numpy(r).cuda()
        z = torch.empty_like(rd)
        dev.apply(rd, z)
        assert np.array_equal(z.cpu().numpy(), orc.bilu_apply(Fo, r))


_CLUSTER8_CHECK = """
import sys
import numpy as np
import torch
sys.path.insert(0, {tests!r})
import paper_2201_01970_b200 as P
from conftest import orc
from test_stencil import _grid, _oracle_bilu
for shape in ((40, 7, 33), (70, 9, 20), (60, 22, 19)):
    F = P.bilu0_factorize(_grid(*shape, seed=2))
    dev = F.device()
    assert dev.stencil
    r = np.random.default_rng(5).standard_normal(3 * F.n)
    rd = torch.from_numpy(r).cuda()
    z = torch.empty_like(rd)
    dev.apply(rd, z)
    assert np.array_equal(z.cpu().numpy(), orc.bilu_apply(_oracle_bilu(F), r)), shape
print("ok")
"""


@pytest.mark.gpu
@pytest.mark.parametrize("cluster", ["8", "4"])
def test_stencil_smaller_cluster_shapes_bitwise(gpu, cluster):
    """The launcher prefers 16-CTA clusters and falls back to 8 (then 4, 2)
    when the device cannot co-schedule them; the kernel reads the cluster
    size at run time.  Forced smaller shapes (fresh process: the choice is
    made once per device) stay bitwise equal to the oracle."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    tests = str(Path(__file__).resolve().parent)
    env = dict(os.environ, CPRB_STENCIL_CLUSTER=cluster, CPRB_STENCIL_MAXCLUS="1",
               PYTHONPATH=str(Path(tests).parent))
    out = subprocess.run([sys.executable, "-c", _CLUSTER8_CHECK.format(tests=tests)], env=env,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-2000:]


@pytest.mark.gpu
def test_stencil_cpr_solve_c1_matches_wave(gpu, monkeypatch):
    """A whole CPR-GMRES solve through the stencil BILU equals the one through
    the general wavefront bit for bit (same factors, same arithmetic)."""
    A = _grid(10, 10, 10)
    b = np.random.default_rng(0).standard_normal(3000)
    cfg = P.SolverConfig(theta=0.0, theta_amg=0.0, cycle="v")
    B = P.build_cpr(A, cfg)
    r1 = P.gmres_solve(A, b, None, B, cfg.gmres_params(), history=True)
    assert B.relaxation.device().stencil
    monkeypatch.setenv("CPRB_STENCIL", "0")
    B2 = P.build_cpr(A, cfg)
    r2 = P.gmres_solve(A, b, None, B2, cfg.gmres_params(), history=True)
    assert not B2.relaxation.device().stencil
    assert (r1.outer, r1.inner) == (r2.outer, r2.inner)
    assert r1.history == r2.history
    assert np.array_equal(r1.x, r2.x)
