"""Slab-partitioned CPR-GMRES across ranks.

One process per GPU.  Block rows (cells) are split into contiguous ranges
made of whole SEGMENTS (SEG_CELLS cells, a fixed global grid): for the
generated problems (x fastest, z slowest, src/problems.py:60-70) a range is
a z-slab.  Every rank holds the full host setup (hierarchy, BILU factors;
identical on every rank because setup is deterministic) and uploads:

* its rows of the Jacobian (BSR SpMV, residual, stage-2 residual), reading
  a contiguous column window [w0, w1) = own rows + one xy-plane of halo per
  side; halos are exchanged with NCCL point-to-point over NVLink;
* its rows of pressure level 0 (colour sweeps with a halo exchange after
  every colour, fused residual + restriction; aggregates are owned by the
  owner of their lowest member and the ~1.5 % that straddle a slab boundary
  get the other member's partial from the neighbour: (0 + r_a) + (0 + r_b)
  equals np.bincount's 0 + r_a + r_b bitwise);
* levels >= 1 are agglomerated on rank 0 (gather the level-1 right-hand
  side, run the device V-cycle from level 1, broadcast the correction), as
  the north star specifies;
* BILU(0) (src/ilu.py:196-223) is ONE global wavefront (SlabBilu): the wave
  plans are cut at the slab boundaries, every rank runs its own chunks and
  stores the rows its neighbour reads straight into the neighbour's output
  array (CUDA IPC peer memory over NVLink), where they are polled like any
  cross-chunk dependency.  The chain is sequential, so this is the Amdahl
  term; bilu="replicated" (all-gather + full solve per rank) serves ranks
  that share one GPU.
* the K-cycle's coarse correction (Krylov steps from level 1) runs on rank 0
  like the V-cycle's (cprb_kcycle_correction).

Reductions are GPU-count invariant: fixed global segments, one partial per
segment reduced in a fixed order by one CTA, all partials summed in global
segment order on every rank (csrc/slab.cu).  So Givens history, iteration
counts and the solution are bitwise identical for 1, 2, 4 and 8 ranks, and
every rank takes the same host decisions without extra collectives.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from . import device as D
from .amg import AmgHierarchy, DeviceAmg
from .cpr import GmresParams, GmresResult, _bsize, _solve_upper

__all__ = ["SEG_CELLS", "SlabPartition", "SlabComm", "SlabMatrix", "SlabCpr", "SlabBilu",
           "gmres_solve_slab", "halo_plan"]

SEG_CELLS = 1024
_SENT_BITS = 0x7FF4C0FFEE5EED01   # csrc/device.cuh CPRB_SENTINEL (not-yet-computed marker)


class SlabPartition:
    """Contiguous cell ranges of whole segments: rank p owns segments
    [nseg*p//N, nseg*(p+1)//N)."""

    def __init__(self, ncells: int, nranks: int, seg_cells: int = SEG_CELLS):
        if nranks < 1 or seg_cells < 1:
            raise ValueError("need nranks >= 1 and seg_cells >= 1")
        self.ncells, self.nranks, self.seg_cells = int(ncells), int(nranks), int(seg_cells)
        self.nseg = -(-self.ncells // self.seg_cells)
        self.seg0 = np.array([self.nseg * p // nranks for p in range(nranks + 1)], dtype=np.int64)
        self.cell0 = np.minimum(self.seg0 * self.seg_cells, self.ncells)

    def rows(self, p: int):
        return int(self.cell0[p]), int(self.cell0[p + 1])

    def owner(self, cells):
        return np.searchsorted(self.cell0, np.asarray(cells), side="right") - 1

    def seg_map(self):
        """(cap, map): partial slot of each global segment in the padded
        all-gather layout [rank][cap]."""
        counts = np.diff(self.seg0)
        cap = int(max(counts.max(), 1))
        s = np.arange(self.nseg, dtype=np.int64)
        q = np.searchsorted(self.seg0, s, side="right") - 1
        return cap, (q * cap + (s - self.seg0[q])).astype(np.int32)


def _windows(A, part: SlabPartition):
    """Column window [w0, w1) (cells) of every rank's rows of A."""
    rp = np.asarray(A.row_ptr, dtype=np.int64)
    ci = np.asarray(A.col_idx, dtype=np.int64)
    n = int(A.nrows)
    w = np.zeros((part.nranks, 2), dtype=np.int64)
    nonempty = rp[1:] > rp[:-1]
    rmin = np.full(n, n, dtype=np.int64)
    rmax = np.full(n, -1, dtype=np.int64)
    if ci.size:
        starts = rp[:-1][nonempty]
        rmin[nonempty] = np.minimum.reduceat(ci, starts)
        rmax[nonempty] = np.maximum.reduceat(ci, starts)
    for q in range(part.nranks):
        a, e = part.rows(q)
        lo = min(int(rmin[a:e].min()) if e > a else a, a)
        hi = max(int(rmax[a:e].max()) + 1 if e > a else e, e)
        w[q] = (lo, hi)
    return w


def halo_plan(part: SlabPartition, windows: np.ndarray, rank: int):
    """(sends, recvs): lists of (peer, a, e) cell ranges.  A send from p to q
    and the matching receive of q from p are the same range computed by the
    same formula on both sides, in the same order."""
    c0, c1 = part.rows(rank)
    w0, w1 = windows[rank]
    sends, recvs = [], []
    for q in range(part.nranks):
        if q == rank:
            continue
        q0, q1 = part.rows(q)
        v0, v1 = windows[q]
        for a, e in ((max(c0, v0), min(c1, q0)), (max(c0, q1), min(c1, v1))):
            if e > a:
                sends.append((q, a, e))
        for a, e in ((max(q0, w0), min(q1, c0)), (max(q0, c1), min(q1, w1))):
            if e > a:
                recvs.append((q, a, e))
    return sends, recvs


class SlabComm:
    """Transport of the partitioned solve.  NCCL: device tensors directly
    (point-to-point halos, all-gather, broadcast on the current stream).
    gloo (tests: several ranks sharing one GPU): staged through host memory."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.rank = dist.get_rank(group)
            self.size = dist.get_world_size(group)
            self.nccl = dist.get_backend(group) == "nccl"
            if self.nccl and self.size > 1:
                # every rank joins one collective before the first (uneven)
                # point-to-point batch creates the communicator
                t = D.zeros(1)
                dist.all_reduce(t, group=group)
        else:
            self.rank, self.size, self.nccl = 0, 1, False

    def exchange(self, sends, recvs):
        """sends / recvs: lists of (peer, tensor)."""
        if self.size == 1 or (not sends and not recvs):
            return
        dist = self.dist
        if self.nccl:
            ops = [dist.P2POp(dist.isend, t, p, self.group) for p, t in sends]
            ops += [dist.P2POp(dist.irecv, t, p, self.group) for p, t in recvs]
            for r in dist.batch_isend_irecv(ops):
                r.wait()
            return
        hs = [(p, t.cpu()) for p, t in sends]
        hr = [(p, D.torch().empty(t.shape, dtype=t.dtype)) for p, t in recvs]
        reqs = [dist.isend(t, p, self.group) for p, t in hs]
        reqs += [dist.irecv(t, p, self.group) for p, t in hr]
        for r in reqs:
            r.wait()
        for (_, t), (_, h) in zip(recvs, hr):
            t.copy_(h)

    def allgather(self, local, out):
        """out[q*cap:(q+1)*cap] = rank q's `local` (cap entries)."""
        if self.size == 1:
            out[:local.shape[0]].copy_(local)
            return
        if self.nccl:
            self.dist.all_gather_into_tensor(out, local, group=self.group)
            return
        t = D.torch()
        parts = [t.empty(local.shape, dtype=local.dtype) for _ in range(self.size)]
        self.dist.all_gather(parts, local.cpu(), group=self.group)
        out.copy_(t.cat(parts))

    def gather0(self, local, out):
        """Rank 0: out[q*cap:(q+1)*cap] = rank q's `local`; other ranks only send."""
        if self.size == 1:
            out[:local.shape[0]].copy_(local)
            return
        cap = local.shape[0]
        if self.nccl:
            parts = [out[q * cap:(q + 1) * cap] for q in range(self.size)] if self.rank == 0 else None
            self.dist.gather(local, parts, dst=0, group=self.group)
            return
        t = D.torch()
        parts = [t.empty(local.shape, dtype=local.dtype) for _ in range(self.size)] \
            if self.rank == 0 else None
        self.dist.gather(local.cpu(), parts, dst=0, group=self.group)
        if self.rank == 0:
            out.copy_(t.cat(parts))

    def broadcast(self, tensor, src: int = 0):
        if self.size == 1:
            return
        if self.nccl:
            self.dist.broadcast(tensor, src, group=self.group)
            return
        h = tensor.cpu()
        self.dist.broadcast(h, src, group=self.group)
        tensor.copy_(h)


class _Gatherer:
    """Padded all-gather of per-rank contiguous pieces into one packed
    vector (rank order)."""

    def __init__(self, counts):
        counts = np.asarray(counts, dtype=np.int64)
        self.nranks = counts.shape[0]
        self.cap = int(max(counts.max(), 1))
        offs = np.zeros(self.nranks + 1, dtype=np.int64)
        np.cumsum(counts, out=offs[1:])
        self.offs = offs
        self.offs_dev = D.upload(offs)
        self.local = D.zeros(self.cap)
        self.buf = D.zeros(self.nranks * self.cap)

    def __call__(self, comm: SlabComm, src, n_local: int, out, root_only: bool = False):
        """root_only: only rank 0 receives (and unpacks) the result."""
        if comm.size == 1:
            out[:n_local].copy_(src[:n_local])
            return
        self.local[:n_local].copy_(src[:n_local])
        if root_only:
            comm.gather0(self.local, self.buf)
            if comm.rank != 0:
                return
        else:
            comm.allgather(self.local, self.buf)
        N.check(N.lib().cprb_unpad(self.nranks, self.cap, D.ptr(self.offs_dev), D.ptr(self.buf),
                                   D.ptr(out), D.stream()))


class SlabMatrix:
    """This rank's block rows of A with columns relative to its window."""

    def __init__(self, A, part: SlabPartition, rank: int):
        D.require_cuda()
        self.b = _bsize(A)
        self.part, self.rank = part, rank
        self.c0, self.c1 = part.rows(rank)
        self.windows = _windows(A, part)
        self.w0, self.w1 = (int(v) for v in self.windows[rank])
        rp = np.asarray(A.row_ptr, dtype=np.int64)
        ci = np.asarray(A.col_idx, dtype=np.int64)
        vals = np.asarray(A.values, dtype=np.float64)
        e0, e1 = int(rp[self.c0]), int(rp[self.c1])
        ptr = rp[self.c0:self.c1 + 1] - e0
        v = vals[e0:e1]
        if self.b == 1:
            v = v.reshape(-1)
        self.sell = D.SellDev(D.sell_rows(ptr, ci[e0:e1] - self.w0, v, self.b, self.c1 - self.c0))
        self.sends, self.recvs = halo_plan(part, self.windows, rank)

    @property
    def n_own(self) -> int:
        return self.c1 - self.c0

    @property
    def win_len(self) -> int:
        return self.w1 - self.w0

    def interior(self, vec, b: int):
        return vec[(self.c0 - self.w0) * b:(self.c1 - self.w0) * b]

    def exchange(self, comm: SlabComm, vec, b: int):
        """Refresh the halo of a window-layout vector (b values per cell)."""
        sl = lambda a, e: vec[(a - self.w0) * b:(e - self.w0) * b]
        comm.exchange([(q, sl(a, e)) for q, a, e in self.sends],
                      [(q, sl(a, e)) for q, a, e in self.recvs])

    def desc_ref(self):
        return C.byref(self.sell.desc)


class SlabLevel0:
    """This rank's rows of pressure level 0 in local colour-permuted order:
    own rows colour by colour (each colour's rows in the global permuted
    order), then the halo cells (natural order: [w0, c0) then [c1, w1))."""

    def __init__(self, h: AmgHierarchy, part: SlabPartition, rank: int):
        lvl = h.levels[0]
        sp = lvl.smoother.split
        A0 = lvl.A
        self.c0, self.c1 = c0, c1 = part.rows(rank)
        n_own = c1 - c0
        self.n_own = n_own
        perm, inv = sp.perm, sp.inv
        crg = np.asarray(sp.color_rows, dtype=np.int64)
        ncol = sp.ncolors
        if ncol < 2:
            raise NotImplementedError("slab partition: a single-colour level 0 is a sequential "
                                      "Gauss-Seidel sweep (src/smoothers.py:296-299)")
        gp = np.sort(inv[c0:c1])                        # global permuted positions
        cells = perm[gp]                                 # natural cell of each local row
        kcol = np.searchsorted(crg, gp, side="right") - 1
        cr = np.zeros(ncol + 1, dtype=np.int64)
        np.cumsum(np.bincount(kcol, minlength=ncol), out=cr[1:])
        self.windows = _windows(A0, part)
        w0, w1 = (int(v) for v in self.windows[rank])
        self.w0, self.w1 = w0, w1
        loc_own = np.empty(n_own, dtype=np.int64)
        loc_own[cells - c0] = np.arange(n_own, dtype=np.int64)
        self.loc_own = loc_own

        def lidx(g):
            g = np.asarray(g, dtype=np.int64)
            out = np.empty(g.shape, dtype=np.int64)
            own = (g >= c0) & (g < c1)
            lo = g < c0
            hi = g >= c1
            out[own] = loc_own[g[own] - c0]
            out[lo] = n_own + (g[lo] - w0)
            out[hi] = n_own + (c0 - w0) + (g[hi] - c1)
            return out

        self.n_x = n_own + (c0 - w0) + (w1 - c1)
        # off-diagonal entries (ascending GLOBAL permuted column = the
        # reference's GS sum order), columns renamed to local indices
        lo_p, hi_p = sp.off_ptr[gp], sp.off_ptr[gp + 1]
        lens = (hi_p - lo_p).astype(np.int64)
        ptr = np.zeros(n_own + 1, dtype=np.int64)
        np.cumsum(lens, out=ptr[1:])
        nnz = int(ptr[-1])
        row_of = np.repeat(np.arange(n_own, dtype=np.int64), lens)
        src = lo_p[row_of] + (np.arange(nnz, dtype=np.int64) - ptr[row_of])
        ent_gp = sp.off_cols[src]
        ent_v = sp.off_vals[src]
        rk = kcol[row_of]
        # colours with intra-colour couplings sweep against a snapshot
        # (src/smoothers.py:301-308); a GLOBAL property of the colour
        g_rows = np.repeat(np.arange(sp.n, dtype=np.int64), np.diff(sp.off_ptr))
        g_k = np.searchsorted(crg, g_rows, side="right") - 1
        intra = (sp.off_cols >= crg[g_k]) & (sp.off_cols < crg[g_k + 1])
        snap = np.zeros(max(ncol, 1), dtype=np.uint8)
        if intra.any():
            snap[np.unique(g_k[intra])] = 1
        ent_l = lidx(perm[ent_gp])
        lo_cnt = np.zeros(n_own, dtype=np.int64)
        np.add.at(lo_cnt, row_of[ent_gp < crg[rk]], 1)
        # SELL-32, each colour padded to whole slices (as ScalarSplit.sell)
        lanes, slices = [], [0]
        for k in range(ncol):
            lanes.append(D.pad_lanes(np.arange(cr[k], cr[k + 1], dtype=np.int32)))
            slices.append(slices[-1] + lanes[-1].shape[0] // 32)
        lane_row = np.concatenate(lanes) if lanes else np.zeros(0, dtype=np.int32)
        L = lane_row.shape[0]
        real = lane_row >= 0
        llen = np.zeros(L, dtype=np.int64)
        llen[real] = lens[lane_row[real]]
        lane_ptr = np.zeros(L + 1, dtype=np.int64)
        np.cumsum(llen, out=lane_ptr[1:])
        lane_lo = np.zeros(L, dtype=np.int32)
        lane_lo[real] = lo_cnt[lane_row[real]]
        hs = D.pack_sell(lane_row, lane_ptr, ent_l, ent_v, 1, n_own, lane_len_lo=lane_lo)
        self.smoother = D.SellDev(hs)
        self.diag = D.upload(sp.diag[gp])
        self.perm_local = D.upload((cells - c0).astype(np.int32))
        self.color_slices = np.asarray(slices, dtype=np.int32)
        self.color_rows = cr.astype(np.int32)
        self.snapshot = snap
        cw = np.zeros(2 * max(ncol, 1), dtype=np.int32)
        for k in range(ncol):
            a, e = int(slices[k]) * 32, int(slices[k + 1]) * 32
            if e > a:
                cw[2 * k] = int(hs.lane_len[a:e].max())
                cw[2 * k + 1] = int(hs.lane_len_lo[a:e].max())
        self.color_width = cw
        self.ncolors = ncol

        # -- residual + restriction: aggregates owned by their lowest member's rank
        agg = np.asarray(lvl.aggregates, dtype=np.int64)
        n0 = agg.shape[0]
        n1 = int(h.levels[1].A.nrows)
        idx = np.arange(n0, dtype=np.int64)
        mlo = np.full(n1, n0, dtype=np.int64)
        np.minimum.at(mlo, agg, idx)
        mhi = np.full(n1, -1, dtype=np.int64)
        np.maximum.at(mhi, agg, idx)
        mhi[mhi == mlo] = -1
        aowner = part.owner(mlo)
        ga = np.flatnonzero(aowner == rank)
        if ga.size and not np.array_equal(ga, np.arange(ga[0], ga[0] + ga.size)):
            raise RuntimeError("slab partition: owned aggregates are not contiguous")
        self.ga0 = int(ga[0]) if ga.size else 0
        self.n_agg = int(ga.size)
        self.agg_counts = np.bincount(aowner, minlength=part.nranks)
        self.agg_offs = np.concatenate([[0], np.cumsum(self.agg_counts)])
        hi_own = (mhi >= c0) & (mhi < c1)
        partial = np.flatnonzero(hi_own & (aowner != rank))     # my member is the upper one
        up = mhi[ga]
        up_ok = (up >= c0) & (up < c1)
        lane_orig = np.full(2 * (ga.size + partial.size), -1, dtype=np.int64)
        lane_orig[0:2 * ga.size:2] = mlo[ga]
        lane_orig[1:2 * ga.size:2] = np.where(up_ok, up, -1)
        lane_orig[2 * ga.size::2] = mhi[partial]
        lane_orig = D.pad_lanes(lane_orig)
        Lr = lane_orig.shape[0]
        realr = lane_orig >= 0
        rp = np.asarray(A0.row_ptr, dtype=np.int64)
        rlen = np.zeros(Lr, dtype=np.int64)
        rlen[realr] = (rp[1:] - rp[:-1])[lane_orig[realr]]
        rptr = np.zeros(Lr + 1, dtype=np.int64)
        np.cumsum(rlen, out=rptr[1:])
        rnnz = int(rptr[-1])
        lane_of = np.repeat(np.arange(Lr, dtype=np.int64), rlen)
        rsrc = rp[lane_orig[lane_of]] + (np.arange(rnnz, dtype=np.int64) - rptr[lane_of])
        rcols = lidx(np.asarray(A0.col_idx, dtype=np.int64)[rsrc])
        rvals = np.asarray(A0.values, dtype=np.float64)[rsrc]
        rlane_row = np.where(realr, lidx(np.maximum(lane_orig, c0)), -1).astype(np.int32)
        agg_out = np.full(Lr // 2, -1, dtype=np.int32)
        agg_out[:ga.size] = np.arange(ga.size, dtype=np.int32)
        agg_out[ga.size:ga.size + partial.size] = ga.size + np.arange(partial.size, dtype=np.int32)
        hr = D.pack_sell(rlane_row, rptr, rcols, rvals, 1, n_own, agg_out=agg_out)
        self.restrict = D.SellDev(hr)
        self.restrict_width = int(hr.lane_len.max()) if hr.lane_len.size else 0
        self.n_partial = int(partial.size)
        # partial sends (grouped by owner, ascending aggregate) and receives
        self.psends = []
        for q in np.unique(aowner[partial]):
            sel = np.flatnonzero(aowner[partial] == q)
            self.psends.append((int(q), ga.size + int(sel[0]), ga.size + int(sel[-1]) + 1))
        self.precvs = []
        pidx = []
        off = 0
        for q in range(part.nranks):
            if q == rank:
                continue
            q0, q1 = part.rows(q)
            m = ga[(up >= q0) & (up < q1)]
            if m.size:
                self.precvs.append((q, off, off + m.size))
                pidx.append(m - self.ga0)
                off += m.size
        self.n_precv = off
        self.precv_idx = D.upload(np.concatenate(pidx).astype(np.int32)) if pidx else None
        self.aggp = D.upload(agg[cells].astype(np.int32))
        # halo of the level-0 x: packed sends (natural cell order), direct receives
        self.sends, self.recvs = halo_plan(part, self.windows, rank)
        pk = [loc_own[np.arange(a, e) - c0] for _, a, e in self.sends]
        self.pack_idx = D.upload(np.concatenate(pk).astype(np.int32)) if pk else None
        self.n_pack = int(sum(e - a for _, a, e in self.sends))
        # device work + descriptor
        self.b = D.zeros(max(n_own, 1))
        self.x = D.zeros(max(self.n_x, 1))
        self.tmp = D.zeros(max(n_own, 1))
        self.bc = D.zeros(max(self.n_agg + self.n_partial, 1))
        self.precv = D.zeros(max(self.n_precv, 1))
        self.packbuf = D.zeros(max(self.n_pack, 1))
        d = N.AmgLevel()
        d.n = n_own
        d.ncolors = ncol
        d.color_slices = N.p32(self.color_slices)
        d.color_rows = N.p32(self.color_rows)
        d.color_snapshot = self.snapshot.ctypes.data_as(N.u8p)
        d.smoother = self.smoother.desc
        d.diag = D.ptr(self.diag)
        d.restrict_op = self.restrict.desc
        d.restrict_width = self.restrict_width
        d.aggp = D.ptr(self.aggp)
        d.b, d.x, d.tmp = D.ptr(self.b), D.ptr(self.x), D.ptr(self.tmp)
        d.color_width = N.p32(self.color_width)
        self.desc = d

    def exchange_x(self, comm: SlabComm):
        if comm.size == 1:
            return
        if self.n_pack:
            N.check(N.lib().cprb_gather(self.n_pack, D.ptr(self.pack_idx), D.ptr(self.x), 1,
                                        D.ptr(self.packbuf), D.stream()))
        sends, off = [], 0
        for q, a, e in self.sends:
            sends.append((q, self.packbuf[off:off + (e - a)]))
            off += e - a
        c0, w0, n_own = self.c0, self.w0, self.n_own

        def hslot(a, e):
            s = n_own + (a - w0) if a < c0 else n_own + (c0 - w0) + (a - self.c1)
            return self.x[s:s + (e - a)]

        comm.exchange(sends, [(q, hslot(a, e)) for q, a, e in self.recvs])

    def combine_partials(self, comm: SlabComm):
        if comm.size == 1:
            return
        sends = [(q, self.bc[a:e]) for q, a, e in self.psends]
        recvs = [(q, self.precv[a:e]) for q, a, e in self.precvs]
        comm.exchange(sends, recvs)
        if self.n_precv:
            N.check(N.lib().cprb_scatter_add(self.n_precv, D.ptr(self.precv_idx),
                                             D.ptr(self.precv), D.ptr(self.bc), D.stream()))


def _sentinel_fill(n: int):
    t = D.torch()
    a = np.full(max(int(n), 1), int(_SENT_BITS), dtype=np.uint64).view(np.float64)
    return t.from_numpy(a).to("cuda")


class SlabBilu:
    """BILU(0) solves of this rank's slab (src/ilu.py:196-223) as part of ONE
    global wavefront: the wave plans are cut at the slab boundaries, each
    rank runs its own chunks, and the rows a neighbour reads are also stored
    into the neighbour's output array (peer memory over NVLink; the L solve
    feeds the next rank, the U solve the previous one).  The consumer polls
    its own memory exactly as for an in-chunk global dependency, so the
    arithmetic and results are those of the single-GPU solve."""

    def __init__(self, F, part: SlabPartition, rank: int, plan=None):
        from .ilu import WaveDev, wave_plan
        D.require_cuda()
        b = F.block_size
        self.b, self.rank = b, rank
        self.c0, self.c1 = part.rows(rank)
        if plan is None:
            cuts = np.asarray(part.cell0[1:-1], dtype=np.int64)
            hl, lslot = wave_plan(F.L, F.l_schedule, b, False, cuts=cuts)
            hu, uslot = wave_plan(F.U, F.u_schedule, b, True, uinv=F.u_diag_inv, cuts=cuts)
            plan = {"hl": hl, "hu": hu, "Lw": WaveDev(hl), "Uw": WaveDev(hu),
                    "l_slot": D.upload(lslot.astype(np.int32)),
                    "u_slot": D.upload(uslot.astype(np.int32)), "n": F.n}
        self.plan = plan
        hl, hu = plan["hl"], plan["hu"]
        self.len_l, self.len_u = max(hl["rhs_len"], 1), max(hu["rhs_len"], 1)
        self.rhs_l = D.zeros(self.len_l)
        self.rhs_u = D.zeros(self.len_u)
        self.zl_step = _sentinel_fill(self.len_l)
        self.y_step = _sentinel_fill(self.len_u)
        t = D.torch()
        self.tickets = t.zeros(8, dtype=t.int32, device="cuda")
        self.lr = tuple(int(v) for v in hl["chunk_range"][rank])
        self.ur = tuple(int(v) for v in hu["chunk_range"][rank])
        ml, mu = hl["mirror"][rank], hu["mirror"][rank]
        self.ml = D.upload(ml) if ml.size else None
        self.mu = D.upload(mu) if mu.size else None
        self.nml, self.nmu = int(ml.size), int(mu.size)
        self.peer_l = 0      # next rank's zl_step (L rows it reads)
        self.peer_u = 0      # previous rank's y_step (U rows it reads)
        self.desc = N.Bilu(plan["n"], b, N.Sell(), N.Sell(), 0, D.ptr(self.tickets), 1,
                           plan["Lw"].desc, plan["Uw"].desc, D.ptr(plan["l_slot"]), 0, 0,
                           D.ptr(plan["u_slot"]), 0, 0, self.len_l, self.len_u)

    def solve(self, mat: "SlabMatrix", zp_win, r, z):
        """z = Pi zp + BILU(r - A Pi zp) on this rank's rows (src/cpr.py:184-186)."""
        lib, st = N.lib(), D.stream()
        d = C.byref(self.desc)
        n_own = self.c1 - self.c0
        N.check(lib.cprb_stage2_residual_steps(mat.desc_ref(), d, self.c0, D.ptr(zp_win), D.ptr(r),
                                               D.ptr(self.rhs_l), D.ptr(self.zl_step),
                                               D.ptr(self.y_step), st))
        self.solve_steps(z, D.ptr(zp_win) + (self.c0 - mat.w0) * 8, n_own)

    def solve_steps(self, z, zp_own: int, n_own: int, st=None):
        self.solve_lower(n_own, st)
        self.solve_upper(z, zp_own, n_own, st)

    def solve_lower(self, n_own: int, st=None):
        """This rank's chunks of the L wavefront (polls the previous rank's
        rows in its own memory), then the L -> U permutation of its rows."""
        lib = N.lib()
        st = D.stream() if st is None else st
        d = C.byref(self.desc)
        N.check(lib.cprb_wave_solve_part(d, 0, self.lr[0], self.lr[1] - self.lr[0],
                                         D.ptr(self.rhs_l), D.ptr(self.zl_step), self.peer_l or None,
                                         D.ptr(self.tickets), st))
        N.check(lib.cprb_l_to_u_rows(d, self.c0, n_own, D.ptr(self.zl_step), D.ptr(self.rhs_u), st))

    def solve_upper(self, z, zp_own: int, n_own: int, st=None):
        """This rank's chunks of the U wavefront, z = Pi zp + y, re-arm."""
        lib = N.lib()
        st = D.stream() if st is None else st
        d = C.byref(self.desc)
        N.check(lib.cprb_wave_solve_part(d, 1, self.ur[0], self.ur[1] - self.ur[0],
                                         D.ptr(self.rhs_u), D.ptr(self.y_step), self.peer_u or None,
                                         D.ptr(self.tickets) + 4, st))
        N.check(lib.cprb_wave_combine_rows(d, self.c0, n_own, D.ptr(self.y_step), zp_own, D.ptr(z),
                                           st))
        self.rearm(st)

    def rearm(self, st=None):
        """Re-arm the slots the neighbours fill (after this rank consumed them;
        the next application's halo exchange orders the neighbours' stores
        after this)."""
        lib = N.lib()
        st = D.stream() if st is None else st
        if self.nml:
            N.check(lib.cprb_fill_sentinel_idx(self.nml, self.b, D.ptr(self.ml),
                                               D.ptr(self.zl_step), st))
        if self.nmu:
            N.check(lib.cprb_fill_sentinel_idx(self.nmu, self.b, D.ptr(self.mu),
                                               D.ptr(self.y_step), st))


def _link_peers(bilu: SlabBilu, comm: SlabComm):
    """Map the neighbours' output arrays (CUDA IPC; NVLink peer memory)."""
    from torch.multiprocessing.reductions import reduce_tensor
    mine = (reduce_tensor(bilu.zl_step), reduce_tensor(bilu.y_step))
    allh = [None] * comm.size
    comm.dist.all_gather_object(allh, mine, group=comm.group)
    bilu._peer_refs = []
    if comm.rank + 1 < comm.size:
        fn, args = allh[comm.rank + 1][0]
        t = fn(*args)
        bilu._peer_refs.append(t)
        bilu.peer_l = D.ptr(t)
    if comm.rank > 0:
        fn, args = allh[comm.rank - 1][1]
        t = fn(*args)
        bilu._peer_refs.append(t)
        bilu.peer_u = D.ptr(t)
    comm.dist.barrier(group=comm.group)


class SlabCpr:
    """Partitioned CPR application z = B r on this rank's rows
    (src/cpr.py:178-186)."""

    def __init__(self, B, part: SlabPartition, comm: SlabComm, bilu: str = "auto"):
        """bilu: "wave" = distributed wavefront (SlabBilu, peer memory),
        "replicated" = all-gather the stage-2 residual and solve the whole
        system on every rank, "auto" = wave on NCCL (one GPU per rank) and for
        one rank, replicated otherwise (ranks sharing a GPU: tests)."""
        D.require_cuda()
        h = B.pressure_solver
        self.cycle = h.params.cycle
        if len(h.levels) < 2:
            raise NotImplementedError("the slab-partitioned path needs at least two AMG levels")
        self.part, self.comm = part, comm
        rank = comm.rank
        self.mat = SlabMatrix(B.A, part, rank)           # stage 2 (build-time matrix)
        self.b = self.mat.b
        self.l0 = SlabLevel0(h, part, rank)
        if (self.l0.w0, self.l0.w1) != (self.mat.w0, self.mat.w1):
            raise NotImplementedError("pressure and block windows differ")
        self.n1 = int(h.levels[1].A.nrows)
        self.gather1 = _Gatherer(self.l0.agg_counts)
        self.b1 = D.zeros(self.n1)
        self.e1 = D.zeros(self.n1)
        self.sub = None
        self.kfull = None
        if rank == 0:
            if self.cycle == "k":
                # K: the coarse correction of level 0 is the Krylov-wrapped
                # recursion from level 1 (src/amg.py:256-263), on rank 0
                self.kfull = DeviceAmg(h, 1)
                if self.kfull.kdesc() is None:
                    raise NotImplementedError("slab-partitioned K-cycle needs the device K-cycle")
                self.perm1 = D.upload(self.kfull.perms[1].astype(np.int32))
            else:
                sub = AmgHierarchy(h.levels[1:], h.coarsest_lu, h.params, symmetric=h.symmetric)
                self.sub = DeviceAmg(sub, 1)
        if bilu == "auto":
            bilu = "wave" if (comm.nccl or comm.size == 1) else "replicated"
        self.bilu_mode = bilu
        nb = B.A.nrows
        if bilu == "wave":
            self.sbilu = SlabBilu(B.relaxation, part, rank)
            if comm.size > 1:
                _link_peers(self.sbilu, comm)
        else:
            self.bilu = B.relaxation.device()
        self.zp = D.zeros(self.mat.win_len)
        if bilu != "wave":
            self.r2 = D.zeros(max(self.mat.n_own * self.b, 1))
            self.r2_full = D.zeros(nb * self.b)
            self.y_full = D.zeros(nb * self.b)
            self.gather_fine = _Gatherer(np.diff(part.cell0) * self.b)

    def apply(self, r, z):
        """r: own rows (3 per cell); z: own rows (any contiguous view)."""
        lib, st, comm, L0 = N.lib(), D.stream(), self.comm, self.l0
        d = C.byref(L0.desc)
        zp_own = D.ptr(self.zp) + (self.mat.c0 - self.mat.w0) * 8
        # level 0: zero-guess forward pass, halo refreshed after every colour
        for k in range(L0.ncolors):
            N.check(lib.cprb_pgs_scm_color(d, k, D.ptr(L0.b), D.ptr(L0.x), 1, D.ptr(r), self.b,
                                           D.ptr(L0.perm_local), None, st))
            L0.exchange_x(comm)
        N.check(lib.cprb_resid_restrict(d, D.ptr(L0.b), D.ptr(L0.x), D.ptr(L0.bc), st))
        L0.combine_partials(comm)
        # levels >= 1 agglomerated on rank 0
        self.gather1(comm, L0.bc, L0.n_agg, self.b1, root_only=True)
        if self.sub is not None:
            N.check(lib.cprb_amg_cycle(C.byref(self.sub.desc), D.ptr(self.b1), D.ptr(self.e1), st))
        elif self.kfull is not None:
            N.check(lib.cprb_kcycle_correction(C.byref(self.kfull.kdesc()), 1, D.ptr(self.perm1),
                                               D.ptr(self.b1), D.ptr(self.e1), st))
        comm.broadcast(self.e1, 0)
        N.check(lib.cprb_prolong(d, D.ptr(self.e1), D.ptr(L0.x), st))
        L0.exchange_x(comm)
        for t in range(L0.ncolors):
            k = L0.ncolors - 1 - t
            N.check(lib.cprb_pgs_scm_color(d, k, D.ptr(L0.b), D.ptr(L0.x), 0, None, 0,
                                           D.ptr(L0.perm_local), zp_own, st))
            if t + 1 < L0.ncolors:
                L0.exchange_x(comm)
        self.mat.exchange(comm, self.zp, 1)
        if self.bilu_mode == "wave":
            # stage 2 + the slab's share of the global BILU wavefront
            self.sbilu.solve(self.mat, self.zp, r, z)
            return
        # stage 2: r2 = r - A Pi zp on own rows; BILU is a global wavefront
        n_loc = self.mat.n_own * self.b
        N.check(lib.cprb_stage2_residual(self.mat.desc_ref(), self.b, D.ptr(self.zp), D.ptr(r),
                                         D.ptr(self.r2), st))
        self.gather_fine(comm, self.r2, n_loc, self.r2_full)
        self.bilu.apply(self.r2_full, self.y_full)
        c0 = self.mat.c0
        N.check(lib.cprb_cpr_combine(self.mat.n_own, self.b, zp_own,
                                     D.ptr(self.y_full) + c0 * self.b * 8, D.ptr(z), st))


class _SegDot:
    """GPU-count-invariant dot products (csrc/slab.cu)."""

    def __init__(self, part: SlabPartition, comm: SlabComm, b: int, rank: int):
        self.comm = comm
        self.seg_len = part.seg_cells * b
        self.nseg = part.nseg
        self.nloc = int(part.seg0[rank + 1] - part.seg0[rank])
        cap, smap = part.seg_map()
        self.cap = cap
        self.partials = D.zeros(cap)
        self.full = D.zeros(part.nranks * cap)
        self.map = D.upload(smap) if comm.size > 1 else None
        self.out = D.zeros(64)

    def stage(self, n, w, vprev, hprev, vdot, hout, sq: int):
        lib, st = N.lib(), D.stream()
        N.check(lib.cprb_seg_partials(n, self.seg_len, D.ptr(w), D.ptr(vprev), hprev, D.ptr(vdot),
                                      D.ptr(self.partials), st))
        if self.comm.size > 1:
            self.comm.allgather(self.partials, self.full)
            src = self.full
        else:
            src = self.partials
        N.check(lib.cprb_seg_finish(self.nseg, D.ptr(src), D.ptr(self.map), hout, sq, st))

    def dot(self, x, y) -> float:
        self.stage(x.shape[0], x, None, None, y, D.ptr(self.out), 0)
        return float(self.out[0].item())


def gmres_solve_slab(A, b_local, x0_local, B, params: GmresParams | None = None,
                     comm: SlabComm | None = None, part: SlabPartition | None = None,
                     history: bool = False, cpr: SlabCpr | None = None) -> GmresResult:
    """Restarted right-preconditioned GMRES (src/cpr.py:231-316) on this
    rank's rows: b_local / x0_local / the returned x are the rows
    part.rows(rank) (b values per cell).  Every rank gets the same outer /
    inner counts, history and convergence decision."""
    params = params or GmresParams()
    comm = comm or SlabComm()
    bsz = _bsize(A)
    part = part or SlabPartition(A.nrows, comm.size)
    if part.nranks != comm.size:
        raise ValueError("partition and communicator sizes differ")
    lib, st, t = N.lib(), D.stream(), D.torch()
    M = _slab_matrix(A, part, comm.rank)
    bd, kind = D.to_device(b_local)
    n = M.n_own * bsz
    if bd.shape[0] != n:
        raise ValueError(f"dimension mismatch: rank {comm.rank} owns {n} rows, rhs has {bd.shape[0]}")
    P = cpr if cpr is not None else (_slab_cpr(B, part, comm) if B is not None else None)
    dots = _SegDot(part, comm, bsz, comm.rank)
    m = params.m
    V = t.empty((m + 1, max(n, 1)), dtype=t.float64, device="cuda")
    hcol = t.zeros(m + 2, dtype=t.float64, device="cuda")
    hcol_host = t.zeros(m + 2, dtype=t.float64).pin_memory()
    xw = D.zeros(M.win_len * bsz)
    if x0_local is not None:
        M.interior(xw, bsz).copy_(D.to_device(x0_local)[0])
    zw = D.zeros(M.win_len * bsz)
    r = D.empty(max(n, 1))
    u = D.empty(max(n, 1))

    def residual(xwin):
        M.exchange(comm, xwin, bsz)
        N.check(lib.cprb_residual(M.desc_ref(), bsz, D.ptr(bd), D.ptr(xwin), D.ptr(r), None, st))
        return float(np.sqrt(dots.dot(r[:n], r[:n])))

    def precondition(v):
        zi = M.interior(zw, bsz)
        if P is None:
            zi.copy_(v)
        else:
            P.apply(v, zi)
        return zi

    beta0 = residual(xw)
    hist: list = []
    if not np.isfinite(beta0):
        raise FloatingPointError("non-finite initial residual in gmres_solve")
    if beta0 == 0.0:
        return GmresResult(D.from_device(M.interior(xw, bsz).clone(), kind), 0, 0, True, 0.0, hist)
    inner_total, converged, rel, outer = 0, False, 1.0, 0
    beta = beta0
    for outer in range(1, params.max_restarts + 1):
        if outer > 1:
            beta = float(np.sqrt(dots.dot(r[:n], r[:n])))
        if beta == 0.0:
            converged = True
            break
        N.check(lib.cprb_div_host(n, D.ptr(r), beta, D.ptr(V[0]), st))
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = beta
        j_used, shrink = 0, None
        for j in range(m):
            zj = precondition(V[j][:n])
            M.exchange(comm, zw, bsz)
            N.check(lib.cprb_spmv(M.desc_ref(), bsz, D.ptr(zw), D.ptr(V[j + 1]), None, st))
            w = V[j + 1]
            for i in range(j + 2):
                vprev = V[i - 1] if i > 0 else None
                hprev = D.ptr(hcol) + 8 * (i - 1) if i > 0 else None
                vdot = V[i] if i <= j else None
                dots.stage(n, w, vprev, hprev, vdot, D.ptr(hcol) + 8 * i, 1 if i == j + 1 else 0)
            N.check(lib.cprb_div_if_nonzero(n, D.ptr(w), D.ptr(hcol) + 8 * (j + 1), st))
            hcol_host[:j + 2].copy_(hcol[:j + 2], non_blocking=True)
            t.cuda.current_stream().synchronize()
            col = hcol_host[:j + 2].numpy()
            if not np.all(np.isfinite(col)):
                raise FloatingPointError("non-finite Krylov vector in gmres_solve")
            H[:j + 2, j] = col
            j_used = j + 1
            inner_total += 1
            breakdown = H[j + 1, j] == 0.0
            for i in range(j):
                tt = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = tt
            denom = float(np.hypot(H[j, j], H[j + 1, j]))
            if denom == 0.0:
                cs[j], sn[j] = 1.0, 0.0
            else:
                cs[j], sn[j] = H[j, j] / denom, H[j + 1, j] / denom
            H[j, j] = denom
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            if history:
                hist.append(abs(g[j + 1]) / beta0)
            if breakdown:
                shrink = j + 1
                break
            if abs(g[j + 1]) < params.tol * beta0:
                break
        y = _solve_upper(H[:j_used, :j_used], g[:j_used])
        yd = t.from_numpy(np.ascontiguousarray(y, dtype=np.float64)).to("cuda")
        N.check(lib.cprb_gemv_t(n, j_used, D.ptr(V), V.shape[1], D.ptr(yd), D.ptr(u), st))
        zi = precondition(u[:n])
        xn = D.zeros(M.win_len * bsz)
        N.check(lib.cprb_add(n, D.ptr(M.interior(xw, bsz)), D.ptr(zi),
                             D.ptr(M.interior(xn, bsz)), st))
        xw = xn
        rel = residual(xw) / beta0
        if not np.isfinite(rel):
            raise FloatingPointError("non-finite residual in gmres_solve (divergence)")
        if history:
            hist.append(("explicit", rel))
        if shrink is not None:
            m = shrink
        if rel < params.tol:
            converged = True
            break
    return GmresResult(D.from_device(M.interior(xw, bsz).clone(), kind), outer, inner_total,
                       converged, rel, hist)


def _slab_matrix(A, part: SlabPartition, rank: int) -> SlabMatrix:
    key = (part.ncells, part.nranks, part.seg_cells, rank)
    cache = getattr(A, "_cprb_slab", None)
    if cache is None or cache[0] != key:
        cache = (key, SlabMatrix(A, part, rank))
        try:
            object.__setattr__(A, "_cprb_slab", cache)
        except (AttributeError, TypeError):
            pass
    return cache[1]


def _slab_cpr(B, part: SlabPartition, comm: SlabComm) -> SlabCpr:
    key = (part.ncells, part.nranks, part.seg_cells, comm.rank)
    cache = getattr(B, "_cprb_slab", None)
    if cache is None or cache[0] != key:
        cache = (key, SlabCpr(B, part, comm))
        try:
            object.__setattr__(B, "_cprb_slab", cache)
        except (AttributeError, TypeError):
            pass
    return cache[1]


def gather_rows(local, part: SlabPartition, comm: SlabComm, b: int):
    """All ranks' rows, packed in rank order (tests, result collection)."""
    g = _Gatherer(np.diff(part.cell0) * b)
    out = D.zeros(part.ncells * b)
    g(comm, local, local.shape[0], out)
    return out
