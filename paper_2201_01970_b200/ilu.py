"""Block ILU(0) (drop-in for cprkit.ilu).

SETUP (host C++): the IKJ factorization restricted to the pattern, pivot
inversion with the reference's perturbation fallback, level schedules
(src/ilu.py:38-193).  SOLVE (device): sync-free level-ordered L and U
substitutions (csrc/bilu.cu), bitwise equal to the reference's
level-scheduled solve for the same factors.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import os

import numpy as np

from . import _native as N
from . import device as D
from .sparse import BlockCsrMatrix, CsrMatrix, to_block

__all__ = ["BiluFactors", "DeviceBiluFactors", "LevelSchedule", "bilu0_factorize",
           "bilu0_factorize_device", "level_schedule", "bilu_apply"]


@dataclass
class LevelSchedule:
    levels: list

    @property
    def n_levels(self) -> int:
        return len(self.levels)


def _levels_from(level: np.ndarray, nlev: int) -> list:
    order = np.argsort(level, kind="stable")
    counts = np.bincount(level, minlength=nlev + 1)[1:]
    bounds = np.concatenate([[0], np.cumsum(counts)])
    return [order[bounds[i]:bounds[i + 1]].astype(np.int64) for i in range(nlev)]


def level_schedule(T) -> LevelSchedule:
    """level(i) = 1 + max level of the in-pattern predecessors (src/ilu.py:38-59)."""
    n = T.nrows
    ptr = np.ascontiguousarray(T.row_ptr, dtype=np.int64)
    cols = np.ascontiguousarray(T.col_idx, dtype=np.int64)
    level = np.zeros(max(n, 1), dtype=np.int64)
    nl = np.zeros(1, dtype=np.int64)
    N.check(N.lib().cprb_level_schedule(n, N.p64(ptr), N.p64(cols if cols.size else np.zeros(1, np.int64)),
                                        N.p64(level), N.p64(nl)))
    return LevelSchedule(_levels_from(level[:n], int(nl[0])) if n else [np.zeros(0, np.int64)])


@dataclass
class BiluFactors:
    """L (unit lower) and U (upper) on A's pattern, inverted U diagonal
    (src/ilu.py:110-131)."""

    L: BlockCsrMatrix
    U: BlockCsrMatrix
    block_size: int
    u_diag_inv: np.ndarray
    l_schedule: LevelSchedule
    u_schedule: LevelSchedule
    _dev: object = field(default=None, repr=False)

    @property
    def n(self) -> int:
        return self.L.nrows

    def device(self, use_wave: bool = True) -> "DeviceBilu":
        if self._dev is None or self._dev.use_wave != (use_wave and self.n > 0):
            self._dev = DeviceBilu(self, use_wave)
        return self._dev


def bilu0_factorize(A) -> BiluFactors:
    """ILU(0) with no fill (src/ilu.py:150-193); a singular pivot with a nonzero
    Frobenius norm is perturbed by 1e-8*||B||_F*I with a RuntimeWarning."""
    if isinstance(A, CsrMatrix) or np.ndim(getattr(A, "values", None)) == 1:
        A = to_block(A if isinstance(A, CsrMatrix) else CsrMatrix(A.nrows, A.ncols, A.row_ptr,
                                                                     A.col_idx, A.values))
    n, b = A.nrows, A.block_size
    if A.nrows != A.ncols:
        raise ValueError("factorization needs a square matrix")
    ptr = np.ascontiguousarray(A.row_ptr, dtype=np.int64)
    cols = np.ascontiguousarray(A.col_idx, dtype=np.int64)
    vals = np.ascontiguousarray(A.values, dtype=np.float64).copy()
    uinv = np.zeros((n, b, b))
    pert = np.zeros(max(n, 1), dtype=np.int64)
    npert = np.zeros(1, dtype=np.int64)
    N.check(N.lib().cprb_bilu0_factorize(n, b, N.p64(ptr), N.p64(cols if cols.size else np.zeros(1, np.int64)),
                                         N.pf64(vals.reshape(-1) if vals.size else np.zeros(1)),
                                         N.pf64(uinv.reshape(-1) if uinv.size else np.zeros(1)),
                                         N.p64(pert), N.p64(npert)))
    for row in pert[:int(npert[0])]:
        N.warn(f"bilu0: perturbing singular pivot block at row {int(row)}", RuntimeWarning, 2)
    return _factors_from(n, b, ptr, cols, vals, uinv)


def _factors_from(n, b, ptr, cols, vals, uinv) -> BiluFactors:
    """Split the in-place factored values on A's pattern into L (strict
    lower + identity diagonal) and U (diagonal + strict upper)."""
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(ptr))
    lower = cols < rows
    # L: strict lower then the identity diagonal (already column-sorted per row)
    nlow = np.bincount(rows[lower], minlength=n)
    lptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(nlow + 1, out=lptr[1:])
    lcols = np.empty(lptr[-1], dtype=np.int64)
    lvals = np.empty((lptr[-1], b, b))
    diag_pos = lptr[1:] - 1
    is_diag = np.zeros(lptr[-1], dtype=bool)
    is_diag[diag_pos] = True
    lcols[~is_diag] = cols[lower]
    lvals[~is_diag] = vals[lower]
    lcols[diag_pos] = np.arange(n)
    lvals[diag_pos] = np.eye(b)
    L = BlockCsrMatrix(b, n, n, lptr, lcols, lvals)
    uptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows[~lower], minlength=n), out=uptr[1:])
    U = BlockCsrMatrix(b, n, n, uptr, cols[~lower].copy(), vals[~lower].copy())
    return BiluFactors(L, U, b, uinv, level_schedule(L), level_schedule(U))


class DeviceBiluFactors(BiluFactors):
    """BILU(0) factored ON THE DEVICE (csrc/factor.cu): the factors stay in
    HBM on A's pattern; the stencil plan of the solves is packed from them
    on the device.  The host view (L, U, u_diag_inv, schedules -- the
    reference's BiluFactors fields) is downloaded on first access and is
    bitwise the host factorization's."""

    def __init__(self, n, b, ptr, cols, csr_d, vals_d, uinv_d):
        self._n, self._b = int(n), int(b)
        self.ptr, self.cols = ptr, cols
        self.csr_d = csr_d            # (row_ptr, col_idx) on the device
        self.vals_d, self.uinv_d = vals_d, uinv_d
        self._host = None
        self._dev = None

    def _h(self) -> BiluFactors:
        if self._host is None:
            vals = self.vals_d.cpu().numpy().reshape(-1, self._b, self._b)
            uinv = self.uinv_d.cpu().numpy().reshape(-1, self._b, self._b)
            self._host = _factors_from(self._n, self._b, self.ptr, self.cols, vals, uinv)
        return self._host

    L = property(lambda self: self._h().L)
    U = property(lambda self: self._h().U)
    u_diag_inv = property(lambda self: self._h().u_diag_inv)
    l_schedule = property(lambda self: self._h().l_schedule)
    u_schedule = property(lambda self: self._h().u_schedule)
    block_size = property(lambda self: self._b)

    @property
    def n(self) -> int:
        return self._n

    def __repr__(self):
        return f"DeviceBiluFactors(n={self._n}, block_size={self._b})"

    def stencil_device(self):
        """Stencil plan (as stencil_plan) packed on the device, or None."""
        if self._b != 3:
            return None
        dims = np.zeros(3, dtype=np.int64)
        if not N.lib().cprb_detect_stencil(self._n, N.p64(self.ptr), N.p64(self.cols), N.p64(dims)):
            return None
        nx, ny, nz = (int(v) for v in dims)
        if nx > 32 * STENCIL_SMAX:
            return None
        doff, P = _stencil_offsets(nx, ny)
        t = D.torch()
        lrec = t.zeros(nz * P * 27, dtype=t.float64, device="cuda")
        urec = t.zeros(nz * P * 37, dtype=t.float64, device="cuda")
        slot = t.empty(self._n, dtype=t.int32, device="cuda")
        doff_d = D.upload(doff.astype(np.int32))
        N.check(N.lib().cprb_stencil_pack(self._n, nx, ny, P, D.ptr(doff_d), D.ptr(self.csr_d[0]),
                                          D.ptr(self.csr_d[1]), D.ptr(self.vals_d),
                                          D.ptr(self.uinv_d), D.ptr(lrec), D.ptr(urec),
                                          D.ptr(slot), D.stream()))
        return {"nx": nx, "ny": ny, "nz": nz, "S": (nx + 31) // 32, "D": nx + ny - 1, "P": P,
                "doff": doff_d, "lrec": lrec, "urec": urec, "slot": slot, "len": 3 * nz * P}


def bilu0_factorize_device(A, dev_csr=None) -> DeviceBiluFactors:
    """src/ilu.py:150-193 on the device (3x3 blocks): the factorization runs
    level by level over the strict-lower dependency schedule
    (csrc/factor.cu), bitwise the host C++ factorization; errors and the
    perturbation warnings are the host path's.  dev_csr = (row_ptr,
    col_idx, values) already in HBM (e.g. from the device generator)."""
    b = int(getattr(A, "block_size", 1))
    n = A.nrows
    if A.nrows != A.ncols:
        raise ValueError("factorization needs a square matrix")
    ptr = np.ascontiguousarray(A.row_ptr, dtype=np.int64)
    cols = np.ascontiguousarray(A.col_idx, dtype=np.int64)
    level = np.zeros(max(n, 1), dtype=np.int64)
    nl = np.zeros(1, dtype=np.int64)
    N.check(N.lib().cprb_lower_level_schedule(n, N.p64(ptr), N.p64(cols if cols.size else level),
                                              N.p64(level), N.p64(nl)))
    nlev = int(nl[0])
    order = np.argsort(level[:n], kind="stable").astype(np.int32)
    lptr = np.zeros(nlev + 1, dtype=np.int64)
    np.cumsum(np.bincount(level[:n], minlength=nlev + 1)[1:], out=lptr[1:])
    t = D.torch()
    if dev_csr is None:
        dev_csr = (D.upload(ptr), D.upload(cols),
                   D.upload(np.ascontiguousarray(A.values, dtype=np.float64).reshape(-1)))
    vals_d = dev_csr[2].clone()
    uinv_d = t.zeros(n * b * b, dtype=t.float64, device="cuda")
    err = t.zeros(4, dtype=t.int32, device="cuda")
    pert = t.zeros(max(n, 1), dtype=t.int64, device="cuda")
    rows_d = D.upload(order)
    N.check(N.lib().cprb_bilu0_factorize_device(n, b, D.ptr(dev_csr[0]), D.ptr(dev_csr[1]),
                                                D.ptr(vals_d), D.ptr(uinv_d), D.ptr(rows_d),
                                                N.p64(lptr), nlev, D.ptr(err), D.ptr(pert),
                                                D.stream()))
    e = err.cpu().numpy()
    bad_diag, bad_piv = int(e[1]), int(e[0])
    if min(bad_diag, bad_piv) < 2**31 - 1:
        if bad_diag < bad_piv:
            raise ValueError(f"diagonal block missing in row {bad_diag}")
        raise np.linalg.LinAlgError(f"singular pivot block at row {bad_piv}")
    for row in np.sort(pert[:int(e[2])].cpu().numpy()):
        N.warn(f"bilu0: perturbing singular pivot block at row {int(row)}", RuntimeWarning, 2)
    return DeviceBiluFactors(n, b, ptr, cols, dev_csr[:2], vals_d, uinv_d)


def _strict(T: BlockCsrMatrix):
    rows = np.repeat(np.arange(T.nrows, dtype=np.int64), np.diff(T.row_ptr))
    off = rows != T.col_idx
    ptr = np.zeros(T.nrows + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows[off], minlength=T.nrows), out=ptr[1:])
    return ptr, T.col_idx[off], T.values[off]


def _level_sell(T: BlockCsrMatrix, sched: LevelSchedule, b: int, uinv=None):
    ptr, cols, vals = _strict(T)
    lanes = [D.pad_lanes(lv.astype(np.int32)) for lv in sched.levels if lv.shape[0]]
    lane_row = np.concatenate(lanes) if lanes else np.zeros(0, dtype=np.int32)
    L = lane_row.shape[0]
    real = lane_row >= 0
    lr = lane_row.astype(np.int64)
    lens = np.zeros(L, dtype=np.int64)
    lens[real] = np.diff(ptr)[lr[real]]
    lane_ptr = np.zeros(L + 1, dtype=np.int64)
    np.cumsum(lens, out=lane_ptr[1:])
    nnz = int(lane_ptr[-1])
    lane_of = np.repeat(np.arange(L, dtype=np.int64), lens)
    src = ptr[lr[lane_of]] + (np.arange(nnz, dtype=np.int64) - lane_ptr[lane_of])
    h = D.pack_sell(lane_row, lane_ptr, cols[src], vals[src] if b > 1 else vals[src].reshape(-1),
                    b, T.nrows)
    ui = None
    if uinv is not None:
        bb = b * b
        ui = np.zeros(max(L * bb, 1))
        l_idx = np.flatnonzero(real)
        s, ln = l_idx // 32, l_idx % 32
        e = np.arange(bb)
        idx = (s[:, None] * bb + e[None, :]) * 32 + ln[:, None]
        ui[idx.reshape(-1)] = uinv.reshape(-1, bb)[lr[real]].reshape(-1)
    return h, ui


WAVE_WMAX = 128         # rows per step == consumer threads per CTA (csrc/wave.cu)
WAVE_DINT = 3           # dependencies at most this many steps back are read from shared memory
WAVE_KMAX = 3           # steps with at most this many dependencies per row are TMA-streamed
WAVE_BANDS = int(os.environ.get("CPRB_WAVE_BANDS", "2"))  # dependency bandwidths (xy-planes) per chunk


def _round16(x):
    return (x + 15) // 16 * 16


def wave_plan(T: BlockCsrMatrix, sched: LevelSchedule, b: int, upper: bool, uinv=None,
              aux_slot=None, nchunk_min: int = 148, cuts=None):
    """Chunked-wavefront plan of a strict triangular factor (see cprb_wave in
    include/cpr_b200.h).  Returns (host arrays dict, row -> rhs slot).

    cuts (slab-partitioned solve): sorted row indices where a rank's slab
    starts.  Chunks never straddle a cut, rows read across a cut carry the
    REMOTE bit (their owner also stores them into the reader's memory), and
    the dict gains per-rank chunk ranges and the output slots each rank
    receives from its neighbour ("mirror")."""
    ptr, cols, vals = _strict(T)
    n = T.nrows
    bb = b * b
    vals = np.asarray(vals, dtype=np.float64).reshape(-1, bb)
    lens = np.diff(ptr)
    rows_of = np.repeat(np.arange(n, dtype=np.int64), lens)
    level = np.zeros(n, dtype=np.int64)
    for li, lv in enumerate(sched.levels):
        level[lv] = li
    bw = int(np.abs(rows_of - cols).max()) if cols.size else 1
    R = max(WAVE_BANDS * bw, -(-n // nchunk_min), 1)
    pos = (n - 1 - np.arange(n)) if upper else np.arange(n)
    if cuts is None:
        chunk = pos // R
    else:
        cuts = np.asarray(cuts, dtype=np.int64)
        cut_pos = np.sort((n - cuts) if upper else cuts)
        starts = np.concatenate([[0], cut_pos])
        ends = np.concatenate([cut_pos, [n]])
        bnd = np.concatenate([np.arange(a0, e0, R) for a0, e0 in zip(starts, ends) if e0 > a0])
        chunk = np.searchsorted(bnd, pos, side="right") - 1
    order = np.lexsort((np.arange(n), level, chunk))     # rows by (chunk, level, index)
    ch_s, lv_s = chunk[order], level[order]
    newg = np.ones(n, dtype=bool)
    newg[1:] = (np.diff(ch_s) != 0) | (np.diff(lv_s) != 0)
    gstart = np.flatnonzero(newg)
    gsize = np.diff(np.append(gstart, n))
    gid = np.repeat(np.arange(gstart.shape[0]), gsize)
    Kg = np.maximum.reduceat(lens[order], gstart) if n else np.zeros(0, np.int64)
    cap = np.full(gstart.shape[0], WAVE_WMAX, dtype=np.int64)
    nsub = -(-gsize // cap)
    gstep0 = np.zeros(gstart.shape[0] + 1, dtype=np.int64)
    np.cumsum(nsub, out=gstep0[1:])
    pin = np.arange(n) - gstart[gid]
    sub = pin // cap[gid]
    step_of_sorted = gstep0[gid] + sub
    p_sorted = pin - sub * cap[gid]
    nsteps = int(gstep0[-1])
    row_step = np.empty(n, dtype=np.int64)
    row_pos = np.empty(n, dtype=np.int64)
    row_step[order] = step_of_sorted
    row_pos[order] = p_sorted
    step_w = np.bincount(step_of_sorted, minlength=nsteps)
    step_k = np.zeros(nsteps, dtype=np.int64)
    np.maximum.at(step_k, step_of_sorted, lens[order])
    step_chunk = np.zeros(nsteps, dtype=np.int64)
    step_chunk[step_of_sorted] = ch_s
    nchunks = int(chunk.max()) + 1 if n else 0
    chunk_step = np.searchsorted(step_chunk, np.arange(nchunks + 1)).astype(np.int32)
    # warp-sliced records: the rows of a step are cut into 32-row warp slices;
    # slice q of step s is one contiguous sub-record
    #   int32 rows[32], lens[32], aux[32], codes[K][32];
    #   f64 vals[K][b*b][32]; (upper) f64 uinv[b*b][32]
    # so each consumer warp streams exactly its own rows (csrc/wave.cu).
    nwarp = (step_w + 31) // 32
    sub = 32 * (12 + 4 * step_k) + 8 * 32 * step_k * bb + (8 * 32 * bb if upper else 0)
    sbytes = nwarp * sub
    soff = np.zeros(nsteps + 1, dtype=np.int64)
    np.cumsum(sbytes, out=soff[1:])
    rbytes = np.array([_round16(int(w) * b * 8) for w in step_w], dtype=np.int64) \
        if nsteps < 4096 else (step_w * b * 8 + 15) // 16 * 16
    roff = np.zeros(nsteps + 1, dtype=np.int64)
    np.cumsum(rbytes // 8, out=roff[1:])
    roff_pad = int(roff[-1]) + 32 * b              # a partial warp slice may read past the end
    # rows some dependant polls from global memory (another chunk, or more
    # than WAVE_DINT steps later): only these are published by the kernel
    e_diff = row_step[rows_of] - row_step[cols]
    e_int = (chunk[cols] == chunk[rows_of]) & (e_diff >= 1) & (e_diff <= WAVE_DINT)
    exported = np.zeros(n, dtype=bool)
    exported[cols[~e_int]] = True
    stream = np.zeros(max(int(soff[-1]), 16), dtype=np.uint8)
    I = stream.view(np.int32)
    F = stream.view(np.float64)
    st = row_step
    rec = soff[st] + (row_pos // 32) * sub[st]          # byte offset of the row's warp slice
    ln = row_pos % 32
    I[rec // 4 + ln] = np.arange(n)                                       # rows
    remote = np.zeros(n, dtype=bool)
    if cuts is not None:
        owner = np.searchsorted(cuts, np.arange(n), side="right")
        cross = owner[cols] != owner[rows_of]
        remote[cols[cross]] = True
        want = owner[cols[cross]] + (-1 if upper else 1)
        if not np.array_equal(owner[rows_of[cross]], want):
            raise NotImplementedError("slab partition: a factor row is read beyond the "
                                      "neighbouring slab (slabs thinner than the bandwidth)")
    I[rec // 4 + 32 + ln] = (lens | (exported.astype(np.int64) << 30)
                             | (remote.astype(np.int64) << 29))   # lens | export | remote
    aux = np.zeros(n, dtype=np.int64) if aux_slot is None else aux_slot
    I[rec // 4 + 64 + ln] = aux                                           # aux (next rhs slot)
    # entries
    ent = np.arange(cols.shape[0], dtype=np.int64)
    m = ent - ptr[rows_of]
    ri = rows_of
    dep = cols
    diff = row_step[ri] - row_step[dep]
    internal = (chunk[dep] == chunk[ri]) & (diff >= 1) & (diff <= WAVE_DINT)
    slot = (diff - 1) * WAVE_WMAX + row_pos[dep]
    # global dependencies are polled in the producer's step-ordered output
    # (the kernel publishes rows contiguously in rhs-slot order)
    pslot = roff[row_step] + row_pos * b
    code = np.where(internal, -(slot + 1), pslot[dep])
    e_st = row_step[ri]
    e_rec = rec[ri]
    e_ln = ln[ri]
    I[e_rec // 4 + 96 + 32 * m + e_ln] = code
    vbase = (e_rec + 32 * (12 + 4 * step_k[e_st])) // 8
    e_idx = np.arange(bb, dtype=np.int64)
    F[(vbase + (m * bb) * 32 + e_ln)[:, None] + e_idx[None, :] * 32] = vals
    if upper:
        ub = (rec + 32 * (12 + 4 * step_k[st]) + 8 * 32 * step_k[st] * bb) // 8
        F[(ub + ln)[:, None] + e_idx[None, :] * 32] = \
            np.asarray(uinv, dtype=np.float64).reshape(n, bb)
    rhs_slot = roff[st] + row_pos * b
    fast = step_k <= WAVE_KMAX
    host = dict(nchunks=nchunks, nsteps=nsteps, stage_max=int(sub[fast].max(initial=16)),
                rhs_max=32 * b * 8, chunk_step=chunk_step,
                step_off=soff[:-1].astype(np.int64), step_bytes=sub.astype(np.int32),
                step_w=step_w.astype(np.int32), step_k=step_k.astype(np.int32),
                rhs_off=roff[:-1].astype(np.int64), rhs_bytes=rbytes.astype(np.int32),
                stream=stream, rhs_len=roff_pad, chunk_rows=R)
    if cuts is not None:
        nr = cuts.shape[0] + 1
        rb = np.concatenate([[0], cuts, [n]])
        rng_ = np.zeros((nr, 2), dtype=np.int64)
        mirror = []
        for q in range(nr):
            a0, e0 = int(rb[q]), int(rb[q + 1])
            if e0 > a0:
                ch = chunk[a0:e0]
                rng_[q] = (int(ch.min()), int(ch.max()) + 1)
            # slots this rank's rows poll that the neighbour produces
            mine = (owner[rows_of] == q) & cross
            src = np.unique(cols[mine])
            mirror.append(rhs_slot[src].astype(np.int32))
        host["chunk_range"] = rng_
        host["mirror"] = mirror
    return host, rhs_slot


STENCIL_SMAX = 4   # x-segments of 32 lanes per warp (csrc/stencil.cu): nx <= 128


def _stencil_offsets(nx, ny):
    """Padded offsets of the anti-diagonals d = ix + iy of one xy-plane
    (widths rounded up to even: 16-byte TMA granules) and the plane size."""
    Dn = nx + ny - 1
    d = np.arange(Dn, dtype=np.int64)
    lo = np.maximum(0, d - (ny - 1))
    hi = np.minimum(nx - 1, d)
    w = hi - lo + 1
    wp = w + (w & 1)
    doff = np.zeros(Dn + 1, dtype=np.int64)
    np.cumsum(wp, out=doff[1:])
    return doff, int(doff[-1])


def stencil_plan(F: BiluFactors):
    """Structured-grid plan of the BILU(0) solves (csrc/stencil.cu), or None.

    Applies when the factors are those of a natural-ordered nx x ny x nz
    7-point grid with every in-range neighbour present (the reference
    generator's Jacobians, src/problems.py:57-155): the strict-lower pattern
    of row (ix, iy, iz) is exactly {-z, -y, -x} in range, the strict-upper
    pattern {+x, +y, +z}.  Rows are laid out per xy-plane in anti-diagonal
    order d = ix + iy (diagonal blocks padded to an even width), each
    row's factor record contiguous (row-major): L fields m*9 + e (m: -z, -y,
    -x), U fields m*9 + e (m: +x, +y, +z) then inv(U_ii) and one pad word.
    Absent neighbours (grid faces) are zero-filled and masked by the kernel."""
    b, n = F.block_size, F.n
    if b != 3 or n < 2:
        return None
    lp, lc, lv = _strict(F.L)
    up, uc, uv = _strict(F.U)
    rows_l = np.repeat(np.arange(n, dtype=np.int64), np.diff(lp))
    offs = np.unique(rows_l - lc)
    if offs.shape[0] != 3 or offs[0] != 1:
        return None
    nx, nxy = int(offs[1]), int(offs[2])
    if nx < 2 or nxy % nx or n % nxy or nxy // nx < 2:
        return None
    ny, nz = nxy // nx, n // nxy
    if nz < 2 or nx > 32 * STENCIL_SMAX:
        return None
    i = np.arange(n, dtype=np.int64)
    ix, iy, iz = i % nx, (i // nx) % ny, i // nxy
    # exact stencil patterns in ascending column order
    hl = np.stack([iz > 0, iy > 0, ix > 0], axis=1)
    hu = np.stack([ix < nx - 1, iy < ny - 1, iz < nz - 1], axis=1)
    if not (np.array_equal(np.diff(lp), hl.sum(1)) and np.array_equal(np.diff(up), hu.sum(1))):
        return None
    ol = np.array([nxy, nx, 1], dtype=np.int64)
    ou = np.array([1, nx, nxy], dtype=np.int64)
    exp_l = (i[:, None] - ol[None, :])[hl]
    exp_u = (i[:, None] + ou[None, :])[hu]
    if not (np.array_equal(exp_l, lc) and np.array_equal(exp_u, uc)):
        return None
    doff, P = _stencil_offsets(nx, ny)
    Dn = nx + ny - 1
    lo = np.maximum(0, np.arange(Dn, dtype=np.int64) - (ny - 1))
    dc = ix + iy
    j = ix - lo[dc]
    pos = iz * P + doff[dc] + j                       # stencil position of every row

    def records(vals, mask, nf, extra=None):
        # row-major per stencil position: fields m*9 + e, then `extra`
        rec = np.zeros((nz * P, nf))
        r_of, m_of = np.nonzero(mask)
        rec[pos[r_of][:, None], (m_of * 9)[:, None] + np.arange(9)[None, :]] = vals.reshape(-1, 9)
        if extra is not None:
            rec[pos, 27:36] = extra.reshape(-1, 9)
        return rec.reshape(-1)

    lrec = records(lv, hl, 27)
    urec = records(uv, hu, 37, F.u_diag_inv)       # 36 + 1 pad (bank-conflict-free stride)
    return {"nx": nx, "ny": ny, "nz": nz, "S": (nx + 31) // 32, "D": Dn, "P": P,
            "doff": doff.astype(np.int32), "lrec": lrec, "urec": urec,
            "slot": (3 * pos).astype(np.int32), "len": 3 * nz * P}


class WaveDev:
    def __init__(self, host):
        self.host = host
        self.t = {k: D.upload(host[k]) for k in ("chunk_step", "step_off", "step_bytes", "step_w",
                                                 "step_k", "rhs_off", "rhs_bytes", "stream")}
        cs = np.asarray(host["chunk_step"], dtype=np.int64)
        mcs = int(np.diff(cs).max()) if cs.shape[0] > 1 else 0
        self.desc = N.Wave(host["nchunks"], host["nsteps"], host["stage_max"], host["rhs_max"],
                           *[D.ptr(self.t[k]) for k in ("chunk_step", "step_off", "step_bytes",
                                                         "step_w", "step_k", "rhs_off",
                                                         "rhs_bytes", "stream")], mcs, 0)


class DeviceBilu:
    """Device plan of the BILU(0) solves: chunked-wavefront plans (default) or
    level-ordered SELL-32 copies of the strict factors (use_wave=False)."""

    def __init__(self, F: BiluFactors, use_wave: bool = True):
        D.require_cuda()
        b = F.block_size
        if b not in (1, 3):
            raise NotImplementedError(f"device BILU supports block sizes 1 and 3, got {b}")
        self.use_wave = bool(F.n > 0 and use_wave)
        st = None
        if self.use_wave and os.environ.get("CPRB_STENCIL", "1") != "0":
            dev_pack = (isinstance(F, DeviceBiluFactors)
                        and os.environ.get("CPRB_DEVICE_STENCIL", "1") != "0")
            st = F.stencil_device() if dev_pack else stencil_plan(F)
        self.stencil = st is not None
        if self.use_wave:
            # the wave plans carry their own copies of the factors; the
            # level-ordered SELL-32 layout is only built for the sync-free variant
            self.L = self.U = self.uinv = None
            ldesc = udesc = N.Sell()
            uptr = 0
        else:
            hl, _ = _level_sell(F.L, F.l_schedule, b)
            hu, ui = _level_sell(F.U, F.u_schedule, b, F.u_diag_inv)
            self.L = D.SellDev(hl)
            self.U = D.SellDev(hu)
            self.uinv = D.upload(ui)
            ldesc, udesc, uptr = self.L.desc, self.U.desc, D.ptr(self.uinv)
        t = D.torch()
        self.tickets = t.zeros(8, dtype=t.int32, device="cuda")
        self.work = D.empty(max(F.n * b, 1))
        self.n, self.b = F.n, b
        stdesc = N.Stencil()
        if st is not None:
            # structured grid: one warp per xy-plane sweeping anti-diagonals
            # (csrc/stencil.cu); rhs, L output and U output share the layout
            self.Lw = self.Uw = None
            up = lambda a: a if D.is_tensor(a) else D.upload(a)   # noqa: E731
            self.st_doff = up(st["doff"])
            self.st_lrec = up(st["lrec"])
            self.st_urec = up(st["urec"])
            self.l_slot = self.u_slot = up(st["slot"])
            self.len_l = self.len_u = max(int(st["len"]), 1)
            self.rhs_l = D.zeros(self.len_l)
            self.rhs_u = self.rhs_l
            self.zl_step = D.zeros(self.len_l)
            self.y_step = D.zeros(self.len_u)
            extra = (D.ptr(self.l_slot), D.ptr(self.rhs_l), D.ptr(self.rhs_u), D.ptr(self.u_slot),
                     D.ptr(self.zl_step), D.ptr(self.y_step), self.len_l, self.len_u)
            wl, wu = N.Wave(), N.Wave()
            stdesc = N.Stencil(st["nx"], st["ny"], st["nz"], st["S"], st["D"], st["P"],
                               D.ptr(self.st_doff), D.ptr(self.st_lrec), D.ptr(self.st_urec))
        elif self.use_wave:
            hu, uslot = wave_plan(F.U, F.u_schedule, b, True, uinv=F.u_diag_inv)
            hl, lslot = wave_plan(F.L, F.l_schedule, b, False)
            self.Lw, self.Uw = WaveDev(hl), WaveDev(hu)
            self.l_slot = D.upload(lslot.astype(np.int32))
            self.u_slot = D.upload(uslot.astype(np.int32))
            self.len_l, self.len_u = max(hl["rhs_len"], 1), max(hu["rhs_len"], 1)
            self.rhs_l = D.zeros(self.len_l)
            self.rhs_u = D.zeros(self.len_u)
            self.zl_step = D.zeros(self.len_l)
            self.y_step = D.zeros(self.len_u)
            extra = (D.ptr(self.l_slot), D.ptr(self.rhs_l), D.ptr(self.rhs_u), D.ptr(self.u_slot),
                     D.ptr(self.zl_step), D.ptr(self.y_step), self.len_l, self.len_u)
            wl, wu = self.Lw.desc, self.Uw.desc
        else:
            wl, wu = N.Wave(), N.Wave()
            extra = (0, 0, 0, 0, 0, 0, 0, 0)
        self.desc = N.Bilu(F.n, b, ldesc, udesc, uptr, D.ptr(self.tickets),
                           (2 if self.stencil else 1) if self.use_wave else 0, wl, wu, *extra,
                           stdesc)

    def apply(self, r, z):
        N.check(N.lib().cprb_bilu_apply(C.byref(self.desc), D.ptr(r), D.ptr(z), D.ptr(self.work),
                                        D.stream()))


def bilu_apply(F: BiluFactors, r, workers: int = 1, sequential: bool = False):
    """z = U^{-1} L^{-1} r (src/ilu.py:196-223).  The device solve is bitwise
    equal to both of the reference's paths, so `sequential` only selects the
    same result."""
    n, b = F.n, F.block_size
    if np.shape(r) != (n * b,):
        raise ValueError(f"dimension mismatch: expected vector of length {n * b}")
    dev = F.device()
    rd, kind = D.to_device(r)
    z = D.empty(n * b)
    dev.apply(rd, z)
    return D.from_device(z, kind)
