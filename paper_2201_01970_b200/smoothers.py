"""Multi-colour Gauss-Seidel (PGS-SCM) on the device (drop-in for
cprkit.smoothers, scalar levels).

Setup (host): the colour-permuted matrix A.permuted(perm) is split into the
diagonal and the off-diagonals in ascending permuted column order
(src/smoothers.py:69-94, :257-271) and packed into SELL-32 with one run of
slices per colour.  Sweeps (device): one kernel per colour, rows of a colour in
parallel, each row summed sequentially from 0.0 exactly as the reference's
scalar loop (src/smoothers.py:106-115), so results are bitwise equal.

Out of scope: PGS-NO (its operator is defined by the CPU worker count,
src/smoothers.py:17-21) and block (b > 1) Gauss-Seidel, which is not on the
CPR-AMG path (every AMG level is scalar).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _native as N
from . import device as D
from .coloring import ColorPartition
from .sparse import BlockCsrMatrix, CsrMatrix

__all__ = ["SmootherSpec", "PgsScmSmoother", "ClassicGsSmoother", "gs_sweep", "pgs_scm_sweep",
           "pgs_no_sweep", "make_smoother", "ScalarSplit"]

_KINDS = ("classic-gs", "pgs-no", "pgs-scm")


@dataclass
class SmootherSpec:
    kind: str = "classic-gs"
    sweeps: int = 1
    direction: str = "forward"
    partition: Optional[ColorPartition] = None

    def __post_init__(self):
        if self.kind not in _KINDS:
            raise ValueError(f"unknown smoother kind {self.kind!r}; expected one of {_KINDS}")
        if self.sweeps < 1:
            raise ValueError("sweeps must be >= 1")
        if self.direction not in ("forward", "backward", "symmetric"):
            raise ValueError(f"unknown sweep direction {self.direction!r}")
        if self.kind == "pgs-scm" and self.partition is None:
            raise ValueError("pgs-scm requires a ColorPartition")


class ScalarSplit:
    """Colour-permuted diagonal / off-diagonal split of a scalar matrix."""

    def __init__(self, A, partition: ColorPartition):
        n = int(A.nrows)
        self.n = n
        self.perm = partition.perm().astype(np.int64)
        inv = np.empty(n, dtype=np.int64)
        inv[self.perm] = np.arange(n, dtype=np.int64)
        self.inv = inv
        ptr = np.ascontiguousarray(A.row_ptr, dtype=np.int64)
        cols = np.ascontiguousarray(A.col_idx, dtype=np.int64)
        vals = np.ascontiguousarray(A.values, dtype=np.float64)
        # A.permuted(perm): rows by permuted index, each row's off-diagonals in
        # ascending permuted column, the diagonal apart (host C++)
        nnz = max(int(ptr[-1]) if n else 0, 1)
        self.off_ptr = np.zeros(n + 1, dtype=np.int64)
        self.off_cols = np.zeros(nnz, dtype=np.int64)
        self.off_vals = np.zeros(nnz)
        self.diag = np.zeros(max(n, 1))
        N.check(N.lib().cprb_scalar_split(n, N.p64(ptr), N.p64(cols if cols.size else self.off_cols),
                                          N.pf64(vals if vals.size else self.off_vals),
                                          N.p64(self.perm), N.p64(inv), N.p64(self.off_ptr),
                                          N.p64(self.off_cols), N.pf64(self.off_vals),
                                          N.pf64(self.diag)))
        k = int(self.off_ptr[-1])
        self.off_cols, self.off_vals, self.diag = self.off_cols[:k], self.off_vals[:k], self.diag[:n]
        self.off_rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(self.off_ptr))
        sizes = np.array([g.shape[0] for g in partition.groups], dtype=np.int64)
        self.color_rows = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
        self.ncolors = len(partition.groups)

    def sell(self):
        """SELL-32 with each colour padded to whole slices; lane_len_lo counts the
        prefix of entries whose columns precede the row's colour."""
        lanes, lane_ptr_parts, slices = [], [], [0]
        row_color_start = np.zeros(self.n, dtype=np.int64)
        snapshot = np.zeros(max(self.ncolors, 1), dtype=np.uint8)
        for k in range(self.ncolors):
            s, e = int(self.color_rows[k]), int(self.color_rows[k + 1])
            lanes.append(D.pad_lanes(np.arange(s, e, dtype=np.int32)))
            slices.append(slices[-1] + lanes[-1].shape[0] // 32)
            row_color_start[s:e] = s
            lo, hi = self.off_ptr[s], self.off_ptr[e]
            c = self.off_cols[lo:hi]
            snapshot[k] = 1 if np.any((c >= s) & (c < e)) else 0
        lane_row = np.concatenate(lanes) if lanes else np.zeros(0, dtype=np.int32)
        L = lane_row.shape[0]
        real = lane_row >= 0
        lens = np.zeros(L, dtype=np.int64)
        lens[real] = np.diff(self.off_ptr)[lane_row[real]]
        lane_ptr = np.zeros(L + 1, dtype=np.int64)
        np.cumsum(lens, out=lane_ptr[1:])
        # real lanes visit rows 0..n-1 in ascending order (colours are contiguous
        # ascending row ranges), so the lane entry lists are the row lists
        ent_cols = self.off_cols
        ent_vals = self.off_vals
        lo_cnt = (self.off_cols < row_color_start[self.off_rows])
        lo_per_row = np.bincount(self.off_rows[lo_cnt], minlength=self.n).astype(np.int64)
        lane_lo = np.zeros(L, dtype=np.int32)
        lane_lo[real] = lo_per_row[lane_row[real]]
        h = D.pack_sell(lane_row, lane_ptr, ent_cols, ent_vals, 1, self.n, lane_len_lo=lane_lo)
        return h, np.asarray(slices, dtype=np.int32), snapshot[:self.ncolors]


class DeviceSmootherLevel:
    """Device half of one smoothed level (SELL smoother + diagonal + work)."""

    def __init__(self, split: ScalarSplit):
        D.require_cuda()
        h, slices, snap = split.sell()
        self.split = split
        self.sell = D.SellDev(h)
        self.diag = D.upload(split.diag)
        self.color_slices = np.ascontiguousarray(slices, dtype=np.int32)
        self.color_rows = np.ascontiguousarray(split.color_rows, dtype=np.int32)
        self.snapshot = np.ascontiguousarray(snap, dtype=np.uint8)
        n = split.n
        self.b = D.empty(n)
        self.x = D.empty(n)
        self.tmp = D.empty(n)
        self.desc = N.AmgLevel()
        self.desc.n = n
        self.desc.ncolors = split.ncolors
        self.desc.color_slices = N.p32(self.color_slices)
        self.desc.color_rows = N.p32(self.color_rows)
        self.desc.color_snapshot = self.snapshot.ctypes.data_as(N.u8p)
        # per colour: max row length, max zero-guess prefix length (kernel
        # register prefetch depth, csrc/amg.cu launch_sweep)
        cw = np.zeros(2 * max(split.ncolors, 1), dtype=np.int32)
        ll, lo = h.lane_len, h.lane_len_lo
        for k in range(split.ncolors):
            a, e = int(slices[k]) * 32, int(slices[k + 1]) * 32
            if e > a:
                cw[2 * k] = int(ll[a:e].max())
                cw[2 * k + 1] = int(lo[a:e].max())
        self.color_width = cw
        self.desc.color_width = N.p32(self.color_width)
        self.desc.smoother = self.sell.desc
        self.desc.diag = D.ptr(self.diag)
        self.desc.b = D.ptr(self.b)
        self.desc.x = D.ptr(self.x)
        self.desc.tmp = D.ptr(self.tmp)

    def passes(self, b, x, sweeps, direction):
        """In-place passes on permuted device vectors b, x."""
        dirs = {"forward": (0,), "backward": (1,), "symmetric": (0, 1)}[direction]
        for _ in range(sweeps):
            for d in dirs:
                N.check(N.lib().cprb_pgs_scm_pass(C.byref(self.desc), D.ptr(b), D.ptr(x), d, 0,
                                                  D.stream()))


def _check_pair(A, b, x):
    n = A.nrows * int(getattr(A, "block_size", 1))
    if np.shape(b) != (n,) or np.shape(x) != (n,):
        raise ValueError(f"vector length must be {n}")


class PgsScmSmoother:
    """Multi-colour sweep on the colour-permuted system (src/smoothers.py:246-318)."""

    def __init__(self, A, partition: ColorPartition):
        if partition.n != A.nrows:
            raise ValueError(f"partition covers {partition.n} vertices, matrix has {A.nrows} rows")
        if isinstance(A, BlockCsrMatrix) or int(getattr(A, "block_size", 1)) > 1:
            raise NotImplementedError("block Gauss-Seidel is outside the device CPR path "
                                      "(AMG levels are scalar)")
        self.partition = partition
        self.perm = partition.perm()
        self.split = ScalarSplit(A, partition)
        self.color_ranges = [(int(self.split.color_rows[i]), int(self.split.color_rows[i + 1]))
                             for i in range(self.split.ncolors)]
        self._dev = None

    def device(self) -> DeviceSmootherLevel:
        if self._dev is None:
            self._dev = DeviceSmootherLevel(self.split)
        return self._dev

    def apply(self, b, x, workers: int = 1, sweeps: int = 1, direction: str = "forward"):
        dev = self.device()
        bd, kind = D.to_device(b)
        xd, _ = D.to_device(x)
        t = D.torch()
        perm = t.from_numpy(self.perm).to("cuda")
        bp = bd.index_select(0, perm).contiguous()
        xp = xd.index_select(0, perm).contiguous()
        dev.passes(bp, xp, sweeps, direction)
        out = t.empty_like(xp)
        out[perm] = xp
        return D.from_device(out, kind)


class ClassicGsSmoother(PgsScmSmoother):
    """Sequential Gauss-Seidel = single-colour PGS-SCM on the identity order."""

    def __init__(self, A):
        part = ColorPartition.from_groups([np.arange(A.nrows, dtype=np.int64)], A.nrows)
        super().__init__(A, part)


def gs_sweep(A, b, x, spec: SmootherSpec | None = None):
    spec = spec or SmootherSpec()
    _check_pair(A, b, x)
    return ClassicGsSmoother(A).apply(b, x, sweeps=spec.sweeps, direction=spec.direction)


def pgs_scm_sweep(A, b, x, partition: ColorPartition, workers: int = 1):
    _check_pair(A, b, x)
    return PgsScmSmoother(A, partition).apply(b, x, workers=workers)


def pgs_no_sweep(A, b, x, nworkers: int):
    raise NotImplementedError("PGS-NO is a CPU-thread baseline whose operator depends on the "
                              "worker count (src/smoothers.py:17-21); it has no device form")


def make_smoother(A, spec: SmootherSpec):
    if spec.kind == "classic-gs":
        return ClassicGsSmoother(A)
    if spec.kind == "pgs-no":
        raise NotImplementedError("PGS-NO has no device form (see pgs_no_sweep)")
    return PgsScmSmoother(A, spec.partition)
