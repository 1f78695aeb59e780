"""Unsmoothed-aggregation AMG for the pressure operator (drop-in for
cprkit.amg).

SETUP (host C++, bit-exact structure): NPAIR aggregation, colour grouping,
Galerkin products, stall rule and level cap exactly as src/amg.py:143-174;
the coarsest level gets a dense inverse (replacing scipy's lu_factor /
lu_solve; values agree to rounding).
SOLVE (device): the V-cycle is one C-ABI call that launches the colour sweeps,
fused residual + restriction, prolongation and coarse solve
(csrc/amg.cu).  The K-cycle (src/amg.py:177-225) is driven from here: the
recursion and the Krylov scalars stay on the host, every vector operation
runs on the device.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _native as N
from . import device as D
from .coloring import ColorPartition, strong_connections, vertices_grouping
from .smoothers import PgsScmSmoother, SmootherSpec, make_smoother
from .sparse import CsrMatrix

__all__ = ["AggregationMap", "AmgParams", "AmgLevel", "AmgHierarchy", "pairwise_aggregate",
           "build_hierarchy", "amg_cycle", "hierarchy_summary"]


@dataclass
class AggregationMap:
    aggregate_of: np.ndarray
    n_aggregates: int


@dataclass
class AmgParams:
    """src/amg.py:41-66 (same fields, defaults and validation)."""

    coarsest_size: int = 200
    max_levels: int = 25
    theta_amg: float = 0.08
    smoother_theta: float = 0.0
    smoother_kind: str = "pgs-scm"
    pre_sweeps: int = 1
    post_sweeps: int = 1
    cycle: str = "k"
    krylov: str = "auto"

    def __post_init__(self):
        if self.cycle not in ("v", "k"):
            raise ValueError(f"cycle must be 'v' or 'k', got {self.cycle!r}")
        if self.krylov not in ("auto", "fcg", "fgmres"):
            raise ValueError(f"unknown krylov selector {self.krylov!r}")


@dataclass
class AmgLevel:
    A: CsrMatrix
    partition: Optional[ColorPartition]
    smoother: object
    P: Optional[CsrMatrix] = None
    aggregates: Optional[np.ndarray] = None


@dataclass
class AmgHierarchy:
    levels: list
    coarsest_lu: tuple          # ("inverse", dense inverse of the coarsest operator)
    params: AmgParams
    symmetric: bool = False
    _dev: object = None

    @property
    def fine_size(self) -> int:
        return self.levels[0].A.nrows

    def device(self, in_stride: int = 1) -> "DeviceAmg":
        if self._dev is None or self._dev.in_stride != in_stride:
            self._dev = DeviceAmg(self, in_stride)
        return self._dev


def _csr_arrays(A):
    return (np.ascontiguousarray(A.row_ptr, dtype=np.int64),
            np.ascontiguousarray(A.col_idx, dtype=np.int64),
            np.ascontiguousarray(A.values, dtype=np.float64))


def pairwise_aggregate(A, theta_amg: float) -> AggregationMap:
    """Greedy pairwise matching (src/amg.py:89-119), host C++."""
    if A.nrows != A.ncols:
        raise ValueError("aggregation needs a square matrix")
    if not 0.0 <= theta_amg <= 1.0:
        raise ValueError(f"theta must lie in [0, 1], got {theta_amg}")
    p, c, v = _csr_arrays(A)
    agg = np.zeros(A.nrows, dtype=np.int64)
    na = np.zeros(1, dtype=np.int64)
    N.check(N.lib().cprb_pairwise_aggregate(A.nrows, N.p64(p), N.p64(c if c.size else np.zeros(1, np.int64)),
                                            N.pf64(v if v.size else np.zeros(1)), float(theta_amg),
                                            N.p64(agg), N.p64(na)))
    return AggregationMap(agg, int(na[0]))


def _prolongation(agg: AggregationMap, n: int) -> CsrMatrix:
    return CsrMatrix(n, agg.n_aggregates, np.arange(n + 1, dtype=np.int64),
                     agg.aggregate_of.copy(), np.ones(n))


def _galerkin(A, agg: AggregationMap) -> CsrMatrix:
    """A_c[I, J] = sum of A_ij over aggregate pairs (src/amg.py:127-132), host C++."""
    p, c, v = _csr_arrays(A)
    cap = max(c.shape[0], 1)
    cp = np.zeros(agg.n_aggregates + 1, dtype=np.int64)
    cc = np.zeros(cap, dtype=np.int64)
    cv = np.zeros(cap)
    nnz = np.zeros(1, dtype=np.int64)
    a = np.ascontiguousarray(agg.aggregate_of, dtype=np.int64)
    N.check(N.lib().cprb_galerkin(A.nrows, N.p64(p), N.p64(c if c.size else np.zeros(1, np.int64)),
                                  N.pf64(v if v.size else np.zeros(1)), N.p64(a), agg.n_aggregates,
                                  N.p64(cp), N.p64(cc), N.pf64(cv), N.p64(nnz)))
    k = int(nnz[0])
    return CsrMatrix(agg.n_aggregates, agg.n_aggregates, cp, cc[:k].copy(), cv[:k].copy())


def _is_symmetric(A, tol: float = 1e-12) -> bool:
    p, c, v = _csr_arrays(A)
    out = np.zeros(1, dtype=np.int32)
    N.check(N.lib().cprb_is_symmetric(A.nrows, N.p64(p), N.p64(c if c.size else np.zeros(1, np.int64)),
                                      N.pf64(v if v.size else np.zeros(1)), tol, N.p32(out)))
    return bool(out[0])


def _dense_inverse(A) -> np.ndarray:
    n = A.nrows
    dense = np.ascontiguousarray(A.to_dense())
    inv = np.zeros((n, n))
    N.check(N.lib().cprb_dense_inverse(n, N.pf64(dense), N.pf64(inv)))
    return inv


_POOL = None


def setup_pool():
    """Host thread pool of the SETUP phase.  The C++ setup kernels are called
    through ctypes (the GIL is released) and the numpy passes release it for
    large arrays, so independent pieces of setup run concurrently."""
    global _POOL
    if _POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        n = int(os.environ.get("CPRB_SETUP_THREADS", str(min(16, os.cpu_count() or 1))))
        _POOL = ThreadPoolExecutor(max_workers=max(1, n), thread_name_prefix="cprb-setup")
    return _POOL


def _smooth_level(A_l, params):
    partition = vertices_grouping(strong_connections(A_l, params.smoother_theta))
    spec = SmootherSpec(kind=params.smoother_kind,
                        partition=partition if params.smoother_kind == "pgs-scm" else None)
    return partition, make_smoother(A_l, spec)


def build_hierarchy(A_p, params: AmgParams | None = None) -> AmgHierarchy:
    """src/amg.py:143-174: aggregate / project until the coarsest target, the
    level cap or a coarsening stall (n_agg > 0.9 n).

    The aggregation -> Galerkin chain is sequential; each level's colouring
    and smoother depend only on that level's matrix and are built on the
    setup pool while the chain continues.  Errors surface in the reference's
    order: a level's smoother error before anything later in the chain."""
    params = params or AmgParams()
    if A_p.nrows != A_p.ncols:
        raise ValueError("hierarchy needs a square matrix")
    if not isinstance(A_p, CsrMatrix):
        A_p = CsrMatrix(A_p.nrows, A_p.ncols, A_p.row_ptr, A_p.col_idx, A_p.values)
    pool = setup_pool()
    pending = []          # (level index, A_l, agg, future)
    levels = []
    A_l = A_p

    def first_smoother_error():
        for _, _, _, fut in pending:
            exc = fut.exception()
            if exc is not None:
                return exc
        return None

    try:
        sym = _is_symmetric(A_p)
        while True:
            if A_l.nrows <= params.coarsest_size or len(pending) + 1 >= params.max_levels:
                break
            agg = pairwise_aggregate(A_l, params.theta_amg)
            if agg.n_aggregates > 0.9 * A_l.nrows:
                break
            pending.append((len(pending), A_l, agg, pool.submit(_smooth_level, A_l, params)))
            A_l = _galerkin(A_l, agg)
        inv = _dense_inverse(A_l)
    except Exception as exc:
        earlier = first_smoother_error()
        if earlier is not None:
            raise earlier from None
        if isinstance(exc, RuntimeError):
            raise RuntimeError(str(exc)) from exc
        raise
    for _, A_s, agg, fut in pending:
        partition, smoother = fut.result()
        levels.append(AmgLevel(A_s, partition, smoother, P=_prolongation(agg, A_s.nrows),
                               aggregates=agg.aggregate_of))
    levels.append(AmgLevel(A_l, None, None))
    return AmgHierarchy(levels, ("inverse", inv), params, symmetric=sym)


def hierarchy_summary(h: AmgHierarchy) -> dict:
    """src/amg.py:270-285."""
    sizes = [lvl.A.nrows for lvl in h.levels]
    nnzs = [lvl.A.nnz for lvl in h.levels]
    return {
        "levels": len(h.levels),
        "sizes": sizes,
        "nnz": nnzs,
        "colors": [lvl.partition.c if lvl.partition is not None else None for lvl in h.levels],
        "operator_complexity": float(sum(nnzs)) / max(nnzs[0], 1),
        "grid_complexity": float(sum(sizes)) / max(sizes[0], 1),
        "cycle": h.params.cycle,
        "coarsest_size": sizes[-1],
        "symmetric": h.symmetric,
    }


# ----------------------------------------------------------------------------
# device plan
# ----------------------------------------------------------------------------


def _restriction_sell(A, agg: np.ndarray, n_agg: int, inv_l: np.ndarray, inv_c: np.ndarray):
    """Rows grouped by aggregate: lane 2I = lower member, lane 2I+1 = upper member
    (or a dummy), entries in the ORIGINAL column order mapped to permuted
    columns; agg_out[I] = permuted coarse index."""
    n = A.nrows
    order = np.argsort(agg, kind="stable")          # members ascending inside each aggregate
    counts = np.bincount(agg, minlength=n_agg)
    first = np.zeros(n_agg + 1, dtype=np.int64)
    np.cumsum(counts, out=first[1:])
    lane_orig = np.full(2 * n_agg, -1, dtype=np.int64)
    lane_orig[0::2] = order[first[:-1]]
    two = counts == 2
    lane_orig[1::2][two] = order[first[:-1][two] + 1]
    lane_orig = D.pad_lanes(lane_orig)
    L = lane_orig.shape[0]
    real = lane_orig >= 0
    lane_row = np.where(real, inv_l[np.maximum(lane_orig, 0)], -1).astype(np.int32)
    agg_out = np.full(L // 2, -1, dtype=np.int32)
    agg_out[:n_agg] = inv_c[np.arange(n_agg)]
    return D.sell_from_rows(lane_orig, A.row_ptr, A.col_idx, A.values, n, colmap=inv_l,
                            lane_row=lane_row, agg_out=agg_out)


def _permuted_rows_sell(A, perm: np.ndarray, inv: np.ndarray):
    """A_l with rows in permuted order, each row in ORIGINAL column order
    (cols mapped to permuted indices): spmv on permuted vectors with the
    reference's row sums (K-cycle Krylov steps)."""
    lane_orig = D.pad_lanes(perm.astype(np.int64))
    return D.sell_from_rows(lane_orig, A.row_ptr, A.col_idx, A.values, A.nrows, colmap=inv)


# persistent single-CTA V-cycle tail (csrc/vtail.cu): the coarse levels whose
# vectors fit TAIL_VEC_BYTES of shared memory run in one launch
# (CPRB_TAIL_ROWS = largest level admitted; 0 = off)
TAIL_ROWS = 0  # off until the tail beats the launched chain (set after measuring)
TAIL_VEC_BYTES = int(os.environ.get("CPRB_TAIL_VEC_KB", "150")) * 1024
TAIL_SMEM = 227 * 1024
TAIL_NSLOT = 4
VT_SWEEP, VT_RR, VT_COARSE, VT_PROLONG = 1, 3, 4, 5


class _ChunkStream:
    """Phase-ordered stream of <= slot-byte records (16-byte aligned
    sections) for the tail's TMA producer."""

    def __init__(self, slot):
        self.slot = slot
        self.parts, self.chunks, self.phases = [], [], []
        self.off = 0

    def phase(self, typ, level, colour):
        self.phases.append((typ, level, colour, len(self.chunks)))

    def chunk(self, rows, *arrays):
        raw = bytearray()
        for a in arrays:
            b = np.ascontiguousarray(a).tobytes()
            raw.extend(b)
            raw.extend(b"\0" * ((-len(b)) % 16))
        if len(raw) > self.slot:
            raise ValueError("tail chunk exceeds its ring slot")
        self.chunks.append((len(self.phases) - 1, self.off // 16, len(raw), rows))
        self.parts.append(bytes(raw))
        self.off += len(raw)

    def rows_per_chunk(self, per_row, fixed=16, multiple=1):
        r = max(1, (self.slot - fixed - 64) // max(per_row, 1))
        return max(multiple, (r // multiple) * multiple)


class DeviceAmg:
    """Device-resident hierarchy: per level the colour-permuted smoother, the
    fused residual/restriction operator, the prolongation map and work
    vectors; the coarsest dense inverse."""

    def __init__(self, h: AmgHierarchy, in_stride: int = 1):
        D.require_cuda()
        self.h = h
        self.in_stride = int(in_stride)
        L = len(h.levels)
        self.nlevels = L
        perms, invs = [], []
        for lvl in h.levels:
            n = lvl.A.nrows
            if lvl.smoother is not None:
                p = lvl.smoother.perm.astype(np.int64)
            else:
                p = np.arange(n, dtype=np.int64)
            inv = np.empty(n, dtype=np.int64)
            inv[p] = np.arange(n, dtype=np.int64)
            perms.append(p)
            invs.append(inv)
        self.perms, self.invs = perms, invs
        self.levels = []
        self.restrict = []
        self.aggp = []
        self.aggp_host = []
        self.kspmv = []
        for lvl in h.levels[:-1]:
            if not isinstance(lvl.smoother, PgsScmSmoother):
                raise NotImplementedError("device AMG levels use the PGS-SCM smoother")

        def pack(l):
            # one level's device layouts (independent of every other level)
            lvl = h.levels[l]
            dl = lvl.smoother.device()
            na = h.levels[l + 1].A.nrows
            R = D.SellDev(_restriction_sell(lvl.A, lvl.aggregates, na, invs[l], invs[l + 1]))
            aggp_h = invs[l + 1][lvl.aggregates[perms[l]]].astype(np.int32)
            return dl, R, D.upload(aggp_h), aggp_h

        packed = list(setup_pool().map(D.bind_current(pack), range(L - 1)))
        for l in range(L - 1):
            lvl = h.levels[l]
            dl, R, aggp, aggp_h = packed[l]
            self.aggp_host.append(aggp_h)
            dl.desc.restrict_op = R.desc
            dl.desc.restrict_width = int(R.host.lane_len.max()) if R.host.lane_len.size else 0
            dl.desc.aggp = D.ptr(aggp)
            self.levels.append(dl)
            self.restrict.append(R)
            self.aggp.append(aggp)
            self.kspmv.append(None)
        self.level_arr = (N.AmgLevel * max(L - 1, 1))()
        for l, dl in enumerate(self.levels):
            self.level_arr[l] = dl.desc
        inv = h.coarsest_lu[1]
        self.n_coarse = inv.shape[0]
        self.coarse_inv = D.upload(np.ascontiguousarray(inv).reshape(-1))
        self.coarse_b = D.empty(self.n_coarse)
        self.coarse_x = D.empty(self.n_coarse)
        self.perm0 = D.upload(perms[0].astype(np.int32))
        self.desc = N.Amg()
        self.desc.nlevels = L
        self.desc.levels = self.level_arr
        self.desc.n_coarse = self.n_coarse
        self.desc.coarse_inv = D.ptr(self.coarse_inv)
        self.desc.coarse_b = D.ptr(self.coarse_b)
        self.desc.coarse_x = D.ptr(self.coarse_x)
        self.desc.perm0 = D.ptr(self.perm0)
        self.desc.in_stride = self.in_stride
        self.desc.cycle = 0
        self.desc.use_fcg = 1 if (h.params.krylov == "fcg" or
                                  (h.params.krylov == "auto" and h.symmetric)) else 0
        self._build_tail()

    def _build_tail(self):
        """Stream of the persistent V-cycle tail (csrc/vtail.cu): the deepest
        run of levels (>= 1) whose b and x fit TAIL_VEC_BYTES of shared
        memory, each with several colours and no intra-colour couplings
        (those levels keep the launched path), plus the coarse solve.  The
        records restate exactly the launched kernels' inputs: sweep rows
        (permuted, ascending permuted columns, the zero-guess prefix length
        on the way down), restriction lane pairs (original column order),
        aggregate maps and coarse-inverse rows."""
        L = self.nlevels
        self.desc.tail_start = L - 1
        if L <= 2:
            return
        limit = int(os.environ.get("CPRB_TAIL_ROWS", str(TAIL_ROWS)))
        nc = self.n_coarse
        ts = L - 1
        vec_bytes = 16 * nc
        for l in range(L - 2, 0, -1):
            dl = self.levels[l]
            n = int(dl.desc.n)
            if (n > limit or n >= 65536 or dl.desc.ncolors < 2 or dl.snapshot.any()
                    or vec_bytes + 16 * n > TAIL_VEC_BYTES):
                break
            vec_bytes += 16 * n
            ts = l
        if ts >= L - 1:
            return
        vec = np.full(2 * L, -1, dtype=np.int32)
        off = 0
        for l in list(range(ts, L - 1)) + [L - 1]:
            n = nc if l == L - 1 else int(self.levels[l].desc.n)
            vec[2 * l], vec[2 * l + 1] = off, off + n
            off += 2 * n
        vec_len = off
        vbytes = (vec_len * 8 + 127) & ~127
        nph = 1 + sum(2 * int(self.levels[l].desc.ncolors) + 2 for l in range(ts, L - 1))
        meta = 64 + 16 * (nph + 1) + 8 * L + 128      # mbarriers, phase table, offsets
        slot = min(32 * 1024, ((TAIL_SMEM - vbytes - meta) // TAIL_NSLOT) // 16 * 16)
        if slot < max(4096, 8 * nc + 64):
            return
        st = _ChunkStream(slot)
        for l in range(ts, L - 1):
            sp = self.h.levels[l].smoother.split
            for k in range(sp.ncolors):
                self._tail_sweep(st, l, sp, k, True)
            self._tail_rr(st, l)
        inv = np.ascontiguousarray(self.h.coarsest_lu[1], dtype=np.float64)
        st.phase(VT_COARSE, L - 1, 0)
        per = st.rows_per_chunk(8 * nc)
        for a in range(0, nc, per):
            e = min(nc, a + per)
            st.chunk(e - a, np.array([e - a, nc, a, 0], dtype=np.int32), inv[a:e])
        for l in range(L - 2, ts - 1, -1):
            aggp = self.aggp_host[l]
            st.phase(VT_PROLONG, l, 0)
            n = aggp.shape[0]
            per = st.rows_per_chunk(4)
            for a in range(0, n, per):
                e = min(n, a + per)
                st.chunk(e - a, np.array([e - a, 0, a, 0], dtype=np.int32), aggp[a:e])
            sp = self.h.levels[l].smoother.split
            for k in range(sp.ncolors - 1, -1, -1):
                self._tail_sweep(st, l, sp, k, False)
        phases = np.asarray(st.phases + [(0, 0, 0, len(st.chunks))], dtype=np.int32)
        self.tail_phase_host = [p + (sum(1 for c in st.chunks if c[0] == i),)
                                for i, p in enumerate(st.phases)]
        self.tail_phases = D.upload(phases.reshape(-1))
        self.tail_chunks = D.upload(np.asarray(st.chunks, dtype=np.int32).reshape(-1))
        self.tail_stream = D.upload(np.frombuffer(b"".join(st.parts), dtype=np.uint8).copy())
        self.tail_vec = D.upload(vec)
        d = self.desc
        d.tail_nphases = len(st.phases)
        d.tail_nchunks = len(st.chunks)
        d.tail_slot = slot
        d.tail_vec_len = vec_len
        d.tail_smem = vbytes + TAIL_NSLOT * slot + meta
        d.tail_phases = D.ptr(self.tail_phases)
        d.tail_chunks = D.ptr(self.tail_chunks)
        d.tail_stream = D.ptr(self.tail_stream)
        d.tail_vec = D.ptr(self.tail_vec)
        d.tail_stream_bytes = st.off
        d.tail_start = ts
        self.tail_bytes = st.off

    @staticmethod
    def _tail_sweep(st, l, sp, k, zg):
        r0, r1 = int(sp.color_rows[k]), int(sp.color_rows[k + 1])
        st.phase(VT_SWEEP, l, k | (0x100 if zg else 0))
        rows = np.arange(r0, r1, dtype=np.int64)
        lo, hi = sp.off_ptr[rows], sp.off_ptr[rows + 1]
        if zg:   # zero guess: only the entries whose columns precede the colour
            lens = np.array([int(np.searchsorted(sp.off_cols[x:y], r0)) for x, y in zip(lo, hi)],
                            dtype=np.int64)
        else:
            lens = hi - lo
        Wp = int(lens.max()) if lens.size else 0
        per = st.rows_per_chunk(12 + 10 * Wp, fixed=48)
        for a in range(0, r1 - r0, per):
            e = min(r1 - r0, a + per)
            cnt = e - a
            ln = lens[a:e]
            W = int(ln.max()) if cnt else 0
            cols = np.zeros((W, cnt), dtype=np.uint16)
            vals = np.zeros((W, cnt), dtype=np.float64)
            for t in range(cnt):
                m = int(ln[t])
                x = int(lo[a + t])
                cols[:m, t] = sp.off_cols[x:x + m]
                vals[:m, t] = sp.off_vals[x:x + m]
            st.chunk(cnt, np.array([cnt, W, r0 + a, int(zg)], dtype=np.int32),
                     ln.astype(np.int32), sp.diag[r0 + a:r0 + e].astype(np.float64), cols, vals)

    def _tail_rr(self, st, l):
        R = self.restrict[l].host
        st.phase(VT_RR, l, 0)
        lr = R.lane_row.astype(np.int64)
        nl_ = lr.shape[0]
        lens_all = np.where(lr >= 0, R.lane_len, 0).astype(np.int64)
        Wp = int(lens_all.max()) if nl_ else 0
        per = st.rows_per_chunk(10 + 10 * Wp, fixed=64, multiple=32)
        for a in range(0, nl_, per):
            e = min(nl_, a + per)
            lanes = np.arange(a, e, dtype=np.int64)
            cnt = e - a
            ln = lens_all[a:e]
            W = int(ln.max()) if cnt else 0
            cols = np.zeros((W, cnt), dtype=np.uint16)
            vals = np.zeros((W, cnt), dtype=np.float64)
            sl, lane = lanes // 32, lanes % 32
            for m in range(W):
                ok = m < ln
                ent = R.slice_ptr[sl[ok]] + 32 * m + lane[ok]
                cols[m, ok] = R.cols[ent]
                vals[m, ok] = R.vals[ent]
            outs = R.agg_out[a // 2:e // 2].astype(np.int32)
            st.chunk(cnt, np.array([cnt, W, 0, 0], dtype=np.int32), lr[a:e].astype(np.int32),
                     ln.astype(np.int32), outs, cols, vals)

    # -- V-cycle: one native call ------------------------------------------------
    def vcycle(self, r, z):
        N.check(N.lib().cprb_amg_cycle(C.byref(self.desc), D.ptr(r), D.ptr(z), D.stream()))

    # -- K-cycle: host recursion over device steps (src/amg.py:245-267) ----------
    def _kspmv(self, l):
        if self.kspmv[l] is None:
            lvl = self.h.levels[l]
            self.kspmv[l] = D.SellDev(_permuted_rows_sell(lvl.A, self.perms[l], self.invs[l]))
        return self.kspmv[l]

    def _spmv_level(self, l, x):
        y = D.empty(x.shape[0])
        N.check(N.lib().cprb_spmv(C.byref(self._kspmv(l).desc), 1, D.ptr(x), D.ptr(y), None,
                                  D.stream()))
        return y

    def _cycle_at(self, l, b, use_fcg, cycle):
        L = self.nlevels
        if l == L - 1:
            x = D.empty(self.n_coarse)
            N.check(N.lib().cprb_coarse_solve(C.byref(self.desc), D.ptr(b), D.ptr(x), D.stream()))
            return x
        dl = self.levels[l]
        p = self.h.params
        # zero guess (src/amg.py:250): with pre_sweeps = 0 nothing overwrites x
        x = D.empty(b.shape[0]) if p.pre_sweeps > 0 else D.zeros(b.shape[0])
        lib, st = N.lib(), D.stream()
        for s in range(p.pre_sweeps):
            N.check(lib.cprb_pgs_scm_pass(C.byref(dl.desc), D.ptr(b), D.ptr(x), 0,
                                          1 if s == 0 else 0, st))
        nc = self.h.levels[l + 1].A.nrows
        rc = D.empty(nc)
        N.check(lib.cprb_resid_restrict(C.byref(dl.desc), D.ptr(b), D.ptr(x), D.ptr(rc), st))
        if cycle == "v" or l + 1 == L - 1:
            ec = self._cycle_at(l + 1, rc, use_fcg, cycle)
        else:
            pre = lambda s: self._cycle_at(l + 1, s, use_fcg, cycle)  # noqa: E731
            ec = (self._fcg if use_fcg else self._fgmres)(l + 1, rc, pre)
        N.check(lib.cprb_prolong(C.byref(dl.desc), D.ptr(ec), D.ptr(x), st))
        for _ in range(p.post_sweeps):
            N.check(lib.cprb_pgs_scm_pass(C.byref(dl.desc), D.ptr(b), D.ptr(x), 1, 0, st))
        return x

    def _fcg(self, l, rhs, precond, steps=2):
        """src/amg.py:177-196 with device vectors."""
        x = D.zeros(rhs.shape[0])
        r = rhs.clone()
        dirs = []
        for _ in range(steps):
            if np.sqrt(D.dot(r, r)) == 0.0:
                break
            z = precond(r)
            p = z
            for pj, apj, pap_j in dirs:
                coef = D.dot(z, apj) / pap_j
                q = D.empty(p.shape[0])
                D.axpy(-coef, pj, p, q)
                p = q
            ap = self._spmv_level(l, p)
            pap = D.dot(p, ap)
            if pap <= 0.0 or not np.isfinite(pap):
                break
            alpha = D.dot(p, r) / pap
            xn = D.empty(x.shape[0])
            D.axpy(alpha, p, x, xn)
            rn = D.empty(r.shape[0])
            D.axpy(-alpha, ap, r, rn)
            x, r = xn, rn
            dirs.append((p, ap, pap))
        return x

    def _fgmres(self, l, rhs, precond, steps=2):
        """src/amg.py:199-225 with device vectors (small least squares on host)."""
        beta = float(np.sqrt(D.dot(rhs, rhs)))
        if beta == 0.0:
            return D.zeros(rhs.shape[0])
        n = rhs.shape[0]
        v0 = D.empty(n)
        N.check(N.lib().cprb_div_host(n, D.ptr(rhs), beta, D.ptr(v0), D.stream()))
        basis, zs = [v0], []
        H = np.zeros((steps + 1, steps))
        m_eff = steps
        for j in range(steps):
            z = precond(basis[j])
            zs.append(z)
            w = self._spmv_level(l, z)
            for i in range(j + 1):
                H[i, j] = D.dot(w, basis[i])
                wn = D.empty(n)
                D.axpy(-H[i, j], basis[i], w, wn)
                w = wn
            H[j + 1, j] = float(np.sqrt(D.dot(w, w)))
            if H[j + 1, j] == 0.0:
                m_eff = j + 1
                break
            vn = D.empty(n)
            N.check(N.lib().cprb_div_host(n, D.ptr(w), float(H[j + 1, j]), D.ptr(vn), D.stream()))
            basis.append(vn)
        e1 = np.zeros(m_eff + 1)
        e1[0] = beta
        y, *_ = np.linalg.lstsq(H[:m_eff + 1, :m_eff], e1, rcond=None)
        x = D.zeros(n)
        for i in range(m_eff):
            xn = D.empty(n)
            D.axpy(float(y[i]), zs[i], x, xn)
            x = xn
        return x

    @property
    def native_ok(self) -> bool:
        p = self.h.params
        return p.pre_sweeps == 1 and p.post_sweeps == 1

    def hostcycle(self, r, z, cycle):
        """Host-driven cycle (K-cycle, or V with several sweeps) on natural-order
        device vectors r (stride in_stride) -> z (natural order)."""
        t = D.torch()
        if not hasattr(self, "_perm0_t"):
            self._perm0_t = t.from_numpy(self.perms[0]).to("cuda")
            self._gidx_t = t.from_numpy(self.perms[0] * self.in_stride).to("cuda")
        b0 = r.index_select(0, self._gidx_t).contiguous()
        x = self._cycle_at(0, b0, bool(self.desc.use_fcg), cycle)
        z[self._perm0_t] = x

    # -- K-cycle on the device (csrc/kcycle.cu): no host synchronisation ---------
    def kdesc(self):
        """Descriptor of the device K-cycle (FCG or FGMRES flavour), or None
        when the host-driven path is requested (CPRB_HOST_KCYCLE=1)."""
        if getattr(self, "_kdesc", None) is not None:
            return self._kdesc
        if os.environ.get("CPRB_HOST_KCYCLE", "0") == "1":
            return None
        L = self.nlevels
        arr = (N.Sell * max(L - 1, 1))()
        for l in range(1, L - 1):
            arr[l] = self._kspmv(l).desc
        h = C.c_void_p()
        p = self.h.params
        N.check(N.lib().cprb_kcycle_create(C.byref(self.desc), arr, p.pre_sweeps, p.post_sweeps,
                                           C.byref(h)))
        self._kplan, self._kspmv_arr = h, arr
        kd = N.Amg.from_buffer_copy(self.desc)
        kd.cycle = 1
        kd.kwork = h.value
        self._kdesc = kd
        return kd

    def __del__(self):
        try:
            if getattr(self, "_kplan", None):
                N.lib().cprb_kcycle_destroy(self._kplan)
        except Exception:
            pass

    def cycle(self, r, z, cycle):
        if cycle == "v" and self.native_ok:
            self.vcycle(r, z)
        elif cycle == "k" and self.kdesc() is not None:
            N.check(N.lib().cprb_amg_cycle(C.byref(self._kdesc), D.ptr(r), D.ptr(z), D.stream()))
        else:
            self.hostcycle(r, z, cycle)


def amg_cycle(h: AmgHierarchy, r, cycle: str | None = None, workers: int = 1):
    """One multigrid cycle from a zero guess, z ~= A^{-1} r (src/amg.py:228-242)."""
    if np.shape(r) != (h.fine_size,):
        raise ValueError(f"dimension mismatch: expected residual of length {h.fine_size}")
    cycle = cycle or h.params.cycle
    dev = h.device(1)
    rd, kind = D.to_device(r)
    z = D.empty(h.fine_size)
    dev.cycle(rd, z, cycle)
    return D.from_device(z, kind)
