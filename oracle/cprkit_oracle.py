"""CPU oracle: a numpy restatement of the reference (cprkit 0.1.0) CPR-GMRES path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package
(``paper_2201_01970_b200``) imports this module.  The only permitted users are
``tests/``, ``__graft_entry__.smoke()`` (as the checker) and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs (as the timed CPU baseline).

Every function restates one reference function; the citation convention is
``src/X.py:N`` = ``/root/reference/pkg/src/cprkit/X.py`` line N.  Arithmetic
orders are kept identical to the reference so that results are bitwise equal
wherever the reference is bitwise deterministic:

* ``np.add.reduceat`` segment sums (``src/_kernels.py:34``) are used directly;
  their order is ``a[0] + pairwise8(a[1:])`` (pinned by ``tests/test_oracle.py``).
* The scalar PGS-SCM row update is a sequential left-to-right sum from 0.0
  (``src/smoothers.py:106-115``); here it is vectorised over the rows of a
  colour, one stored entry position at a time, which is the same per-row order.
* ``np.einsum('kij,kj->ki')`` and batched ``@`` are used where the reference
  uses them (batched ``@`` is bitwise equal to per-block ``@``, see
  tests/test_oracle.py).
* BILU(0) factor values come from OpenBLAS ``dgemm`` (DYNAMIC_ARCH) exactly as
  in the reference, so they are bitwise equal to the reference on the same
  host CPU only.

Parity pinning: tests/golden/*.npz are produced by tests/golden/make_golden.py,
which imports the unmodified reference; tests/test_oracle.py checks this module
against every fixture (structure bit-exact, values bit-exact or to the stated
tolerance).
"""

from __future__ import annotations

import heapq
import math
import warnings
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import scipy.linalg

# --------------------------------------------------------------------------
# storage (src/sparse.py)
# --------------------------------------------------------------------------


class Csr:
    """Canonical scalar CSR (src/sparse.py:67-200)."""

    def __init__(self, nrows, ncols, ptr, cols, vals):
        self.nrows = int(nrows)
        self.ncols = int(ncols)
        self.ptr = np.ascontiguousarray(ptr, dtype=np.int64)
        self.cols = np.ascontiguousarray(cols, dtype=np.int64)
        self.vals = np.ascontiguousarray(vals, dtype=np.float64)

    @property
    def nnz(self):
        return int(self.cols.shape[0])

    def rows(self):
        return np.repeat(np.arange(self.nrows, dtype=np.int64), np.diff(self.ptr))

    def to_dense(self):
        out = np.zeros((self.nrows, self.ncols))
        out[self.rows(), self.cols] = self.vals
        return out

    def diagonal(self):
        """src/sparse.py:149-158: structurally missing diagonal reads 0."""
        d = np.zeros(self.nrows)
        r = self.rows()
        on = r == self.cols
        d[r[on]] = self.vals[on]
        return d


class Bsr:
    """Canonical block CSR, values (nnz, b, b) row-major (src/sparse.py:203-308)."""

    def __init__(self, b, nrows, ncols, ptr, cols, vals):
        self.b = int(b)
        self.nrows = int(nrows)
        self.ncols = int(ncols)
        self.ptr = np.ascontiguousarray(ptr, dtype=np.int64)
        self.cols = np.ascontiguousarray(cols, dtype=np.int64)
        self.vals = np.ascontiguousarray(vals, dtype=np.float64).reshape(-1, self.b, self.b)
        self._expanded = None

    @property
    def nnz(self):
        return int(self.cols.shape[0])

    def rows(self):
        return np.repeat(np.arange(self.nrows, dtype=np.int64), np.diff(self.ptr))

    def expanded(self) -> Csr:
        """Scalar CSR of the b*n system keeping all b*b entries per block
        (src/sparse.py:275-286).  Expanded row (i, r) lists, for every block m
        of block row i in ascending block column, the entries c = 0..b-1."""
        if self._expanded is None:
            b = self.b
            cnt = np.diff(self.ptr)
            ptr_e = np.zeros(self.nrows * b + 1, dtype=np.int64)
            ptr_e[1:] = np.cumsum(np.repeat(cnt * b, b))
            rows_b = self.rows()
            m = np.arange(self.nnz, dtype=np.int64) - self.ptr[rows_b]
            r = np.arange(b)[None, :, None]
            c = np.arange(b)[None, None, :]
            dest = (b * b * self.ptr[rows_b])[:, None, None] + r * b * cnt[rows_b][:, None, None] \
                + (m * b)[:, None, None] + c
            vals_e = np.empty(self.nnz * b * b)
            cols_e = np.empty(self.nnz * b * b, dtype=np.int64)
            vals_e[dest.reshape(-1)] = self.vals.reshape(-1)
            cols_e[dest.reshape(-1)] = np.broadcast_to(self.cols[:, None, None] * b + c,
                                                       dest.shape).reshape(-1)
            self._expanded = Csr(self.nrows * b, self.ncols * b, ptr_e, cols_e, vals_e)
        return self._expanded

    def to_dense(self):
        return self.expanded().to_dense()


def csr_from_coo(rows, cols, vals, shape, sum_duplicates=False) -> Csr:
    """src/sparse.py:88-110: stable lexsort by (row, col); duplicate runs
    collapsed with np.add.reduceat in their sorted (stable) order."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    if rows.size:
        dup = (np.diff(rows) == 0) & (np.diff(cols) == 0)
        if dup.any():
            if not sum_duplicates:
                raise ValueError("duplicate (i, j) entries in COO input")
            keep = np.concatenate(([True], ~dup))
            vals = np.add.reduceat(vals, np.flatnonzero(keep))
            rows, cols = rows[keep], cols[keep]
    ptr = np.zeros(shape[0] + 1, dtype=np.int64)
    np.add.at(ptr[1:], rows, 1)
    np.cumsum(ptr, out=ptr)
    return Csr(shape[0], shape[1], ptr, cols, vals)


def bsr_from_block_coo(b, rows, cols, blocks, shape, sum_duplicates=False) -> Bsr:
    """src/sparse.py:237-257."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    blocks = np.asarray(blocks, dtype=np.float64)
    order = np.lexsort((cols, rows))
    rows, cols, blocks = rows[order], cols[order], blocks[order]
    if rows.size:
        dup = (np.diff(rows) == 0) & (np.diff(cols) == 0)
        if dup.any():
            if not sum_duplicates:
                raise ValueError("duplicate (i, j) blocks in COO input")
            keep = np.concatenate(([True], ~dup))
            blocks = np.add.reduceat(blocks, np.flatnonzero(keep), axis=0)
            rows, cols = rows[keep], cols[keep]
    ptr = np.zeros(shape[0] + 1, dtype=np.int64)
    np.add.at(ptr[1:], rows, 1)
    np.cumsum(ptr, out=ptr)
    return Bsr(b, shape[0], shape[1], ptr, cols, blocks)


def permuted(A: Csr, perm) -> Csr:
    """src/sparse.py:173-181: result[i, j] = A[perm[i], perm[j]]."""
    perm = np.asarray(perm, dtype=np.int64)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.shape[0], dtype=np.int64)
    return csr_from_coo(inv[A.rows()], inv[A.cols], A.vals, (A.nrows, A.ncols))


def transpose(A: Csr) -> Csr:
    return csr_from_coo(A.cols, A.rows(), A.vals, (A.ncols, A.nrows))


# --------------------------------------------------------------------------
# kernels (src/_kernels.py, src/sparse.py:322-369)
# --------------------------------------------------------------------------


def segment_sums(products, ptr):
    """src/_kernels.py:17-40 (np.add.reduceat, empty segments -> 0)."""
    nseg = ptr.shape[0] - 1
    shape = (nseg,) if products.ndim == 1 else (nseg, products.shape[1])
    out = np.zeros(shape)
    if nseg == 0 or products.shape[0] == 0:
        return out
    starts = ptr[:-1]
    nonempty = ptr[1:] > starts
    if nonempty.all():
        np.add.reduceat(products, starts, axis=0, out=out)
    else:
        out[nonempty] = np.add.reduceat(products, starts[nonempty], axis=0)
    return out


def pairwise_sum(a) -> float:
    """numpy's pairwise summation (the order np.add.reduce / reduceat use on a
    contiguous float64 segment), restated in pure Python for pinning."""
    n = len(a)
    if n < 8:
        s = 0.0
        for v in a:
            s += float(v)
        return s
    if n <= 128:
        r = [float(v) for v in a[:8]]
        i = 8
        while i + 8 <= n:
            for k in range(8):
                r[k] += float(a[i + k])
            i += 8
        s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            s += float(a[i])
            i += 1
        return s
    n2 = n // 2
    n2 -= n2 % 8
    return pairwise_sum(a[:n2]) + pairwise_sum(a[n2:])


def segment_sum_scalar(a) -> float:
    """One reduceat segment: a[0] + pairwise(a[1:])."""
    if len(a) == 0:
        return 0.0
    return float(a[0]) + pairwise_sum(a[1:])


def spmv(A, x):
    """src/sparse.py:322-351; BSR goes through the expanded scalar CSR."""
    x = np.asarray(x, dtype=np.float64)
    S = A.expanded() if isinstance(A, Bsr) else A
    if x.shape != (S.ncols,):
        raise ValueError(f"dimension mismatch: matrix has {S.ncols} columns, "
                         f"vector has length {x.shape[0]}")
    return segment_sums(S.vals * x[S.cols], S.ptr)


def dot(x, y) -> float:
    """src/sparse.py:361-365."""
    if x.shape != y.shape:
        raise ValueError("dimension mismatch in dot")
    return float(np.add.reduce(x * y))


def norm2(x) -> float:
    return math.sqrt(dot(x, x))


def invert_small_blocks(blocks):
    """src/sparse.py:372-396, vectorised over blocks with identical per-block
    element operations (pivot = first max |a|; rows with a zero multiplier are
    left untouched exactly as the reference's `a[r, col] != 0.0` guard)."""
    blocks = np.asarray(blocks, dtype=np.float64)
    m, b, _ = blocks.shape
    a = blocks.copy()
    inv = np.broadcast_to(np.eye(b), (m, b, b)).copy()
    ar = np.arange(m)
    for col in range(b):
        p = col + np.argmax(np.abs(a[:, col:, col]), axis=1)
        bad = a[ar, p, col] == 0.0
        if bad.any():
            k = int(np.flatnonzero(bad)[0])
            raise np.linalg.LinAlgError(f"singular diagonal block at row {k}")
        sw = p != col
        if sw.any():
            idx = ar[sw]
            pc = p[sw]
            ra, rp = a[idx, col].copy(), a[idx, pc].copy()
            a[idx, col], a[idx, pc] = rp, ra
            ia, ip = inv[idx, col].copy(), inv[idx, pc].copy()
            inv[idx, col], inv[idx, pc] = ip, ia
        piv = a[:, col, col].copy()
        a[:, col] /= piv[:, None]
        inv[:, col] /= piv[:, None]
        for r in range(b):
            if r == col:
                continue
            f = a[:, r, col].copy()
            nz = f != 0.0
            if nz.any():
                a[nz, r] = a[nz, r] - f[nz, None] * a[nz, col]
                inv[nz, r] = inv[nz, r] - f[nz, None] * inv[nz, col]
    return inv


# --------------------------------------------------------------------------
# strong connections + colouring (src/coloring.py)
# --------------------------------------------------------------------------


@dataclass
class Pattern:
    """Pattern-only CSR (StrongConnectionMatrix, src/coloring.py:39-76)."""
    n: int
    ptr: np.ndarray
    cols: np.ndarray

    def neighbors(self, i):
        return self.cols[self.ptr[i]:self.ptr[i + 1]]


def frobenius(A: Bsr) -> Csr:
    """src/sparse.py:288-295."""
    norms = np.sqrt(np.einsum("kij,kij->k", A.vals, A.vals))
    return Csr(A.nrows, A.ncols, A.ptr.copy(), A.cols.copy(), norms)


def strong_connections(A, theta) -> Pattern:
    """src/coloring.py:79-114: S_ij iff i != j and |a_ij| > theta * sum_k |a_ik|
    (row sum in reduceat order, diagonal included)."""
    if not 0.0 <= theta <= 1.0:
        raise ValueError(f"theta must lie in [0, 1], got {theta}")
    if isinstance(A, Bsr):
        A = frobenius(A)
    absvals = np.abs(A.vals)
    row_sums = segment_sums(absvals, A.ptr)
    rows = A.rows()
    strong = (absvals > theta * row_sums[rows]) & (A.cols != rows)
    ptr = np.zeros(A.nrows + 1, dtype=np.int64)
    np.add.at(ptr[1:], rows[strong], 1)
    np.cumsum(ptr, out=ptr)
    return Pattern(A.nrows, ptr, A.cols[strong].copy())


def symmetrized(S: Pattern) -> Pattern:
    """src/coloring.py:58-71: S union S^T, sorted, deduplicated."""
    rows = np.repeat(np.arange(S.n, dtype=np.int64), np.diff(S.ptr))
    rr = np.concatenate([rows, S.cols])
    cc = np.concatenate([S.cols, rows])
    order = np.lexsort((cc, rr))
    rr, cc = rr[order], cc[order]
    if rr.size:
        keep = np.concatenate(([True], (np.diff(rr) != 0) | (np.diff(cc) != 0)))
        rr, cc = rr[keep], cc[keep]
    ptr = np.zeros(S.n + 1, dtype=np.int64)
    np.add.at(ptr[1:], rr, 1)
    np.cumsum(ptr, out=ptr)
    return Pattern(S.n, ptr, cc)


def _adjacency(S: Pattern):
    ptr = S.ptr.tolist()
    cols = S.cols.tolist()
    return [cols[ptr[i]:ptr[i + 1]] for i in range(S.n)]


def vertices_splitting(vertices, influence, nb, n):
    """src/coloring.py:171-235 (one greedy round).  Candidate priority is the
    tuple (-influence, index); frontier entries are validated lazily at pop."""
    und = bytearray(n)
    for v in vertices:
        und[v] = 1
    deferred = bytearray(n)
    in_front = bytearray(n)
    in_w = bytearray(n)
    v_heap = [(-influence[v], v) for v in vertices]
    heapq.heapify(v_heap)
    f_heap: list = []
    w_list = []
    remaining = len(vertices)
    push, pop = heapq.heappush, heapq.heappop
    while remaining > 0:
        v = -1
        while f_heap:
            _, cand = pop(f_heap)
            if in_front[cand] and und[cand]:
                in_front[cand] = 0
                v = cand
                break
            in_front[cand] = 0
        if v < 0:
            while v_heap:
                _, cand = pop(v_heap)
                if und[cand]:
                    v = cand
                    break
            if v < 0:
                break
        neigh = nb[v]
        if any(in_w[k] for k in neigh):
            deferred[v] = 1
            und[v] = 0
            remaining -= 1
            continue
        in_w[v] = 1
        w_list.append(v)
        und[v] = 0
        remaining -= 1
        for k in neigh:
            if und[k]:
                deferred[k] = 1
                und[k] = 0
                remaining -= 1
        for k in neigh:
            for j in nb[k]:
                if und[j] and not in_front[j] and j != v:
                    in_front[j] = 1
                    push(f_heap, (-influence[j], j))
    w = sorted(w_list)
    w_bar = np.flatnonzero(np.frombuffer(bytes(deferred), dtype=np.uint8)).tolist()
    return w, w_bar


def vertices_grouping(S: Pattern) -> list:
    """src/coloring.py:238-256: repeated splitting over the symmetrised graph;
    influence = symmetrised degree, fixed for all rounds."""
    Ssym = symmetrized(S)
    influence = np.diff(Ssym.ptr).tolist()
    nb = _adjacency(Ssym)
    vertices = list(range(S.n))
    groups = []
    while vertices:
        w, w_bar = vertices_splitting(vertices, influence, nb, S.n)
        if not w:
            raise RuntimeError("vertices_splitting returned an empty group")
        groups.append(np.array(w, dtype=np.int64))
        vertices = w_bar
    return groups


def verify_groups(A, theta, groups) -> bool:
    """Core checks of src/coloring.py:273-326: cover, disjoint, no strong edge
    inside a group."""
    S = symmetrized(strong_connections(A, theta))
    n = S.n
    color = np.zeros(n, dtype=np.int64)
    counts = np.zeros(n, dtype=np.int64)
    for c, g in enumerate(groups, start=1):
        np.add.at(counts, g, 1)
        color[g] = c
    if not ((counts == 1).all()):
        return False
    rows = np.repeat(np.arange(n), np.diff(S.ptr))
    return not bool((color[rows] == color[S.cols]).any())


# --------------------------------------------------------------------------
# smoother (src/smoothers.py)
# --------------------------------------------------------------------------


class ScmSmoother:
    """PGS-SCM on the colour-permuted scalar matrix (src/smoothers.py:246-318,
    _ScalarSplit :69-115)."""

    def __init__(self, A: Csr, groups):
        self.groups = groups
        self.perm = np.concatenate(groups) if groups else np.zeros(0, dtype=np.int64)
        Ap = permuted(A, self.perm)
        rows = Ap.rows()
        off = rows != Ap.cols
        counts = np.zeros(Ap.nrows, dtype=np.int64)
        np.add.at(counts, rows[off], 1)
        self.ptr = np.zeros(Ap.nrows + 1, dtype=np.int64)
        np.cumsum(counts, out=self.ptr[1:])
        self.cols = Ap.cols[off].copy()
        self.vals = Ap.vals[off].copy()
        diag = Ap.diagonal()
        zero = np.flatnonzero(diag == 0.0)
        if zero.size:
            raise np.linalg.LinAlgError(f"zero diagonal at row {int(zero[0])}")
        self.diag = diag
        sizes = np.array([g.shape[0] for g in groups], dtype=np.int64)
        bounds = np.concatenate([[0], np.cumsum(sizes)])
        self.color_ranges = [(int(bounds[i]), int(bounds[i + 1])) for i in range(len(groups))]
        self.n = Ap.nrows

    def _rows_update(self, bp, xp, s, e):
        """x_i <- (b_i - sum_p v_p x_{c_p}) / d_i, sum sequential from 0.0,
        reading the snapshot xp (src/smoothers.py:106-115)."""
        lo = self.ptr[s:e]
        ln = self.ptr[s + 1:e + 1] - lo
        acc = np.zeros(e - s)
        for k in range(int(ln.max(initial=0))):
            m = ln > k
            idx = lo[m] + k
            acc[m] = acc[m] + self.vals[idx] * xp[self.cols[idx]]
        return (bp[s:e] - acc) / self.diag[s:e]

    def _sequential(self, bp, xp, reverse):
        rng = range(self.n - 1, -1, -1) if reverse else range(self.n)
        ptr, cols, vals, diag = self.ptr, self.cols, self.vals, self.diag
        for i in rng:
            acc = 0.0
            for p in range(ptr[i], ptr[i + 1]):
                acc += vals[p] * xp[cols[p]]
            xp[i] = (bp[i] - acc) / diag[i]

    def apply(self, b, x, sweeps=1, direction="forward"):
        bp = np.asarray(b, dtype=np.float64)[self.perm]
        xp = np.asarray(x, dtype=np.float64)[self.perm].copy()
        passes = {"forward": (False,), "backward": (True,), "symmetric": (False, True)}[direction]
        for _ in range(sweeps):
            for reverse in passes:
                if len(self.color_ranges) == 1:
                    self._sequential(bp, xp, reverse)
                    continue
                ranges = self.color_ranges[::-1] if reverse else self.color_ranges
                for s, e in ranges:
                    xp[s:e] = self._rows_update(bp, xp, s, e)
        out = np.empty_like(xp)
        out[self.perm] = xp
        return out


def gs_sweep(A: Csr, b, x, reverse=False):
    """Classic sequential GS (src/smoothers.py:174-197, scalar path)."""
    sm = ScmSmoother(A, [np.arange(A.nrows, dtype=np.int64)])
    return sm.apply(b, x, direction="backward" if reverse else "forward")


# --------------------------------------------------------------------------
# AMG (src/amg.py)
# --------------------------------------------------------------------------


def pairwise_aggregate(A: Csr, theta_amg):
    """src/amg.py:89-119 (NPAIR).  Returns (aggregate_of, n_aggregates)."""
    n = A.nrows
    S = strong_connections(A, theta_amg)
    rows = A.rows()
    W = csr_from_coo(np.concatenate([rows, A.cols]), np.concatenate([A.cols, rows]),
                     np.concatenate([np.abs(A.vals), np.abs(A.vals)]), (n, n),
                     sum_duplicates=True)
    sp, sc = S.ptr.tolist(), S.cols.tolist()
    wp, wc, wv = W.ptr.tolist(), W.cols.tolist(), W.vals.tolist()
    agg = [-1] * n
    na = 0
    for i in range(n):
        if agg[i] >= 0:
            continue
        best_j, best_w = -1, None
        wlo, whi = wp[i], wp[i + 1]
        q = wlo
        for j in sc[sp[i]:sp[i + 1]]:
            if agg[j] >= 0:
                continue
            while wc[q] < j:
                q += 1
            wgt = wv[q]
            if best_w is None or wgt > best_w:
                best_j, best_w = j, wgt
        if best_j >= 0:
            agg[best_j] = na
        agg[i] = na
        na += 1
    return np.array(agg, dtype=np.int64), na


def galerkin(A: Csr, agg, n_agg) -> Csr:
    """src/amg.py:127-132."""
    return csr_from_coo(agg[A.rows()], agg[A.cols], A.vals, (n_agg, n_agg), sum_duplicates=True)


def is_symmetric(A: Csr, tol=1e-12) -> bool:
    """src/amg.py:135-140."""
    At = transpose(A)
    if not (np.array_equal(A.ptr, At.ptr) and np.array_equal(A.cols, At.cols)):
        return False
    scale = np.abs(A.vals).max(initial=0.0)
    return bool(np.abs(A.vals - At.vals).max(initial=0.0) <= tol * max(scale, 1.0))


@dataclass
class AmgParams:
    """src/amg.py:41-66."""
    coarsest_size: int = 200
    max_levels: int = 25
    theta_amg: float = 0.08
    smoother_theta: float = 0.0
    pre_sweeps: int = 1
    post_sweeps: int = 1
    cycle: str = "k"
    krylov: str = "auto"


@dataclass
class Level:
    A: Csr
    groups: Optional[list] = None
    smoother: Optional[ScmSmoother] = None
    aggregates: Optional[np.ndarray] = None


@dataclass
class Hierarchy:
    levels: list
    coarsest_lu: tuple
    params: AmgParams
    symmetric: bool


def build_hierarchy(A_p: Csr, params: AmgParams | None = None) -> Hierarchy:
    """src/amg.py:143-174."""
    params = params or AmgParams()
    levels = []
    A_l = A_p
    sym = is_symmetric(A_p)
    while True:
        if A_l.nrows <= params.coarsest_size or len(levels) + 1 >= params.max_levels:
            levels.append(Level(A_l))
            break
        agg, na = pairwise_aggregate(A_l, params.theta_amg)
        if na > 0.9 * A_l.nrows:
            levels.append(Level(A_l))
            break
        groups = vertices_grouping(strong_connections(A_l, params.smoother_theta))
        levels.append(Level(A_l, groups, ScmSmoother(A_l, groups), agg))
        A_l = galerkin(A_l, agg, na)
    try:
        lu = scipy.linalg.lu_factor(levels[-1].A.to_dense())
    except (ValueError, scipy.linalg.LinAlgError) as exc:
        raise RuntimeError(f"coarsest-level dense factorization failed: {exc}") from exc
    return Hierarchy(levels, lu, params, sym)


def _fcg_steps(A, rhs, precond, steps=2):
    """src/amg.py:177-196."""
    x = np.zeros_like(rhs)
    r = rhs.copy()
    dirs = []
    for _ in range(steps):
        if norm2(r) == 0.0:
            break
        z = precond(r)
        p = z
        for pj, apj, pap in dirs:
            p = p - (dot(z, apj) / pap) * pj
        ap = spmv(A, p)
        pap = dot(p, ap)
        if pap <= 0.0 or not np.isfinite(pap):
            break
        alpha = dot(p, r) / pap
        x = x + alpha * p
        r = r - alpha * ap
        dirs.append((p, ap, pap))
    return x


def _fgmres_steps(A, rhs, precond, steps=2):
    """src/amg.py:199-225."""
    beta = norm2(rhs)
    if beta == 0.0:
        return np.zeros_like(rhs)
    basis = [rhs / beta]
    zs = []
    H = np.zeros((steps + 1, steps))
    m_eff = steps
    for j in range(steps):
        z = precond(basis[j])
        zs.append(z)
        w = spmv(A, z)
        for i in range(j + 1):
            H[i, j] = dot(w, basis[i])
            w = w - H[i, j] * basis[i]
        H[j + 1, j] = norm2(w)
        if H[j + 1, j] == 0.0:
            m_eff = j + 1
            break
        basis.append(w / H[j + 1, j])
    e1 = np.zeros(m_eff + 1)
    e1[0] = beta
    y, *_ = np.linalg.lstsq(H[:m_eff + 1, :m_eff], e1, rcond=None)
    x = np.zeros_like(rhs)
    for i in range(m_eff):
        x = x + y[i] * zs[i]
    return x


def amg_cycle(h: Hierarchy, r, cycle=None, coarse_solve=None):
    """src/amg.py:228-242.  ``coarse_solve`` optionally replaces the
    coarsest lu_solve (used by tests that feed the product's factors)."""
    if r.shape != (h.levels[0].A.nrows,):
        raise ValueError("dimension mismatch: expected residual of length "
                         f"{h.levels[0].A.nrows}")
    cycle = cycle or h.params.cycle
    use_fcg = h.params.krylov == "fcg" or (h.params.krylov == "auto" and h.symmetric)
    return _cycle_at(h, 0, np.asarray(r, dtype=np.float64), cycle, use_fcg, coarse_solve)


def _cycle_at(h, l, r, cycle, use_fcg, coarse_solve):
    """src/amg.py:245-267."""
    lvl = h.levels[l]
    if l == len(h.levels) - 1:
        if coarse_solve is not None:
            return coarse_solve(r)
        return scipy.linalg.lu_solve(h.coarsest_lu, r)
    p = h.params
    x = lvl.smoother.apply(r, np.zeros_like(r), sweeps=p.pre_sweeps, direction="forward")
    resid = r - spmv(lvl.A, x)
    rc = np.bincount(lvl.aggregates, weights=resid, minlength=h.levels[l + 1].A.nrows)
    if cycle == "v" or l + 1 == len(h.levels) - 1:
        ec = _cycle_at(h, l + 1, rc, cycle, use_fcg, coarse_solve)
    else:
        A_c = h.levels[l + 1].A
        pre = lambda s: _cycle_at(h, l + 1, s, cycle, use_fcg, coarse_solve)  # noqa: E731
        ec = (_fcg_steps if use_fcg else _fgmres_steps)(A_c, rc, pre)
    x = x + ec[lvl.aggregates]
    x = lvl.smoother.apply(r, x, sweeps=p.post_sweeps, direction="backward")
    return x


# --------------------------------------------------------------------------
# BILU(0) (src/ilu.py)
# --------------------------------------------------------------------------


def level_schedule(ptr, cols, n):
    """src/ilu.py:38-59: level(i) = 1 + max level of in-pattern predecessors;
    orientation inferred from the off-diagonal pattern."""
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(ptr))
    off = rows != cols
    below = cols[off] < rows[off]
    if below.size and below.any() and not below.all():
        raise ValueError("pattern is neither lower nor upper triangular")
    lower = bool(below.all()) if below.size else True
    level = np.zeros(n, dtype=np.int64)
    pl, cl = ptr.tolist(), cols.tolist()
    lv = [0] * n
    order = range(n) if lower else range(n - 1, -1, -1)
    for i in order:
        m = 0
        for p in range(pl[i], pl[i + 1]):
            j = cl[p]
            if j != i and lv[j] > m:
                m = lv[j]
        lv[i] = 1 + m
    level[:] = lv
    nlev = int(level.max(initial=1))
    order_rows = np.argsort(level, kind="stable")
    counts = np.bincount(level, minlength=nlev + 1)[1:]
    bounds = np.concatenate([[0], np.cumsum(counts)])
    return [order_rows[bounds[i]:bounds[i + 1]].astype(np.int64) for i in range(nlev)]


@dataclass
class Bilu:
    """BiluFactors (src/ilu.py:110-131): strict-lower L blocks, strict-upper U
    blocks (both canonical, ascending columns), inverted U diagonal."""
    n: int
    b: int
    l_ptr: np.ndarray
    l_cols: np.ndarray
    l_vals: np.ndarray
    u_ptr: np.ndarray
    u_cols: np.ndarray
    u_vals: np.ndarray
    u_diag_inv: np.ndarray
    l_levels: list
    u_levels: list
    perturbed_rows: list = field(default_factory=list)


def _invert_pivot(block, row, perturbed):
    """src/ilu.py:134-147."""
    try:
        return invert_small_blocks(block[np.newaxis])[0]
    except np.linalg.LinAlgError:
        fro = float(np.sqrt(np.sum(block * block)))
        if fro == 0.0:
            raise np.linalg.LinAlgError(f"singular pivot block at row {row}") from None
        warnings.warn(f"bilu0: perturbing singular pivot block at row {row}",
                      RuntimeWarning, stacklevel=3)
        perturbed.append(row)
        bumped = block + 1e-8 * fro * np.eye(block.shape[0])
        try:
            return invert_small_blocks(bumped[np.newaxis])[0]
        except np.linalg.LinAlgError:
            raise np.linalg.LinAlgError(f"singular pivot block at row {row}") from None


def _as_block(A):
    if isinstance(A, Csr):
        return Bsr(1, A.nrows, A.ncols, A.ptr, A.cols, A.vals.reshape(-1, 1, 1))
    return A


def _split_factors(A, vals, uinv, perturbed):
    n, b = A.nrows, A.b
    ptr, cols = A.ptr, A.cols
    rows = A.rows()
    lower = cols < rows
    upper = cols > rows
    lp = np.zeros(n + 1, dtype=np.int64)
    np.add.at(lp[1:], rows[lower], 1)
    np.cumsum(lp, out=lp)
    up = np.zeros(n + 1, dtype=np.int64)
    np.add.at(up[1:], rows[upper], 1)
    np.cumsum(up, out=up)
    # level schedules of L (strict lower + diag) and U (diag + strict upper)
    lcols_full, ucols_full = cols[cols <= rows], cols[cols >= rows]
    lp_full = lp + np.arange(n + 1)
    up_full = up + np.arange(n + 1)
    return Bilu(n, b, lp, cols[lower].copy(), vals[lower].copy(), up, cols[upper].copy(),
                vals[upper].copy(), uinv, level_schedule(lp_full, lcols_full, n),
                level_schedule(up_full, ucols_full, n), perturbed)


def bilu0_factorize(A) -> Bilu:
    """src/ilu.py:150-193: row-wise IKJ restricted to the pattern, 3x3 `@`
    products, pivot inversion with perturbation fallback.  Plain loop form."""
    A = _as_block(A)
    n, b = A.nrows, A.b
    if A.nrows != A.ncols:
        raise ValueError("factorization needs a square matrix")
    vals = A.vals.copy()
    ptr, cols = A.ptr, A.cols
    uinv = np.empty((n, b, b))
    perturbed: list = []
    for i in range(n):
        lo, hi = int(ptr[i]), int(ptr[i + 1])
        row_cols = cols[lo:hi]
        dk = int(np.searchsorted(row_cols, i))
        if dk >= hi - lo or row_cols[dk] != i:
            raise ValueError(f"diagonal block missing in row {i}")
        for p in range(lo, lo + dk):
            k = int(cols[p])
            vals[p] = vals[p] @ uinv[k]
            klo, khi = int(ptr[k]), int(ptr[k + 1])
            kcols = cols[klo:khi]
            for q in range(p + 1, hi):
                j = int(cols[q])
                pos = int(np.searchsorted(kcols, j))
                if pos < kcols.shape[0] and kcols[pos] == j:
                    vals[q] = vals[q] - vals[p] @ vals[klo + pos]
        uinv[i] = _invert_pivot(vals[lo + dk], i, perturbed)
    return _split_factors(A, vals, uinv, perturbed)


def bilu0_factorize_fast(A) -> Bilu:
    """Same arithmetic as :func:`bilu0_factorize`, batched over the rows of one
    L-level (rows of a level only read finished rows of earlier levels), and
    over lower-entry position t in ascending order (the reference's p loop).
    Batched `@` is bitwise equal to per-block `@` (tests/test_oracle.py)."""
    A = _as_block(A)
    n, b = A.nrows, A.b
    vals = A.vals.copy()
    ptr, cols = A.ptr, A.cols
    rows = A.rows()
    diag_pos = np.flatnonzero(cols == rows)
    if diag_pos.shape[0] != n:
        raise ValueError("diagonal block missing")
    nlow = diag_pos - ptr[:-1]
    # (row, p, q, kpos) update list: q > p in row i with cols[q] in row k=cols[p]
    key = rows * (A.ncols + 1) + cols          # sorted ascending (canonical)
    rows_l = rows[cols < rows]
    p_l = np.flatnonzero(cols < rows)
    # candidate (p, q) pairs: all q in the same row after p
    cnt = ptr[rows_l + 1] - p_l - 1
    p_rep = np.repeat(p_l, cnt)
    q_rep = p_rep + 1 + (np.arange(cnt.sum()) - np.repeat(np.cumsum(cnt) - cnt, cnt))
    k_rep = cols[p_rep]
    j_rep = cols[q_rep]
    want = k_rep * (A.ncols + 1) + j_rep
    pos = np.searchsorted(key, want)
    pos_c = np.minimum(pos, key.shape[0] - 1)
    hit = key[pos_c] == want
    p_rep, q_rep, kpos = p_rep[hit], q_rep[hit], pos_c[hit]
    t_of_p = p_l - ptr[rows_l]
    t_lookup = np.full(A.nnz, -1, dtype=np.int64)
    t_lookup[p_l] = t_of_p
    lev_rows = level_schedule(ptr, cols * (cols <= rows) + rows * (cols > rows), n)
    row_level = np.empty(n, dtype=np.int64)
    for li, lr in enumerate(lev_rows):
        row_level[lr] = li
    uinv = np.empty((n, b, b))
    perturbed: list = []
    upd_level = row_level[rows[p_rep]]
    upd_t = t_lookup[p_rep]
    order = np.lexsort((upd_t, upd_level))
    p_rep, q_rep, kpos, upd_level, upd_t = (p_rep[order], q_rep[order], kpos[order],
                                            upd_level[order], upd_t[order])
    lp_level = row_level[rows_l]
    for li, lr in enumerate(lev_rows):
        maxt = int(nlow[lr].max(initial=0))
        for t in range(maxt):
            sel = lr[nlow[lr] > t]
            p = ptr[sel] + t
            vals[p] = vals[p] @ uinv[cols[p]]
            a = np.searchsorted(upd_level, li, "left")
            z = np.searchsorted(upd_level, li, "right")
            seg_t = upd_t[a:z]
            s0 = a + np.searchsorted(seg_t, t, "left")
            s1 = a + np.searchsorted(seg_t, t, "right")
            if s1 > s0:
                pp, qq, kk = p_rep[s0:s1], q_rep[s0:s1], kpos[s0:s1]
                vals[qq] = vals[qq] - vals[pp] @ vals[kk]
        d = diag_pos[lr]
        try:
            uinv[lr] = invert_small_blocks(vals[d])
        except np.linalg.LinAlgError:
            for i, di in zip(lr.tolist(), d.tolist()):
                uinv[i] = _invert_pivot(vals[di], i, perturbed)
    del lp_level
    return _split_factors(A, vals, uinv, perturbed)


def bilu_apply(F: Bilu, r, sequential=False):
    """src/ilu.py:196-223: level-scheduled L then U substitution; block
    products through einsum, row sums through reduceat."""
    n, b = F.n, F.b
    if r.shape != (n * b,):
        raise ValueError(f"dimension mismatch: expected vector of length {n * b}")
    r2 = np.asarray(r, dtype=np.float64).reshape(n, b)
    z2 = r2.copy()

    def level_sums(ptr, cols, vals, lvl, x2):
        lo = ptr[lvl]
        ln = ptr[lvl + 1] - lo
        lptr = np.zeros(lvl.shape[0] + 1, dtype=np.int64)
        np.cumsum(ln, out=lptr[1:])
        idx = np.repeat(lo - lptr[:-1], ln) + np.arange(int(lptr[-1]))
        prods = np.einsum("kij,kj->ki", vals[idx], x2[cols[idx]])
        return segment_sums(prods, lptr)

    if sequential:
        for i in range(n):
            lvl = np.array([i])
            z2[i] = r2[i] - level_sums(F.l_ptr, F.l_cols, F.l_vals, lvl, z2)[0]
        y2 = np.zeros_like(z2)
        for i in range(n - 1, -1, -1):
            lvl = np.array([i])
            rhs = z2[i] - level_sums(F.u_ptr, F.u_cols, F.u_vals, lvl, y2)[0]
            y2[i] = np.einsum("kij,kj->ki", F.u_diag_inv[i:i + 1], rhs[np.newaxis, :])[0]
        return y2.reshape(-1)
    for lvl in F.l_levels:
        z2[lvl] = r2[lvl] - level_sums(F.l_ptr, F.l_cols, F.l_vals, lvl, z2)
    y2 = np.zeros_like(z2)
    for lvl in F.u_levels:
        t = level_sums(F.u_ptr, F.u_cols, F.u_vals, lvl, y2)
        y2[lvl] = np.einsum("kij,kj->ki", F.u_diag_inv[lvl], z2[lvl] - t)
    return y2.reshape(-1)


# --------------------------------------------------------------------------
# CPR + GMRES (src/cpr.py)
# --------------------------------------------------------------------------


@dataclass
class SolverConfig:
    """src/cpr.py:63-111 (solver knobs used on the path)."""
    theta: float = 0.0
    mu: int = 0
    m: int = 28
    tol: float = 1e-5
    max_restarts: int = 100
    cycle: str = "k"
    coarsest_size: int = 200
    sweeps: int = 1
    mu_counter: str = "inner"
    theta_amg: float = 0.08
    max_levels: int = 25
    krylov: str = "auto"

    def amg_params(self):
        return AmgParams(self.coarsest_size, self.max_levels, self.theta_amg, self.theta,
                         self.sweeps, self.sweeps, self.cycle, self.krylov)


def pressure_matrix(A):
    """src/cpr.py:148-153."""
    if isinstance(A, Bsr):
        return Csr(A.nrows, A.ncols, A.ptr.copy(), A.cols.copy(), A.vals[:, 0, 0].copy())
    return A


def fingerprint_of(A):
    """src/cpr.py:141-145."""
    if isinstance(A, Bsr):
        return (A.nrows * A.b, A.nnz)
    return (A.nrows, A.nnz)


@dataclass
class Cpr:
    """CprPreconditioner (src/cpr.py:156-165)."""
    pidx: np.ndarray
    fine_size: int
    hierarchy: Hierarchy
    bilu: Bilu
    A: object
    fingerprint: tuple
    coarse_solve: object = None

    def apply(self, r, workers=1):
        return apply_cpr(self, r)


def build_cpr(A, config: SolverConfig | None = None, fast_bilu=True) -> Cpr:
    """src/cpr.py:168-175."""
    config = config or SolverConfig()
    if isinstance(A, Bsr):
        pidx = np.arange(A.nrows, dtype=np.int64) * A.b
        fine = A.nrows * A.b
    else:
        pidx = np.arange(A.nrows, dtype=np.int64)
        fine = A.nrows
    h = build_hierarchy(pressure_matrix(A), config.amg_params())
    F = bilu0_factorize_fast(A) if fast_bilu else bilu0_factorize(A)
    return Cpr(pidx, fine, h, F, A, fingerprint_of(A))


def apply_cpr(B: Cpr, r):
    """src/cpr.py:178-186: z = z1 + BILU^{-1}(r - A z1), z1 = Pi AMG(Pi^T r)."""
    if r.shape != (B.fine_size,):
        raise ValueError(f"dimension mismatch: expected residual of length {B.fine_size}")
    zp = amg_cycle(B.hierarchy, r[B.pidx], coarse_solve=B.coarse_solve)
    z1 = np.zeros(B.fine_size)
    z1[B.pidx] = zp
    r2 = r - spmv(B.A, z1)
    return z1 + bilu_apply(B.bilu, r2)


@dataclass
class GmresResult:
    x: np.ndarray
    outer: int
    inner: int
    converged: bool
    rel_residual: float
    history: list = field(default_factory=list)


def _solve_upper(R, g):
    """src/cpr.py:224-228."""
    if np.all(np.abs(np.diag(R)) > 0.0):
        return scipy.linalg.solve_triangular(R, g)
    y, *_ = np.linalg.lstsq(R, g, rcond=None)
    return y


def gmres_solve(A, b, x0, B, m=28, max_restarts=100, tol=1e-5) -> GmresResult:
    """src/cpr.py:231-316.  Additionally records the Givens residual estimate
    |g_{j+1}|/beta0 per inner step and ('explicit', rel) per restart."""
    n = b.shape[0]
    x = np.zeros(n) if x0 is None else np.asarray(x0, dtype=np.float64).copy()
    b = np.asarray(b, dtype=np.float64)
    r = b - spmv(A, x)
    beta0 = norm2(r)
    hist: list = []
    if not np.isfinite(beta0):
        raise FloatingPointError("non-finite initial residual in gmres_solve")
    if beta0 == 0.0:
        return GmresResult(x, 0, 0, True, 0.0, hist)
    inner_total = 0
    converged = False
    rel = 1.0
    outer = 0
    for outer in range(1, max_restarts + 1):
        beta = norm2(r)
        if beta == 0.0:
            converged = True
            break
        V = np.zeros((m + 1, n))
        V[0] = r / beta
        H = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        j_used = 0
        shrink = None
        for j in range(m):
            z = V[j] if B is None else B.apply(V[j])
            w = spmv(A, z)
            if not np.isfinite(w).all():
                raise FloatingPointError("non-finite Krylov vector in gmres_solve")
            for i in range(j + 1):
                H[i, j] = dot(w, V[i])
                w = w - H[i, j] * V[i]
            H[j + 1, j] = norm2(w)
            j_used = j + 1
            inner_total += 1
            breakdown = H[j + 1, j] == 0.0
            if not breakdown:
                V[j + 1] = w / H[j + 1, j]
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            denom = float(np.hypot(H[j, j], H[j + 1, j]))
            if denom == 0.0:
                cs[j], sn[j] = 1.0, 0.0
            else:
                cs[j], sn[j] = H[j, j] / denom, H[j + 1, j] / denom
            H[j, j] = denom
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            hist.append(abs(g[j + 1]) / beta0)
            if breakdown:
                shrink = j + 1
                break
            if abs(g[j + 1]) < tol * beta0:
                break
        y = _solve_upper(H[:j_used, :j_used], g[:j_used])
        u = y @ V[:j_used]
        x_new = x + (u if B is None else B.apply(u))
        r_new = b - spmv(A, x_new)
        if not np.isfinite(r_new).all():
            raise FloatingPointError("non-finite residual in gmres_solve (divergence)")
        x, r = x_new, r_new
        rel = norm2(r) / beta0
        hist.append(("explicit", rel))
        if shrink is not None:
            m = shrink
        if rel < tol:
            converged = True
            break
    return GmresResult(x, outer, inner_total, converged, rel, hist)


def ascpr_gmres_sequence(systems, mu, config: SolverConfig | None = None):
    """src/cpr.py:349-382 (reuse rule src/cpr.py:204-212).  Returns a list of
    (outer, inner, converged, rel, rebuilt, x) and the setup-call count."""
    config = config or SolverConfig()
    prev, prev_iters, calls = None, None, 0
    out = []
    for k, (A, rhs) in enumerate(systems, start=1):
        reuse = (k > 1 and prev is not None and prev_iters is not None and prev_iters <= mu
                 and prev.fingerprint == fingerprint_of(A))
        if reuse:
            B = prev
        else:
            B = build_cpr(A, config)
            calls += 1
        res = gmres_solve(A, rhs, None, B, config.m, config.max_restarts, config.tol)
        prev = B
        prev_iters = res.inner if config.mu_counter == "inner" else res.outer
        out.append((res.outer, res.inner, res.converged, res.rel_residual, not reuse, res.x))
    return out, calls


# --------------------------------------------------------------------------
# synthetic problems (src/problems.py)
# --------------------------------------------------------------------------


def neighbor_links(nx, ny, nz):
    """src/problems.py:57-71, vectorised in the same (iz, iy, ix, axis) order."""
    n = nx * ny * nz
    c = np.arange(n, dtype=np.int64)
    ix = c % nx
    iy = (c // nx) % ny
    iz = c // (nx * ny)
    cand_b = np.stack([c + 1, c + nx, c + nx * ny], axis=1)
    valid = np.stack([ix + 1 < nx, iy + 1 < ny, iz + 1 < nz], axis=1)
    axis = np.broadcast_to(np.arange(3, dtype=np.int64), (n, 3))
    a = np.broadcast_to(c[:, None], (n, 3))
    return np.stack([a[valid], cand_b[valid], axis[valid]], axis=1)


def assemble_step(ncells, links, aniso, perm, conv_scale, couple, drift) -> Bsr:
    """src/problems.py:113-155."""
    a, bv, axis = links[:, 0], links[:, 1], links[:, 2]
    trans = aniso[axis] * 2.0 / (1.0 / perm[a] + 1.0 / perm[bv])
    conv = conv_scale[a] * trans
    nl = links.shape[0]
    rows = np.empty(2 * nl + ncells, dtype=np.int64)
    cols = np.empty_like(rows)
    blocks = np.zeros((rows.shape[0], 3, 3))
    rows[:nl], cols[:nl] = a, bv
    blocks[:nl, 0, 0] = -trans
    rows[nl:2 * nl], cols[nl:2 * nl] = bv, a
    blocks[nl:2 * nl, 0, 0] = -trans
    blocks[nl:2 * nl, 1, 1] = -conv
    blocks[nl:2 * nl, 2, 2] = -0.8 * conv
    blocks[nl:2 * nl, 1, 0] = -drift * 0.5 * conv
    blocks[nl:2 * nl, 2, 0] = -drift * 0.3 * conv
    d = 2 * nl + np.arange(ncells)
    rows[d] = np.arange(ncells)
    cols[d] = np.arange(ncells)
    p_diag = 0.05 * perm.copy()
    w_diag = np.full(ncells, 1.0)
    o_diag = np.full(ncells, 1.0)
    np.add.at(p_diag, a, trans)
    np.add.at(p_diag, bv, trans)
    np.add.at(w_diag, bv, conv)
    np.add.at(o_diag, bv, 0.8 * conv)
    blocks[d, 0, 0] = p_diag
    blocks[d, 1, 1] = w_diag
    blocks[d, 2, 2] = o_diag
    blocks[d, 0, 1] = drift * couple[:, 0]
    blocks[d, 0, 2] = drift * couple[:, 1]
    blocks[d, 1, 0] = drift * couple[:, 2]
    blocks[d, 1, 2] = drift * 0.2 * couple[:, 3]
    blocks[d, 2, 0] = drift * couple[:, 4]
    blocks[d, 2, 1] = drift * 0.2 * couple[:, 5]
    return bsr_from_block_coo(3, rows, cols, blocks, (ncells, ncells), sum_duplicates=True)


def manufactured_solution(ncells):
    """src/problems.py:93-97."""
    t = np.linspace(0.0, 2.0 * np.pi, ncells, endpoint=False)
    xs = np.empty(3 * ncells)
    xs[0::3] = 1.0 + 0.3 * np.sin(t)
    xs[1::3] = 0.4 + 0.2 * np.cos(2.0 * t)
    xs[2::3] = 0.5 - 0.1 * np.sin(3.0 * t)
    return xs


def generate_blackoil_like_sequence(nx, ny, nz, nsteps, drift, seed, with_rhs=True):
    """src/problems.py:74-110: list of (A, b) with b = spmv(A, x*)."""
    if min(nx, ny, nz) < 1 or nsteps < 1:
        raise ValueError("grid dimensions and nsteps must be >= 1")
    rng = np.random.default_rng(seed)
    n = nx * ny * nz
    links = neighbor_links(nx, ny, nz)
    aniso = np.array([1.0, 1.0, 0.2])
    logk = rng.normal(0.0, 1.0, n)
    conv_scale = rng.uniform(0.2, 0.5, n)
    couple = rng.standard_normal((n, 6)) * 0.5
    xs = manufactured_solution(n)
    out = []
    for step in range(nsteps):
        if step > 0:
            logk = logk + drift * rng.normal(0.0, 1.0, n)
            conv_scale = conv_scale * np.exp(drift * rng.normal(0.0, 1.0, n))
        A = assemble_step(n, links, aniso, np.exp(logk), conv_scale, couple, drift)
        out.append((A, spmv(A, xs) if with_rhs else None))
    return out


def pressure_operator(nx, ny, nz, seed=0, drift=0.0):
    """C2 input: the (0,0) block of the first generated system (depends only on
    the first RNG draw); SURVEY.md Appendix B.2."""
    rng = np.random.default_rng(seed)
    n = nx * ny * nz
    links = neighbor_links(nx, ny, nz)
    logk = rng.normal(0.0, 1.0, n)
    conv = rng.uniform(0.2, 0.5, n)
    cpl = rng.standard_normal((n, 6)) * 0.5
    A = assemble_step(n, links, np.array([1.0, 1.0, 0.2]), np.exp(logk), conv, cpl, drift)
    return pressure_matrix(A)
