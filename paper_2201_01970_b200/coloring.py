"""Strong-connection graph and greedy multi-colour grouping (drop-in for
cprkit.coloring).  The greedy heap algorithm runs in the host C++ setup
library (csrc/setup.cpp) and reproduces the reference's groups bit-exactly
(src/coloring.py:79-256)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .sparse import BlockCsrMatrix, CsrMatrix

__all__ = ["StrongConnectionMatrix", "ColorPartition", "strong_connections",
           "vertices_grouping", "verify_partition", "PartitionReport", "dump_partition",
           "load_partition"]


@dataclass
class StrongConnectionMatrix:
    """Pattern-only CSR of S(A, theta); no self edges (src/coloring.py:39-76)."""

    n: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    theta: float

    def neighbors(self, i: int) -> np.ndarray:
        return self.col_idx[self.row_ptr[i]:self.row_ptr[i + 1]]

    def degrees(self) -> np.ndarray:
        return np.diff(self.row_ptr)

    @property
    def n_edges(self) -> int:
        return int(self.col_idx.shape[0])

    def symmetrized(self) -> "StrongConnectionMatrix":
        rows = np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.row_ptr))
        rr = np.concatenate([rows, self.col_idx])
        cc = np.concatenate([self.col_idx, rows])
        order = np.lexsort((cc, rr))
        rr, cc = rr[order], cc[order]
        if rr.size:
            keep = np.concatenate(([True], (np.diff(rr) != 0) | (np.diff(cc) != 0)))
            rr, cc = rr[keep], cc[keep]
        ptr = np.zeros(self.n + 1, dtype=np.int64)
        np.add.at(ptr[1:], rr, 1)
        np.cumsum(ptr, out=ptr)
        return StrongConnectionMatrix(self.n, ptr, cc, self.theta)

    def has_edge(self, i: int, j: int) -> bool:
        cols = self.neighbors(i)
        k = np.searchsorted(cols, j)
        return bool(k < cols.shape[0] and cols[k] == j)


def _scalar_view(A):
    if isinstance(A, BlockCsrMatrix) or int(getattr(A, "block_size", 1)) > 1 or \
            np.ndim(getattr(A, "values", np.zeros(1))) == 3:
        return A.frobenius()
    return A


def strong_connections(A, theta: float, workers: int = 1) -> StrongConnectionMatrix:
    """S_ij = 1 iff |a_ij| > theta * sum_k |a_ik| and i != j (src/coloring.py:79-114)."""
    if not 0.0 <= theta <= 1.0:
        raise ValueError(f"theta must lie in [0, 1], got {theta}")
    A = _scalar_view(A)
    if A.nrows != A.ncols:
        raise ValueError("strong connections need a square matrix")
    n = A.nrows
    ptr = np.ascontiguousarray(A.row_ptr, dtype=np.int64)
    cols = np.ascontiguousarray(A.col_idx, dtype=np.int64)
    vals = np.ascontiguousarray(A.values, dtype=np.float64)
    sp = np.zeros(n + 1, dtype=np.int64)
    sc = np.zeros(max(cols.shape[0], 1), dtype=np.int64)
    N.check(N.lib().cprb_strong_connections(n, N.p64(ptr), N.p64(cols), N.pf64(vals), float(theta),
                                            N.p64(sp), N.p64(sc)))
    return StrongConnectionMatrix(n, sp, sc[:sp[-1]].copy(), float(theta))


@dataclass
class ColorPartition:
    """Ordered disjoint vertex groups; colours are 1-based in vertex_color."""

    groups: list
    n: int
    vertex_color: np.ndarray

    @property
    def c(self) -> int:
        return len(self.groups)

    def perm(self) -> np.ndarray:
        return np.concatenate(self.groups) if self.groups else np.zeros(0, dtype=np.int64)

    @classmethod
    def from_groups(cls, groups, n: int) -> "ColorPartition":
        vc = np.zeros(n, dtype=np.int64)
        for c, g in enumerate(groups, start=1):
            vc[g] = c
        return cls([np.asarray(g, dtype=np.int64) for g in groups], n, vc)


def vertices_grouping(S: StrongConnectionMatrix) -> ColorPartition:
    """Repeated greedy splitting rounds over S ∪ S^T (src/coloring.py:238-256)."""
    n = S.n
    perm = np.zeros(n, dtype=np.int64)
    sizes = np.zeros(max(n, 1), dtype=np.int64)
    nc = np.zeros(1, dtype=np.int64)
    sp = np.ascontiguousarray(S.row_ptr, dtype=np.int64)
    sc = np.ascontiguousarray(S.col_idx, dtype=np.int64)
    if sc.size == 0:
        sc = np.zeros(1, dtype=np.int64)
    N.check(N.lib().cprb_vertices_grouping(n, N.p64(sp), N.p64(sc), N.p64(perm), N.p64(sizes),
                                           N.p64(nc)))
    bounds = np.concatenate([[0], np.cumsum(sizes[:int(nc[0])])])
    groups = [perm[bounds[i]:bounds[i + 1]].copy() for i in range(int(nc[0]))]
    return ColorPartition.from_groups(groups, n)


@dataclass
class PartitionReport:
    checks: dict
    details: dict

    @property
    def ok(self) -> bool:
        return all(self.checks.values())

    def lines(self):
        return [f"{'PASS' if v else 'FAIL'} {k}" + (f" ({self.details[k]})" if k in self.details else "")
                for k, v in self.checks.items()]


def verify_partition(A, theta: float, partition: ColorPartition) -> PartitionReport:
    """Audit a partition against the grouping contracts (src/coloring.py:273-326)."""
    S = strong_connections(A, theta).symmetrized()
    n = S.n
    checks, details = {}, {}
    counts = np.zeros(n, dtype=np.int64)
    for g in partition.groups:
        np.add.at(counts, g, 1)
    checks["cover"] = bool((counts >= 1).all()) and partition.n == n
    checks["disjoint"] = bool((counts <= 1).all())
    color = partition.vertex_color
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(S.row_ptr))
    ok_c = True
    if S.n_edges:
        same = color[rows] == color[S.col_idx]
        ok_c = not bool(same.any())
        if not ok_c:
            k = int(np.flatnonzero(same)[0])
            details["independent_groups"] = (f"strong edge ({rows[k]}, {S.col_idx[k]}) inside "
                                             f"color {color[rows[k]]}")
    checks["independent_groups"] = ok_c
    bound = int(S.degrees().max(initial=0)) + 1
    checks["color_bound"] = partition.c <= bound
    details["color_bound"] = f"c={partition.c} bound={bound}"
    scalar = _scalar_view(A)
    sr = np.repeat(np.arange(scalar.nrows, dtype=np.int64), np.diff(scalar.row_ptr))
    same_group = color[sr] == color[scalar.col_idx]
    off = same_group & (sr != scalar.col_idx)
    ok_blocks = True
    if off.any():
        srow, scol = sr[off], scalar.col_idx[off]
        ok_blocks = not any(S.has_edge(int(a), int(b)) for a, b in zip(srow, scol))
    checks["group_strong_blocks_diagonal"] = ok_blocks
    if theta == 0.0:
        checks["theta0_group_value_diagonal"] = not bool(np.any(scalar.values[off] != 0.0))
    return PartitionReport(checks, details)


def dump_partition(partition: ColorPartition, fh) -> None:
    for g in partition.groups:
        fh.write(" ".join(str(int(v)) for v in g) + "\n")


def load_partition(fh, n: int) -> ColorPartition:
    groups = []
    for line in fh:
        line = line.strip()
        if line:
            groups.append(np.array([int(t) for t in line.split()], dtype=np.int64))
    return ColorPartition.from_groups(groups, n)
