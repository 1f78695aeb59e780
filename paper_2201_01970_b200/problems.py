"""Synthetic black-oil-like Jacobian sequences (drop-in for
cprkit.problems.generate_blackoil_like_sequence, src/problems.py:74-155).

The assembly is written directly into the 7-point BSR structure (no COO
sort): each row's blocks are ordered (z-, y-, x-, diag, x+, y+, z+), which is
the canonical ascending-column order.  Every value is produced by the same
elementwise float64 operations, in the same accumulation order, as the
reference's COO assembly (np.add.at over links in (cell, axis) order), so the
matrices and right-hand sides are bitwise identical for the same seed
(tests/test_problems.py checks this against the reference's fixtures).
The right-hand side b = A x* uses the reference's row-sum order
(a0 + pairwise(rest) over the expanded row, src/sparse.py:322-351).
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .sparse import BlockCsrMatrix, CsrMatrix

__all__ = ["ProblemSequence", "generate_blackoil_like_sequence", "poisson_2d",
           "pressure_operator", "manufactured_solution", "save_sequence", "load_sequence"]


@dataclass
class ProblemSequence:
    systems: list
    provenance: dict = field(default_factory=dict)

    @property
    def block_size(self) -> int:
        return int(getattr(self.systems[0][0], "block_size", 1))

    def __len__(self) -> int:
        return len(self.systems)


def _pairwise_rows(E: np.ndarray) -> np.ndarray:
    """numpy pairwise summation applied to every row of E (n columns)."""
    n = E.shape[1]
    if n < 8:
        s = np.zeros(E.shape[0])
        for t in range(n):
            s = s + E[:, t]
        return s
    if n <= 128:
        r = [E[:, k].copy() for k in range(8)]
        i = 8
        while i + 8 <= n:
            for k in range(8):
                r[k] = r[k] + E[:, i + k]
            i += 8
        s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            s = s + E[:, i]
            i += 1
        return s
    n2 = n // 2
    n2 -= n2 % 8
    return _pairwise_rows(E[:, :n2]) + _pairwise_rows(E[:, n2:])


def bsr_matvec_reference_order(A: BlockCsrMatrix, x: np.ndarray) -> np.ndarray:
    """Host y = A x with the reference's expanded-row reduceat order; used only
    to synthesise right-hand sides (input generation, not the solve path)."""
    b = A.block_size
    cnt = np.diff(A.row_ptr)
    y = np.zeros(A.nrows * b)
    x2 = x.reshape(-1, b)
    for k in np.unique(cnt):
        rows = np.flatnonzero(cnt == k)
        if k == 0:
            continue
        pos = A.row_ptr[rows][:, None] + np.arange(k)[None, :]           # (R, k)
        blk = A.values[pos]                                              # (R, k, b, b)
        xv = x2[A.col_idx[pos]]                                          # (R, k, b)
        for r in range(b):
            E = (blk[:, :, r, :] * xv).reshape(rows.shape[0], k * b)     # (m, c) order
            y[rows * b + r] = E[:, 0] + _pairwise_rows(E[:, 1:])
    return y


def manufactured_solution(ncells: int) -> np.ndarray:
    """x* of src/problems.py:93-97."""
    t = np.linspace(0.0, 2.0 * np.pi, ncells, endpoint=False)
    xs = np.empty(3 * ncells)
    xs[0::3] = 1.0 + 0.3 * np.sin(t)
    xs[1::3] = 0.4 + 0.2 * np.cos(2.0 * t)
    xs[2::3] = 0.5 - 0.1 * np.sin(3.0 * t)
    return xs


class _Grid:
    def __init__(self, nx, ny, nz):
        self.nx, self.ny, self.nz = nx, ny, nz
        n = nx * ny * nz
        self.n = n
        c = np.arange(n, dtype=np.int64)
        ix, iy, iz = c % nx, (c // nx) % ny, c // (nx * ny)
        self.step = (1, nx, nx * ny)
        self.has_plus = (ix + 1 < nx, iy + 1 < ny, iz + 1 < nz)
        self.has_minus = (ix > 0, iy > 0, iz > 0)
        # slot order within a row: z-, y-, x-, diag, x+, y+, z+
        flags = np.stack([self.has_minus[2], self.has_minus[1], self.has_minus[0],
                          np.ones(n, dtype=bool), self.has_plus[0], self.has_plus[1],
                          self.has_plus[2]], axis=1)
        cnt = flags.sum(axis=1)
        self.ptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(cnt, out=self.ptr[1:])
        before = np.cumsum(flags, axis=1) - flags
        self.slot = np.where(flags, self.ptr[:-1, None] + before, -1)     # (n, 7)
        cols = np.empty(self.ptr[-1], dtype=np.int64)
        off = (-nx * ny, -nx, -1, 0, 1, nx, nx * ny)
        for s in range(7):
            m = flags[:, s]
            cols[self.slot[m, s]] = c[m] + off[s]
        self.cols = cols


def _assemble(g: _Grid, perm, conv_scale, couple, drift) -> BlockCsrMatrix:
    """Values of src/problems.py:113-155 written into the structured BSR."""
    n = g.n
    aniso = np.array([1.0, 1.0, 0.2])
    vals = np.zeros((g.ptr[-1], 3, 3))
    trans_p, conv_p = [], []
    for axis in range(3):
        a = np.flatnonzero(g.has_plus[axis])
        bb = a + g.step[axis]
        tr = aniso[np.full(a.shape[0], axis)] * 2.0 / (1.0 / perm[a] + 1.0 / perm[bb])
        cv = conv_scale[a] * tr
        trans_p.append((a, bb, tr))
        conv_p.append(cv)
        # row a, col b (upper): pressure diffusion only
        up = g.slot[a, 4 + axis]
        vals[up, 0, 0] = -tr
        # row b, col a (lower): diffusion, upwind convection, drift couplings
        lo = g.slot[bb, 2 - axis]
        vals[lo, 0, 0] = -tr
        vals[lo, 1, 1] = -cv
        vals[lo, 2, 2] = -0.8 * cv
        vals[lo, 1, 0] = -drift * 0.5 * cv
        vals[lo, 2, 0] = -drift * 0.3 * cv
    # diagonal accumulation in np.add.at order: first every link with the cell
    # as its lower end (links ordered x, y, z), then every link with the cell as
    # its upper end (ordered by the lower cell index: z, y, x)
    p_diag = 0.05 * perm.copy()
    w_diag = np.full(n, 1.0)
    o_diag = np.full(n, 1.0)
    for axis in range(3):
        a, _, tr = trans_p[axis]
        p_diag[a] = p_diag[a] + tr
    for axis in (2, 1, 0):
        _, bb, tr = trans_p[axis]
        cv = conv_p[axis]
        p_diag[bb] = p_diag[bb] + tr
        w_diag[bb] = w_diag[bb] + cv
        o_diag[bb] = o_diag[bb] + 0.8 * cv
    d = g.slot[:, 3]
    vals[d, 0, 0] = p_diag
    vals[d, 1, 1] = w_diag
    vals[d, 2, 2] = o_diag
    vals[d, 0, 1] = drift * couple[:, 0]
    vals[d, 0, 2] = drift * couple[:, 1]
    vals[d, 1, 0] = drift * couple[:, 2]
    vals[d, 1, 2] = drift * 0.2 * couple[:, 3]
    vals[d, 2, 0] = drift * couple[:, 4]
    vals[d, 2, 1] = drift * 0.2 * couple[:, 5]
    return BlockCsrMatrix(3, n, n, g.ptr, g.cols, vals)


def _cuda_ok() -> bool:
    try:
        import torch
        if not torch.cuda.is_available():
            return False
        from . import _native as N
        N.lib()
        return True
    except (ImportError, OSError, RuntimeError):
        return False


class _DeviceAssembler:
    """Device assembly (csrc/gen.cu) of one grid's Jacobians: row pointers
    once, then per step the three random fields in, the BSR (int64 columns,
    3x3 blocks) out -- bitwise the host restatement's values.  The matrix
    keeps its device copy (packed straight from the device CSR, no upload)
    for the solve that follows, and b = A x* is the device SpMV."""

    def __init__(self, nx, ny, nz, xs):
        from . import _native as N
        from . import device as D
        t = D.torch()
        self.dims = (nx, ny, nz)
        self.n = nx * ny * nz
        cnt = t.empty(self.n, dtype=t.int64, device="cuda")
        N.check(N.lib().cprb_gen_row_counts(nx, ny, nz, D.ptr(cnt), D.stream()))
        self.ptr_d = t.zeros(self.n + 1, dtype=t.int64, device="cuda")
        t.cumsum(cnt, 0, out=self.ptr_d[1:])
        self.ptr = self.ptr_d.cpu().numpy()
        self.nnz = int(self.ptr[-1])
        self.cols_d = None
        self.xs_d = D.upload(xs)

    def assemble(self, perm, conv_scale, couple, drift, with_rhs):
        from . import _native as N
        from . import device as D
        t = D.torch()
        f64 = D.upload
        perm_d, conv_d, cpl_d = f64(perm), f64(conv_scale), f64(couple)
        cols_d = t.empty(self.nnz, dtype=t.int64, device="cuda")
        vals_d = t.empty(self.nnz * 9, dtype=t.float64, device="cuda")
        N.check(N.lib().cprb_gen_assemble(*self.dims, float(drift), D.ptr(perm_d), D.ptr(conv_d),
                                          D.ptr(cpl_d), D.ptr(self.ptr_d), D.ptr(cols_d),
                                          D.ptr(vals_d), D.stream()))
        if self.cols_d is None:
            self.cols = cols_d.cpu().numpy()
            self.cols_d = cols_d
        A = BlockCsrMatrix(3, self.n, self.n, self.ptr, self.cols,
                           vals_d.cpu().numpy().reshape(-1, 3, 3))
        M = D.device_matrix(A, (self.ptr_d, self.cols_d, vals_d))
        b = None
        if with_rhs:
            y = D.empty(3 * self.n)
            N.check(N.lib().cprb_spmv(M.desc_ref(), 3, D.ptr(self.xs_d), D.ptr(y), None,
                                      D.stream()))
            b = y.cpu().numpy()
        return A, b


def generate_blackoil_like_sequence(nx: int, ny: int, nz: int, nsteps: int, drift: float,
                                    seed: int, with_rhs: bool = True) -> ProblemSequence:
    """Deterministic-by-seed sequence of 3x3-block 7-point systems
    (src/problems.py:74-110).

    The random fields and np.exp are drawn on the host exactly as the
    reference does; with a B200 present the Jacobians are assembled in HBM
    (csrc/gen.cu, bitwise equal to the host restatement _assemble) and each
    matrix keeps its device copy for the solve (device.release_device(A)
    frees it); otherwise the host restatement assembles them."""
    if min(nx, ny, nz) < 1 or nsteps < 1:
        raise ValueError("grid dimensions and nsteps must be >= 1")
    rng = np.random.default_rng(seed)
    n = nx * ny * nz
    logk = rng.normal(0.0, 1.0, n)
    conv_scale = rng.uniform(0.2, 0.5, n)
    couple = rng.standard_normal((n, 6)) * 0.5
    xs = manufactured_solution(n)
    dev = _DeviceAssembler(nx, ny, nz, xs) if _cuda_ok() else None
    g = None if dev is not None else _Grid(nx, ny, nz)
    systems = []
    for step in range(nsteps):
        if step > 0:
            logk = logk + drift * rng.normal(0.0, 1.0, n)
            conv_scale = conv_scale * np.exp(drift * rng.normal(0.0, 1.0, n))
        if dev is not None:
            systems.append(dev.assemble(np.exp(logk), conv_scale, couple, drift, with_rhs))
            continue
        A = _assemble(g, np.exp(logk), conv_scale, couple, drift)
        systems.append((A, bsr_matvec_reference_order(A, xs) if with_rhs else None))
    return ProblemSequence(systems, provenance={"kind": "synthetic", "nx": nx, "ny": ny,
                                                "nz": nz, "nsteps": nsteps, "drift": drift,
                                                "seed": seed})


def pressure_operator(nx: int, ny: int, nz: int, seed: int = 0, drift: float = 0.0) -> CsrMatrix:
    """The (0,0) pressure block of the first generated system (config 2 input;
    depends only on the first RNG draw)."""
    rng = np.random.default_rng(seed)
    g = _Grid(nx, ny, nz)
    logk = rng.normal(0.0, 1.0, g.n)
    conv = rng.uniform(0.2, 0.5, g.n)
    cpl = rng.standard_normal((g.n, 6)) * 0.5
    A = _assemble(g, np.exp(logk), conv, cpl, drift)
    return CsrMatrix(A.nrows, A.ncols, A.row_ptr, A.col_idx, A.values[:, 0, 0].copy())


def poisson_2d(nx: int, ny: int) -> CsrMatrix:
    """5-point Laplacian (src/problems.py:197-208)."""
    n = nx * ny
    c = np.arange(n)
    ix, iy = c % nx, c // nx
    rows, cols, vals = [c], [c], [np.full(n, 4.0)]
    for dx, dy in ((-1, 0), (1, 0), (0, -1), (0, 1)):
        m = (ix + dx >= 0) & (ix + dx < nx) & (iy + dy >= 0) & (iy + dy < ny)
        rows.append(c[m])
        cols.append((ix + dx + nx * (iy + dy))[m])
        vals.append(np.full(int(m.sum()), -1.0))
    return CsrMatrix.from_coo(np.concatenate(rows), np.concatenate(cols), np.concatenate(vals),
                              (n, n))


def save_sequence(seq: ProblemSequence, out_dir) -> Path:
    """Matrices and right-hand sides as MatrixMarket files plus manifest.json
    (src/problems.py:158-177); returns the manifest path."""
    from .mmio import write_block_matrix_market, write_matrix_market, write_vector
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    entries = []
    for k, (A, rhs) in enumerate(seq.systems, start=1):
        mpath = out / f"system_{k:03d}.mtx"
        vpath = out / f"rhs_{k:03d}.mtx"
        if isinstance(A, BlockCsrMatrix):
            write_block_matrix_market(mpath, A)
            bs = A.block_size
        else:
            write_matrix_market(mpath, A)
            bs = 1
        write_vector(vpath, rhs)
        entries.append({"matrix": mpath.name, "rhs": vpath.name, "block_size": bs})
    manifest = {"systems": entries, "provenance": seq.provenance}
    mpath = out / "manifest.json"
    mpath.write_text(json.dumps(manifest, indent=2) + "\n")
    return mpath


def load_sequence(manifest_path) -> ProblemSequence:
    """Recorded Jacobian sequence from a manifest (src/problems.py:180-194)."""
    from .mmio import read_block_matrix_market, read_matrix_market, read_vector
    manifest_path = Path(manifest_path)
    manifest = json.loads(manifest_path.read_text())
    base = manifest_path.parent
    systems = []
    for entry in manifest["systems"]:
        path = base / entry["matrix"]
        A = (read_block_matrix_market(path) if entry.get("block_size", 1) > 1
             else read_matrix_market(path))
        systems.append((A, read_vector(base / entry["rhs"])))
    return ProblemSequence(systems, provenance=manifest.get("provenance", {}))
