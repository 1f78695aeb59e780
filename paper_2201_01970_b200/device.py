"""Device plumbing: vectors, SELL-32 layouts and the device plans the C ABI
consumes.

PyTorch owns device memory and the stream; the sm_100a library does all the
arithmetic.  Layout builders here are host-side numpy (setup time only): they
rearrange stored values without changing any of them, and keep each row's
entries in the order the reference sums them.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _native as N

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("the CPR-GMRES solve path needs a CUDA device (B200); there is no "
                           "CPU fallback")
    N.lib()


def stream() -> int:
    return torch().cuda.current_stream().cuda_stream


_SETUP_SYNC = os.environ.get("CPRB_SETUP_SYNC", "0") == "1"


def bind_current(fn):
    """Wrap fn so that, run on a setup-pool thread, it uses the caller's CUDA
    device and stream (torch keeps both per thread)."""
    t = torch()
    dev = t.cuda.current_device()
    st = t.cuda.current_stream()

    def run(*args, **kw):
        with t.cuda.device(dev), t.cuda.stream(st):
            out = fn(*args, **kw)
            if _SETUP_SYNC:
                t.cuda.current_stream().synchronize()
            return out
    return run


def is_tensor(a) -> bool:
    return type(a).__module__.startswith("torch")


def ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def empty(n: int, dtype=None):
    t = torch()
    return t.empty(int(n), dtype=dtype or t.float64, device="cuda")


def zeros(n: int, dtype=None):
    t = torch()
    return t.zeros(int(n), dtype=dtype or t.float64, device="cuda")


def to_device(x):
    """(CUDA float64 tensor, kind) for a numpy array / host tensor / CUDA tensor.
    kind tells from_device how to hand results back."""
    require_cuda()
    t = torch()
    if isinstance(x, t.Tensor):
        if x.is_cuda:
            if x.dtype != t.float64 or not x.is_contiguous():
                x = x.to(t.float64).contiguous()
            return x, "cuda"
        return x.to(device="cuda", dtype=t.float64, non_blocking=x.is_pinned()), "host_tensor"
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    return t.from_numpy(a).to("cuda"), "numpy"


def from_device(y, kind):
    """Hand a device result back in the caller's kind; host copies land in
    pinned memory (torch's caching host allocator), which DMA fills at full
    PCIe rate instead of staging through pageable memory."""
    if kind == "cuda":
        return y
    out = torch().empty(y.shape, dtype=y.dtype, pin_memory=True)
    out.copy_(y)
    return out if kind == "host_tensor" else out.numpy()


def upload(a: np.ndarray, dtype=None):
    t = torch()
    a = np.ascontiguousarray(a)
    return t.from_numpy(a).to("cuda")


# -- reductions / vector ops -------------------------------------------------


class _Scratch:
    def __init__(self):
        t = torch()
        self.partials = t.zeros(N_RED, dtype=t.float64, device="cuda")
        self.ticket = t.zeros(4, dtype=t.int32, device="cuda")
        self.out = t.zeros(64, dtype=t.float64, device="cuda")


N_RED = 1184
_scratch = {}


def scratch() -> _Scratch:
    dev = torch().cuda.current_device()
    if dev not in _scratch:
        _scratch[dev] = _Scratch()
    return _scratch[dev]


def dot(x, y) -> float:
    s = scratch()
    N.check(N.lib().cprb_dot(x.shape[0], ptr(x), ptr(y), ptr(s.out), ptr(s.partials),
                             ptr(s.ticket), stream()))
    return float(s.out[0].item())


def dot_dev(x, y, out, s=None):
    """(x, y) into the device scalar `out` (no host sync)."""
    s = s or scratch()
    N.check(N.lib().cprb_dot(x.shape[0], ptr(x), ptr(y), ptr(out), ptr(s.partials),
                             ptr(s.ticket), stream()))


def axpy(alpha: float, x, y, out):
    N.check(N.lib().cprb_axpy(x.shape[0], float(alpha), ptr(x), ptr(y), ptr(out), stream()))


# -- SELL-32 packing -----------------------------------------------------------


def pad_lanes(rows: np.ndarray) -> np.ndarray:
    """Pad a lane->row list with -1 to a multiple of 32."""
    L = rows.shape[0]
    P = (-L) % 32
    if P:
        rows = np.concatenate([rows, np.full(P, -1, dtype=rows.dtype)])
    return rows


@dataclass
class SellHost:
    nslices: int
    nrows: int
    slice_ptr: np.ndarray
    lane_row: np.ndarray
    lane_len: np.ndarray
    cols: np.ndarray
    vals: np.ndarray
    lane_len_lo: np.ndarray | None = None
    agg_out: np.ndarray | None = None


def pack_sell(lane_row, lane_ptr, ent_cols, ent_vals, bs, nrows, lane_len_lo=None,
              agg_out=None) -> SellHost:
    """Pack per-lane entry lists into SELL-32.

    lane_row: (L,) rows (L % 32 == 0, -1 = padding); lane_ptr: (L+1,) entry
    offsets of each lane's list in ent_cols/ent_vals; ent_vals (nnz,) scalars or
    (nnz, bs, bs) blocks.  Entry m of lane l lands at slice_ptr[s] + 32m + l;
    block value (r, c) at (slice_ptr[s] + 32m)*bs*bs + (r*bs + c)*32 + l.
    """
    lane_row = np.asarray(lane_row, dtype=np.int32)
    L = lane_row.shape[0]
    assert L % 32 == 0
    ns = L // 32
    lens = np.diff(np.asarray(lane_ptr, dtype=np.int64)).astype(np.int64)
    width = lens.reshape(ns, 32).max(axis=1) if ns else np.zeros(0, dtype=np.int64)
    slice_ptr = np.zeros(ns + 1, dtype=np.int64)
    np.cumsum(width * 32, out=slice_ptr[1:])
    total = int(slice_ptr[-1])
    bb = bs * bs
    cols = np.zeros(max(total, 1), dtype=np.int32)
    vals = np.zeros(max(total * bb, 1))
    lp = np.ascontiguousarray(lane_ptr, dtype=np.int64)
    ec = np.ascontiguousarray(ent_cols, dtype=np.int64)
    ev = np.ascontiguousarray(ent_vals, dtype=np.float64).reshape(-1)
    if L and ec.size:
        N.check(N.lib().cprb_sell_fill_lanes(L, N.p64(lp), N.p64(slice_ptr), N.p64(ec), N.pf64(ev),
                                             bs, N.p32(cols), N.pf64(vals)))
    return SellHost(ns, int(nrows), slice_ptr, lane_row, lens.astype(np.int32), cols, vals,
                    None if lane_len_lo is None else np.asarray(lane_len_lo, dtype=np.int32),
                    None if agg_out is None else np.asarray(agg_out, dtype=np.int32))


class SellDev:
    """Device copy of a SellHost plus its C descriptor."""

    def __init__(self, h: SellHost):
        self.host = h
        self.t = {k: upload(getattr(h, k)) for k in
                  ("slice_ptr", "lane_row", "lane_len", "cols", "vals")}
        for k in ("lane_len_lo", "agg_out"):
            v = getattr(h, k)
            self.t[k] = upload(v) if v is not None else None
        self.desc = N.Sell(h.nslices, h.nrows, ptr(self.t["slice_ptr"]), ptr(self.t["lane_row"]),
                           ptr(self.t["lane_len"]), ptr(self.t["lane_len_lo"]),
                           ptr(self.t["cols"]), ptr(self.t["vals"]), ptr(self.t["agg_out"]))

    def nbytes(self) -> int:
        return sum(int(v.numel() * v.element_size()) for v in self.t.values() if v is not None)


def sell_from_rows(lane_src, ptr_, cols, vals, nrows, colmap=None, **extra) -> SellHost:
    """SELL-32 whose lane l holds row lane_src[l] of a scalar CSR (-1 =
    padding) in its stored entry order, columns renumbered through colmap
    (native fill: no per-entry index arrays on the host)."""
    lane_src = np.ascontiguousarray(lane_src, dtype=np.int64)
    L = lane_src.shape[0]
    assert L % 32 == 0
    ns = L // 32
    ptr_ = np.ascontiguousarray(ptr_, dtype=np.int64)
    real = lane_src >= 0
    lens = np.zeros(L, dtype=np.int64)
    lens[real] = (ptr_[1:] - ptr_[:-1])[lane_src[real]]
    width = lens.reshape(ns, 32).max(axis=1) if ns else np.zeros(0, dtype=np.int64)
    slice_ptr = np.zeros(ns + 1, dtype=np.int64)
    np.cumsum(width * 32, out=slice_ptr[1:])
    total = int(slice_ptr[-1])
    out_c = np.zeros(max(total, 1), dtype=np.int32)
    out_v = np.zeros(max(total, 1))
    c = np.ascontiguousarray(cols, dtype=np.int64)
    v = np.ascontiguousarray(vals, dtype=np.float64)
    cm = None if colmap is None else np.ascontiguousarray(colmap, dtype=np.int64)
    if L and c.size:
        N.check(N.lib().cprb_sell_fill_rows(L, N.p64(lane_src), N.p64(slice_ptr), N.p64(ptr_),
                                            N.p64(c), N.pf64(v), None if cm is None else N.p64(cm),
                                            N.p32(out_c), N.pf64(out_v)))
    lane_row = extra.pop("lane_row", np.where(real, np.arange(L), -1).astype(np.int32))
    return SellHost(ns, int(nrows), slice_ptr, np.asarray(lane_row, dtype=np.int32),
                    lens.astype(np.int32), out_c, out_v, extra.get("lane_len_lo"),
                    None if extra.get("agg_out") is None else np.asarray(extra["agg_out"],
                                                                         dtype=np.int32))


def sell_rows(ptr_, cols, vals, bs, nrows) -> SellHost:
    """SELL-32 of a (block) CSR in natural row order."""
    lane_row = pad_lanes(np.arange(nrows, dtype=np.int32))
    lp = np.zeros(lane_row.shape[0] + 1, dtype=np.int64)
    lp[1:nrows + 1] = ptr_[1:]
    lp[nrows + 1:] = ptr_[-1]
    return pack_sell(lane_row, lp, cols, vals, bs, nrows)


class _PackedSell:
    """SELL-32 of a (block) CSR in natural row order, packed ON the device
    from the raw CSR arrays (csrc/spmv.cu k_pack_bsr_sell): the upload of a
    new Jacobian is one H2D copy of the CSR plus one kernel, not a host
    repack.  Same layout and values as sell_rows()."""

    def __init__(self, A, bs: int, dev_csr=None):
        t = torch()
        n = int(A.nrows)
        rp = np.ascontiguousarray(A.row_ptr, dtype=np.int64)
        lens = np.diff(rp)
        L = -(-n // 32) * 32
        lp = np.zeros(L, dtype=np.int64)
        lp[:n] = lens
        ns = L // 32
        width = lp.reshape(ns, 32).max(axis=1) if ns else np.zeros(0, dtype=np.int64)
        slice_ptr = np.zeros(ns + 1, dtype=np.int64)
        np.cumsum(width * 32, out=slice_ptr[1:])
        total = int(slice_ptr[-1])
        bb = bs * bs
        lane_row = np.full(L, -1, dtype=np.int32)
        lane_row[:n] = np.arange(n, dtype=np.int32)
        self.t = {"slice_ptr": upload(slice_ptr), "lane_row": upload(lane_row),
                  "lane_len": upload(lp.astype(np.int32)),
                  "cols": t.zeros(max(total, 1), dtype=t.int32, device="cuda"),
                  "vals": t.zeros(max(total * bb, 1), dtype=t.float64, device="cuda")}
        nnz = int(rp[-1])
        if n and nnz:
            if dev_csr is not None:        # CSR already in HBM (device generator)
                rp_d, ci_d, v_d = dev_csr
            else:
                rp_d = upload(rp)
                ci_d = upload(np.ascontiguousarray(A.col_idx, dtype=np.int64))
                v_d = upload(np.ascontiguousarray(A.values, dtype=np.float64).reshape(-1))
            N.check(N.lib().cprb_pack_bsr_sell(n, bs, ptr(rp_d), ptr(ci_d), ptr(v_d),
                                               ptr(self.t["slice_ptr"]), ptr(self.t["cols"]),
                                               ptr(self.t["vals"]), stream()))
            del rp_d, ci_d, v_d
        self.host = None
        self.desc = N.Sell(ns, n, ptr(self.t["slice_ptr"]), ptr(self.t["lane_row"]),
                           ptr(self.t["lane_len"]), 0, ptr(self.t["cols"]), ptr(self.t["vals"]), 0)

    def nbytes(self) -> int:
        return sum(int(v.numel() * v.element_size()) for v in self.t.values())


class DeviceMatrix:
    """A CsrMatrix / BlockCsrMatrix resident on the device (SELL-32)."""

    def __init__(self, A, dev_csr=None):
        require_cuda()
        bs = int(getattr(A, "block_size", 1))
        self.b = bs
        self.nrows = int(A.nrows)
        self.sell = _PackedSell(A, bs, dev_csr)
        # the CSR itself when it was born on the device (device generator):
        # the device BILU(0) factorization starts from it without an upload
        self.csr = dev_csr

    def desc_ref(self):
        return C.byref(self.sell.desc)


def device_matrix(A, dev_csr=None) -> DeviceMatrix:
    """Device copy cached on the matrix object (matrices are immutable after
    construction in the reference's contract, src/sparse.py:217-218).
    dev_csr = (row_ptr, col_idx, values) already on the device: packed
    without an upload.  release_device(A) drops the cached copy."""
    M = getattr(A, "_cprb_dev", None)
    if M is None:
        M = DeviceMatrix(A, dev_csr)
        try:
            object.__setattr__(A, "_cprb_dev", M)
        except (AttributeError, TypeError):
            pass
    return M


def cuda_ok() -> bool:
    """A CUDA device and the native library are both available."""
    try:
        if not torch().cuda.is_available():
            return False
        N.lib()
        return True
    except (ImportError, OSError, RuntimeError):
        return False


def cached_device_matrix(A):
    return getattr(A, "_cprb_dev", None)


def release_device(A) -> None:
    """Free the device copy cached on A (it is rebuilt on the next use)."""
    try:
        object.__setattr__(A, "_cprb_dev", None)
    except (AttributeError, TypeError):
        pass
