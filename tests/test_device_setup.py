"""SETUP on the device (csrc/factor.cu, csrc/gen.cu): the level-scheduled
BILU(0) factorization is bitwise the host C++ factorization (which the CPU
suite pins to the reference's factors), with the host path's perturbation
warnings and error messages; the device stencil packing equals the host
stencil plan; build_cpr with device setup reproduces the reference's C1
solve."""

import json

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, random_block

import paper_2201_01970_b200 as P
from paper_2201_01970_b200 import ilu as I

pytestmark = pytest.mark.gpu


def _bsr(o):
    return P.BlockCsrMatrix(o.b, o.nrows, o.ncols, o.ptr, o.cols, o.vals)


def _same(F, G):
    assert np.array_equal(F.L.row_ptr, G.L.row_ptr) and np.array_equal(F.L.col_idx, G.L.col_idx)
    assert np.array_equal(F.U.row_ptr, G.U.row_ptr) and np.array_equal(F.U.col_idx, G.U.col_idx)
    assert np.array_equal(F.L.values.view(np.uint64), G.L.values.view(np.uint64))
    assert np.array_equal(F.U.values.view(np.uint64), G.U.values.view(np.uint64))
    assert np.array_equal(F.u_diag_inv.view(np.uint64), G.u_diag_inv.view(np.uint64))
    for a, b in zip(F.l_schedule.levels, G.l_schedule.levels):
        assert np.array_equal(a, b)
    for a, b in zip(F.u_schedule.levels, G.u_schedule.levels):
        assert np.array_equal(a, b)


def test_device_bilu0_bitwise_equals_host(gpu, rng):
    g = load_golden("gen_c1.npz")
    mats = [P.BlockCsrMatrix(3, 1000, 1000, g["ptr"], g["cols"], g["vals"])]
    mats += [_bsr(random_block(rng, n)) for n in (1, 7, 300, 2000)]
    mats += [s[0] for s in P.generate_blackoil_like_sequence(17, 9, 6, 2, 0.2, 3).systems]
    for A in mats:
        _same(I.bilu0_factorize_device(A), P.bilu0_factorize(A))


def test_device_bilu0_perturbation_and_errors(gpu):
    # zero pivot with nonzero norm -> perturbed, with the host warning
    blocks = np.zeros((3, 3, 3))
    blocks[0] = np.diag([1.0, 1.0, 0.0])
    blocks[1] = np.eye(3) * 2.0
    blocks[2] = np.eye(3) * 3.0
    A = P.BlockCsrMatrix.from_block_coo(3, [0, 1, 2], [0, 1, 2], blocks, (3, 3))
    with pytest.warns(RuntimeWarning, match="row 0"):
        F = I.bilu0_factorize_device(A)
    with pytest.warns(RuntimeWarning, match="row 0"):
        G = P.bilu0_factorize(A)
    _same(F, G)
    # an exactly zero pivot block -> LinAlgError naming the (lowest) row,
    # raised before any perturbation warning (as the host path does)
    blocks[1] = 0.0
    blocks[2] = 0.0
    A = P.BlockCsrMatrix.from_block_coo(3, [0, 1, 2], [0, 1, 2], blocks, (3, 3))
    for fn in (I.bilu0_factorize_device, P.bilu0_factorize):
        with pytest.raises(np.linalg.LinAlgError, match="row 1"):
            fn(A)


def test_device_stencil_pack_equals_host_plan(gpu):
    (A, _), = P.generate_blackoil_like_sequence(21, 13, 7, 1, 0.03, 2).systems
    Fd = I.bilu0_factorize_device(A)
    sd = Fd.stencil_device()
    sh = I.stencil_plan(P.bilu0_factorize(A))
    assert sd is not None and sh is not None
    for k in ("nx", "ny", "nz", "S", "D", "P", "len"):
        assert sd[k] == sh[k], k
    for k in ("doff", "slot"):
        assert np.array_equal(sd[k].cpu().numpy(), sh[k]), k
    for k in ("lrec", "urec"):
        assert np.array_equal(sd[k].cpu().numpy().view(np.uint64), sh[k].view(np.uint64)), k
    # a non-grid pattern is not a stencil
    rng = np.random.default_rng(3)
    assert I.bilu0_factorize_device(_bsr(random_block(rng, 64))).stencil_device() is None


def test_build_cpr_device_setup_c1_against_reference(gpu, monkeypatch):
    """build_cpr with the device factorization (default on a GPU) against
    the unmodified reference's C1 run (tests/golden/c1_v0.npz)."""
    g = load_golden("gen_c1.npz")
    A = P.BlockCsrMatrix(3, 1000, 1000, g["ptr"], g["cols"], g["vals"])
    ref = load_golden("c1_v0.npz")
    s = json.loads((GOLDEN / "summary.json").read_text())["v0"]
    cfg = P.SolverConfig(theta=0.0, theta_amg=0.0, cycle="v")
    B = P.build_cpr(A, cfg)
    assert isinstance(B.relaxation, I.DeviceBiluFactors)
    res = P.gmres_solve(A, g["b"], None, B, cfg.gmres_params(), history=True)
    assert (res.outer, res.inner, res.converged) == (s["outer"], s["inner"], s["converged"])
    hist = np.array([h if not isinstance(h, tuple) else -h[1] for h in res.history])
    np.testing.assert_allclose(hist, ref["hist"], rtol=1e-8)
    monkeypatch.setenv("CPRB_DEVICE_SETUP", "0")
    B0 = P.build_cpr(A, cfg)
    assert not isinstance(B0.relaxation, I.DeviceBiluFactors)
    res0 = P.gmres_solve(A, g["b"], None, B0, cfg.gmres_params())
    assert np.array_equal(res.x, res0.x)
