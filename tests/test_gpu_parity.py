"""Device (sm_100a) parity against the oracle and the reference's fixtures.

Bit-exact where the reference is deterministic (SpMV, smoother sweeps, BILU
solves for identical factors, residual/restriction); solve-level parity per
BASELINE.json north_star: same iteration counts, Givens residual history
within 1e-8 relative, solutions within 1e-6 relative (tighter where the
fixtures allow)."""

import json

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, orc, poisson_2d, random_block, random_sparse, tridiag

import paper_2201_01970_b200 as P
from paper_2201_01970_b200.ilu import _strict

pytestmark = pytest.mark.gpu
SUMMARY = json.loads((GOLDEN / "summary.json").read_text())


def _csr(o):
    return P.CsrMatrix(o.nrows, o.ncols, o.ptr, o.cols, o.vals)


def _bsr(o):
    return P.BlockCsrMatrix(o.b, o.nrows, o.ncols, o.ptr, o.cols, o.vals)


def _c1():
    g = load_golden("gen_c1.npz")
    return P.BlockCsrMatrix(3, 1000, 1000, g["ptr"], g["cols"], g["vals"]), g["b"]


def _oracle_bilu(F):
    lp, lc, lv = _strict(F.L)
    up, uc, uv = _strict(F.U)
    return orc.Bilu(F.n, F.block_size, lp, lc, lv, up, uc, uv, F.u_diag_inv,
                    F.l_schedule.levels, F.u_schedule.levels)


# -- K1: SpMV ----------------------------------------------------------------


def test_spmv_block_bitwise(gpu):
    g = load_golden("random_block.npz")
    for ci in range(int(g["ncases"])):
        p = f"c{ci}_"
        n = g[p + "ptr"].shape[0] - 1
        A = P.BlockCsrMatrix(3, n, n, g[p + "ptr"], g[p + "cols"], g[p + "vals"])
        assert np.array_equal(P.spmv(A, g[p + "x"]), g[p + "spmv"]), ci


def test_spmv_scalar_bitwise(gpu):
    g = load_golden("random_scalar.npz")
    for ci in range(int(g["ncases"])):
        p = f"c{ci}_"
        n = g[p + "ptr"].shape[0] - 1
        A = P.CsrMatrix(n, n, g[p + "ptr"], g[p + "cols"], g[p + "vals"])
        assert np.array_equal(P.spmv(A, g[p + "x0"]), g[p + "spmv"]), ci


def test_spmv_c1_rhs_and_long_rows(gpu):
    A, b = _c1()
    gen = P.generate_blackoil_like_sequence(10, 10, 10, 1, 0.01, 0)
    assert np.array_equal(P.spmv(A, P.problems.manufactured_solution(1000)), b)
    rng = np.random.default_rng(9)
    for n, avg in ((1, 1), (40, 30), (300, 60), (200, 150)):       # rows beyond 8 blocks / 129 entries
        M = random_sparse(rng, n, avg_nnz=avg, dominant=False)
        x = rng.standard_normal(n)
        assert np.array_equal(P.spmv(_csr(M), x), orc.spmv(M, x)), n
        B = random_block(rng, max(n // 3, 1), b=3, avg_nnz=min(avg, 40))
        xb = rng.standard_normal(B.nrows * 3)
        assert np.array_equal(P.spmv(_bsr(B), xb), orc.spmv(B, xb)), n
    del gen


def test_generator_rhs_device_equals_host_order(gpu):
    """Input generation computes b = A x* with the device SpMV when a GPU is
    present: bitwise equal to the host reference-order product."""
    (A, b), = P.generate_blackoil_like_sequence(23, 17, 9, 1, 0.01, 5).systems
    xs = P.problems.manufactured_solution(A.nrows)
    assert np.array_equal(b, P.problems.bsr_matvec_reference_order(A, xs))


def test_device_sell_packing_matches_host_layout(gpu, rng):
    """Jacobian uploads pack SELL-32 on the device (csrc/spmv.cu
    k_pack_bsr_sell): identical arrays to the host packer."""
    from paper_2201_01970_b200 import device as D
    for M in (_bsr(random_block(rng, 333, 3)), _csr(random_sparse(rng, 517))):
        bs = int(getattr(M, "block_size", 1))
        vals = np.asarray(M.values, dtype=np.float64)
        h = D.sell_rows(np.asarray(M.row_ptr, dtype=np.int64), np.asarray(M.col_idx),
                        vals if bs > 1 else vals.reshape(-1), bs, M.nrows)
        d = D._PackedSell(M, bs)
        for k in ("slice_ptr", "lane_row", "lane_len", "cols", "vals"):
            assert np.array_equal(d.t[k].cpu().numpy(), np.asarray(getattr(h, k))), k


def test_spmv_api_edges(gpu):
    A = P.CsrMatrix(3, 3, [0, 0, 0, 0], [], [])
    assert np.array_equal(P.spmv(A, np.ones(3)), np.zeros(3))
    with pytest.raises(ValueError, match="dimension mismatch"):
        P.spmv(P.CsrMatrix.identity(3), np.ones(4))
    assert P.dot(np.array([1.0, 0.0]), np.array([0.0, 1.0])) == 0.0
    assert P.norm2(np.array([3.0, 4.0])) == 5.0
    assert np.array_equal(P.axpy(2.0, np.array([1.0, 1.0]), np.array([1.0, 0.0])), [3.0, 2.0])
    import torch
    x = torch.arange(3, dtype=torch.float64, device="cuda")
    y = P.spmv(P.CsrMatrix.identity(3), x)
    assert y.is_cuda and torch.equal(y, x)


def test_dot_deterministic(gpu):
    rng = np.random.default_rng(1)
    x = rng.standard_normal(3_366_000)
    y = rng.standard_normal(3_366_000)
    d = P.dot(x, y)
    assert all(P.dot(x, y) == d for _ in range(3))
    assert abs(d - float(np.dot(x, y))) <= 1e-12 * np.abs(x * y).sum()


# -- K4: PGS-SCM sweeps ---------------------------------------------------------


def test_pgs_scm_sweep_bitwise(gpu):
    g = load_golden("random_scalar.npz")
    for ci in range(int(g["ncases"])):
        p = f"c{ci}_"
        n = g[p + "ptr"].shape[0] - 1
        A = P.CsrMatrix(n, n, g[p + "ptr"], g[p + "cols"], g[p + "vals"])
        part = P.vertices_grouping(P.strong_connections(A, float(g[p + "theta"])))
        got = P.pgs_scm_sweep(A, g[p + "b"], g[p + "x0"], part)
        assert np.array_equal(got, g[p + "sweep"]), ci


def test_gs_kats(gpu):
    A = P.CsrMatrix.from_dense([[2.0, -1.0], [-1.0, 2.0]])
    assert np.array_equal(P.gs_sweep(A, np.ones(2), np.zeros(2)), [0.5, 0.75])
    T = _csr(tridiag(4))
    part = P.vertices_grouping(P.strong_connections(T, 1.0))
    assert part.c == 1
    assert np.array_equal(P.pgs_scm_sweep(T, np.ones(4), np.zeros(4), part),
                          [0.5, 0.75, 0.875, 0.9375])
    rng = np.random.default_rng(99)
    for _ in range(8):
        n = int(rng.integers(5, 120))
        M = random_sparse(rng, n, avg_nnz=5, symmetric=bool(rng.integers(0, 2)))
        for theta in (0.0, 0.3):
            groups = orc.vertices_grouping(orc.strong_connections(M, theta))
            part = P.ColorPartition.from_groups(groups, n)
            b = rng.standard_normal(n)
            x0 = rng.standard_normal(n)
            ref = orc.ScmSmoother(M, groups)
            for d in ("forward", "backward", "symmetric"):
                got = P.PgsScmSmoother(_csr(M), part).apply(b, x0, direction=d)
                assert np.array_equal(got, ref.apply(b, x0, direction=d)), (n, theta, d)


# -- K8: BILU(0) solves ---------------------------------------------------------


@pytest.mark.parametrize("wave", [True, False])
def test_bilu_apply_bitwise_given_factors(gpu, wave):
    """Both device solvers (chunked wavefront / level-ordered sync-free) are
    bitwise equal to the reference's level-scheduled solve."""
    import torch
    rng = np.random.default_rng(5)
    A, _ = _c1()
    (A2, _), = P.generate_blackoil_like_sequence(13, 7, 9, 1, 0.05, 3).systems
    cases = [A, A2] + [_bsr(random_block(rng, int(rng.integers(2, 150)), 3,
                                         int(rng.integers(2, 7)))) for _ in range(6)]
    cases += [_csr(random_sparse(rng, int(rng.integers(3, 300)), 6)),
              _bsr(random_block(rng, 1, 3, 1)), _bsr(random_block(rng, 700, 3, 12))]
    for ci, M in enumerate(cases):
        F = P.bilu0_factorize(M)
        Fo = _oracle_bilu(F)
        r = rng.standard_normal(Fo.n * Fo.b)
        dev = F.device(use_wave=wave)
        rd = torch.from_numpy(r).cuda()
        z = torch.empty_like(rd)
        for _ in range(2):                                   # re-armed tickets / sentinels
            dev.apply(rd, z)
            assert np.array_equal(z.cpu().numpy(), orc.bilu_apply(Fo, r)), ci


def test_bilu_apply_c1_vs_reference(gpu):
    A, _ = _c1()
    g = load_golden("c1_v0.npz")
    F = P.bilu0_factorize(A)
    np.testing.assert_allclose(P.bilu_apply(F, g["r_test"]), g["z_bilu"], rtol=1e-11, atol=1e-13)
    with pytest.raises(ValueError, match="dimension mismatch"):
        P.bilu_apply(F, np.ones(5))


# -- AMG cycle + CPR apply ----------------------------------------------------------


@pytest.mark.parametrize("tag", ["v0", "vd", "k0", "kd"])
def test_amg_cycle_and_cpr_apply_c1(gpu, tag):
    A, _ = _c1()
    g = load_golden(f"c1_{tag}.npz")
    B = P.build_cpr(A, P.SolverConfig(theta=0.0, theta_amg=0.0 if tag[1] == "0" else 0.08,
                                      cycle=tag[0]))
    zp = P.amg_cycle(B.pressure_solver, g["rp_test"])
    np.testing.assert_allclose(zp, g["zp_cycle"], rtol=1e-10, atol=1e-12)
    z = B.apply(g["r_test"])
    np.testing.assert_allclose(z, g["z_apply"], rtol=1e-10, atol=1e-12)


def test_vcycle_matches_oracle_with_same_coarse_solve(gpu):
    A, _ = _c1()
    B = P.build_cpr(A, P.SolverConfig(theta=0.0, theta_amg=0.0, cycle="v"))
    Bo = orc.build_cpr(orc.Bsr(3, 1000, 1000, A.row_ptr, A.col_idx, A.values),
                       orc.SolverConfig(theta=0.0, theta_amg=0.0, cycle="v"))
    inv = B.pressure_solver.coarsest_lu[1]
    rng = np.random.default_rng(3)
    r = rng.standard_normal(1000)
    zo = orc.amg_cycle(Bo.hierarchy, r, coarse_solve=lambda b: inv @ b)
    np.testing.assert_allclose(P.amg_cycle(B.pressure_solver, r), zo, rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("tail_rows", ["0", "300", "600", "5000", "100000"])
def test_vcycle_persistent_tail_bitwise(gpu, monkeypatch, tail_rows):
    """The persistent single-CTA tail (csrc/vtail.cu: shared-memory vectors,
    TMA-streamed records) runs the launched kernels' arithmetic: bitwise
    equal cycles with the tail off, starting at a deep level, a middle
    level, or covering every level that fits."""
    A, _ = _c1()
    (A2, _), = P.generate_blackoil_like_sequence(40, 30, 20, 1, 0.01, 2).systems
    rng = np.random.default_rng(11)
    for M in (A, A2):
        cfg = P.SolverConfig(theta=0.0, theta_amg=0.0, cycle="v")
        monkeypatch.setenv("CPRB_TAIL_ROWS", "0")
        h0 = P.build_hierarchy(P.pressure_matrix(M), cfg.amg_params())
        r = rng.standard_normal(M.nrows)
        z0 = P.amg_cycle(h0, r)
        assert h0.device().desc.tail_start == len(h0.levels) - 1
        monkeypatch.setenv("CPRB_TAIL_ROWS", tail_rows)
        h1 = P.build_hierarchy(P.pressure_matrix(M), cfg.amg_params())
        z1 = P.amg_cycle(h1, r)
        if tail_rows in ("5000", "100000"):
            assert h1.device().desc.tail_start < len(h1.levels) - 1
        monkeypatch.delenv("CPRB_TAIL_ROWS")
        assert np.array_equal(z0, z1)


def test_vcycle_tail_skips_snapshot_levels(gpu, monkeypatch):
    """theta_amg > 0 levels with intra-colour couplings stay on the launched
    path; the cycle is unchanged bitwise."""
    A, _ = _c1()
    cfg = P.SolverConfig(theta=0.0, theta_amg=0.08, cycle="v")
    r = np.random.default_rng(3).standard_normal(A.nrows)
    monkeypatch.setenv("CPRB_TAIL_ROWS", "0")
    z0 = P.amg_cycle(P.build_hierarchy(P.pressure_matrix(A), cfg.amg_params()), r)
    monkeypatch.delenv("CPRB_TAIL_ROWS")
    monkeypatch.setenv("CPRB_TAIL_ROWS", "100000")
    z1 = P.amg_cycle(P.build_hierarchy(P.pressure_matrix(A), cfg.amg_params()), r)
    assert np.array_equal(z0, z1)


def test_device_kcycle_bitwise_equals_host_kcycle(gpu):
    """The C++-driven K-cycle with device Krylov scalars (csrc/kcycle.cu)
    performs the host-driven K-cycle's arithmetic: bitwise equal."""
    from paper_2201_01970_b200 import device as D
    A, _ = _c1()
    (A2, _), = P.generate_blackoil_like_sequence(24, 20, 12, 1, 0.01, 4).systems
    rng = np.random.default_rng(21)
    for M in (A, A2):
        cfg = P.SolverConfig(theta=0.0, theta_amg=0.0, cycle="k")
        h = P.build_hierarchy(P.pressure_matrix(M), cfg.amg_params())
        dev = h.device(1)
        assert dev.kdesc() is not None and len(h.levels) >= 4
        r = D.upload(rng.standard_normal(M.nrows))
        z_host = D.empty(M.nrows)
        z_dev = D.empty(M.nrows)
        dev.hostcycle(r, z_host, "k")
        dev.cycle(r, z_dev, "k")
        assert np.array_equal(z_host.cpu().numpy(), z_dev.cpu().numpy())


def test_device_kcycle_fgmres_flavour_matches_host(gpu):
    """FGMRES flavour (non-symmetric pressure operators, src/amg.py:199-225)
    of the device K-cycle against the host-driven one: equal up to the small
    least-squares solve (Givens QR on the device, LAPACK lstsq on the host)."""
    from paper_2201_01970_b200 import device as D
    (M, _), = P.generate_blackoil_like_sequence(24, 20, 12, 1, 0.01, 4).systems
    params = P.AmgParams(theta_amg=0.0, cycle="k", krylov="fgmres")
    h = P.build_hierarchy(P.pressure_matrix(M), params)
    dev = h.device(1)
    assert not dev.desc.use_fcg and dev.kdesc() is not None
    r = D.upload(np.random.default_rng(22).standard_normal(M.nrows))
    z_host, z_dev = D.empty(M.nrows), D.empty(M.nrows)
    dev.hostcycle(r, z_host, "k")
    dev.cycle(r, z_dev, "k")
    np.testing.assert_allclose(z_dev.cpu().numpy(), z_host.cpu().numpy(), rtol=1e-9, atol=1e-12)


def test_cpr_product_form_identity(gpu):
    """Eq. 8 (tests/test_cpr.py:98-118): I - B A = (I - R A)(I - Pi B_P Pi^T A)."""
    rng = np.random.default_rng(20240817)
    for A in (_bsr(random_block(rng, 12, b=3)), _csr(random_sparse(rng, 40, avg_nnz=5))):
        cfg = P.SolverConfig(coarsest_size=40, cycle="v", tol=1e-8, m=30)
        B = P.build_cpr(A, cfg)
        n = B.projector.fine_size
        Ad = A.to_dense()

        def assemble(op, size):
            M = np.zeros((size, size))
            for j in range(size):
                e = np.zeros(size)
                e[j] = 1.0
                M[:, j] = op(e)
            return M

        Bm = assemble(B.apply, n)
        Rm = assemble(lambda v: P.bilu_apply(B.relaxation, v), n)
        idx = B.projector.pressure_indices
        Pi = np.zeros((n, idx.shape[0]))
        Pi[idx, np.arange(idx.shape[0])] = 1.0
        BP = assemble(lambda v: P.amg_cycle(B.pressure_solver, v), idx.shape[0])
        lhs = np.eye(n) - Bm @ Ad
        rhs = (np.eye(n) - Rm @ Ad) @ (np.eye(n) - Pi @ BP @ Pi.T @ Ad)
        assert np.abs(lhs - rhs).max() <= 1e-10


# -- GMRES ------------------------------------------------------------------------


@pytest.mark.parametrize("tag", ["v0", "k0", "vd", "kd"])
def test_gmres_c1_against_reference(gpu, tag):
    A, b = _c1()
    g = load_golden(f"c1_{tag}.npz")
    cfg = P.SolverConfig(theta=0.0, theta_amg=0.0 if tag[1] == "0" else 0.08, cycle=tag[0])
    B = P.build_cpr(A, cfg)
    res = P.gmres_solve(A, b, None, B, cfg.gmres_params(), history=True)
    s = SUMMARY[tag]
    assert (res.outer, res.inner, res.converged) == (s["outer"], s["inner"], s["converged"])
    assert abs(res.rel_residual - s["rel"]) <= 1e-8 * s["rel"]
    hist = np.array([h if not isinstance(h, tuple) else -h[1] for h in res.history])
    np.testing.assert_allclose(hist, g["hist"], rtol=1e-8)
    assert np.linalg.norm(res.x - g["x"]) <= 1e-9 * np.linalg.norm(g["x"])


def test_gmres_kats(gpu):
    A = P.CsrMatrix.identity(9)
    b = np.linspace(1, 2, 9)
    res = P.gmres_solve(A, b, None, None, P.GmresParams(m=5, tol=1e-10))
    assert res.converged and res.outer == 1 and np.allclose(res.x, b, atol=1e-14)
    A = P.CsrMatrix.from_dense(np.diag(np.arange(1.0, 11.0)))
    res = P.gmres_solve(A, np.ones(10), None, None, P.GmresParams(m=10, tol=1e-5))
    assert res.converged and res.outer == 1
    assert np.linalg.norm(res.x - 1.0 / np.arange(1.0, 11.0)) <= 1e-8
    A = P.CsrMatrix.from_dense(np.diag([3.0, 5.0, 7.0]))
    res = P.gmres_solve(A, np.array([0.0, 2.0, 0.0]), None, None, P.GmresParams(m=5, tol=1e-12))
    assert res.converged and res.inner == 1 and np.allclose(res.x, [0.0, 0.4, 0.0], atol=1e-14)
    rng = np.random.default_rng(1)
    M = _csr(random_sparse(rng, 8))
    res = P.gmres_solve(M, np.zeros(8), None, None)
    assert res.converged and res.outer == 0 and res.inner == 0
    Pm = _csr(poisson_2d(10, 10))
    res = P.gmres_solve(Pm, rng.standard_normal(100), None, None,
                        P.GmresParams(m=2, max_restarts=3, tol=1e-14))
    assert not res.converged and res.outer == 3
    D = P.CsrMatrix.from_dense([[1e308, 0.0], [0.0, 1e308]])
    with pytest.raises(FloatingPointError):
        P.gmres_solve(D, np.array([1e308, 1e308]), np.array([1e308, 1e308]), None)


def test_gmres_matches_oracle_unpreconditioned(gpu):
    rng = np.random.default_rng(1234)
    for _ in range(6):
        n = int(rng.integers(5, 120))
        M = random_sparse(rng, n, avg_nnz=6)
        xs = rng.standard_normal(n)
        b = orc.spmv(M, xs)
        res = P.gmres_solve(_csr(M), b, None, None, P.GmresParams(m=30, max_restarts=400, tol=1e-8))
        ro = orc.gmres_solve(M, b, None, None, 30, 400, 1e-8)
        assert (res.outer, res.inner) == (ro.outer, ro.inner)
        assert np.linalg.norm(res.x - ro.x) <= 1e-9 * np.linalg.norm(ro.x)


def test_poisson32_vcycle_acceptance(gpu):
    A = _csr(poisson_2d(32, 32))
    h = P.build_hierarchy(A, P.AmgParams(coarsest_size=256, cycle="v"))
    b = np.ones(A.nrows)
    x = np.zeros(A.nrows)
    res = SUMMARY["poisson32"]["res"]
    for k in range(25):
        x = x + P.amg_cycle(h, b - P.spmv(A, x))
        # late cycles: |r| ~ 1e-7 |b|, so rounding of the coarse solve (dense
        # inverse vs the reference's LU) shows at ~1e-14 |b|
        assert abs(np.linalg.norm(b - P.spmv(A, x)) - res[k]) <= 1e-8 * res[k] + 1e-13 * 32.0
    assert np.linalg.norm(b) / res[-1] >= 1e6


def test_pressure16_vcycle(gpu):
    s = SUMMARY["press16"]
    A = P.problems.pressure_operator(16, 16, 16)
    h = P.build_hierarchy(A, P.AmgParams(theta_amg=0.0, cycle="v"))
    b = np.ones(A.nrows)
    x = np.zeros(A.nrows)
    for k in range(6):
        x = x + P.amg_cycle(h, b - P.spmv(A, x))
        rel = np.linalg.norm(b - P.spmv(A, x)) / np.linalg.norm(b)
        assert abs(rel - s["rel"][k]) <= 1e-9 * s["rel"][k]


def test_acceptance_sequence_iter50(gpu):
    """pkg/test_output.txt:203 (Iter=50, SetupCalls=1 on 32x32x4x10, mu=15)."""
    s = SUMMARY["accept_seq"]
    seq = P.generate_blackoil_like_sequence(32, 32, 4, 10, 0.01, seed=20240817)
    cfg = P.SolverConfig(theta=0.0, mu=15, m=28, tol=1e-5, cycle="v", coarsest_size=200)
    out = P.ascpr_gmres_sequence(seq.systems, 15, cfg)
    assert out.setup_calls == s["setup_calls"] and out.total_inner == s["total_inner"]
    assert [r.rebuilt for r in out.records] == s["rebuilt"]
    np.testing.assert_allclose([r.rel_residual for r in out.records], s["rel"], rtol=1e-8)


def test_ascpr_rules(gpu):
    rng = np.random.default_rng(7)
    A = _bsr(random_block(rng, 20, b=3))
    systems = [(A, P.spmv(A, rng.standard_normal(60))) for _ in range(4)]
    for mu, calls in ((0, 4), (10_000, 1)):
        out = P.ascpr_gmres_sequence(systems, mu=mu,
                                     config=P.SolverConfig(coarsest_size=40, cycle="v", tol=1e-9))
        assert out.setup_calls == calls and out.all_converged
        for (Ak, bk), rec in zip(systems, out.records):
            assert np.linalg.norm(bk - P.spmv(Ak, rec.x)) <= 1e-8 * np.linalg.norm(bk)


@pytest.mark.slow
def test_spe10_shape_c3_against_reference(gpu):
    """Config 3 (60x220x85, 3,366,000 DOF), theta_amg = 0, V-cycle: the
    reference's iteration counts, Givens history (1e-8) and solution (1e-6)."""
    path = GOLDEN / "c3_v0.json"
    if not path.exists():
        pytest.skip("c3 fixture not generated")
    ref = json.loads(path.read_text())
    (A, b), = P.generate_blackoil_like_sequence(60, 220, 85, 1, 0.01, 0).systems
    cfg = P.SolverConfig(theta=0.0, theta_amg=0.0, cycle="v")
    B = P.build_cpr(A, cfg)
    h = B.pressure_solver
    assert [l.A.nrows for l in h.levels] == ref["sizes"]
    assert [l.partition.c if l.partition else None for l in h.levels] == ref["colors"]
    res = P.gmres_solve(A, b, None, B, cfg.gmres_params(), history=True)
    assert (res.outer, res.inner) == (ref["outer"], ref["inner"])
    hist = np.array([hh if not isinstance(hh, tuple) else -hh[1] for hh in res.history])
    np.testing.assert_allclose(hist, ref["hist"], rtol=1e-8)
    xs = np.asarray(ref["x_sample"])
    got = res.x[::ref["x_sample_stride"]]
    assert np.linalg.norm(got - xs) <= 1e-6 * np.linalg.norm(xs)
    assert abs(np.linalg.norm(res.x) - ref["x_norm"]) <= 1e-6 * ref["x_norm"]


@pytest.mark.slow
def test_c2_pressure128_vcycle_against_survey(gpu):
    """Config 2: 128^3 pressure system (2,097,152 rows), stationary V(1,1)
    cycles from x = 0, b = ones.  Structure (levels, colours) is bit-exact to
    the reference run of SURVEY.md section 0.3 / Appendix C; the per-cycle
    relative residuals match the reference's printed values (4 digits)."""
    A = P.problems.pressure_operator(128, 128, 128)
    h = P.build_hierarchy(A, P.AmgParams(theta_amg=0.0, cycle="v"))
    sizes = [l.A.nrows for l in h.levels]
    assert len(sizes) == 15 and sizes[0] == 2097152 and sizes[-1] == 186
    assert [l.partition.c for l in h.levels[:-1]] == [2, 8, 9, 10, 11, 12, 12, 12, 12, 12, 12,
                                                       11, 12, 10]
    ref = [0.2716, 0.0953, 0.0384, 0.0173, 0.00841, 0.00429, 0.00227, 0.00123, 6.83e-4, 3.85e-4]
    import torch
    Ad = torch.from_numpy(np.ones(A.nrows)).cuda()
    b = Ad.clone()
    x = torch.zeros_like(b)
    nb = float(torch.linalg.vector_norm(b))
    for k in range(10):
        r = b - P.spmv(A, x)
        x = x + P.amg_cycle(h, r)
        rel = float(torch.linalg.vector_norm(b - P.spmv(A, x))) / nb
        assert abs(rel - ref[k]) <= 6e-3 * ref[k] + 1e-6, (k, rel, ref[k])


@pytest.mark.slow
def test_c4_sequence_reuse_against_survey(gpu):
    """Config 4 (all 10 SPE10-shaped Newton systems, mu = 5, V, theta_amg = 0):
    one setup, every solve 1 outer / 5 inner, and the final residuals of the
    reference run within 1e-8 relative -- the aging
    reused preconditioner (stage 2 multiplies by the FIRST system's matrix,
    src/cpr.py:185) must degrade exactly as the reference's does."""
    seq = P.generate_blackoil_like_sequence(60, 220, 85, 10, 0.01, 0)
    cfg = P.SolverConfig(theta=0.0, theta_amg=0.0, cycle="v")
    out = P.ascpr_gmres_sequence(seq.systems, 5, cfg, keep_solutions=False)
    assert out.setup_calls == 1
    assert [(r.outer, r.inner) for r in out.records] == [(1, 5)] * 10
    assert [r.rebuilt for r in out.records] == [True] + [False] * 9
    ref = [4.539505890669102e-06, 4.81992118102329e-06, 5.0585008937417845e-06,
           5.229715500921409e-06, 5.426977527133912e-06, 5.5681979247532605e-06,
           5.6903747842288935e-06, 5.837020329973612e-06, 6.001836858286181e-06,
           6.082489454699883e-06]
    np.testing.assert_allclose([r.rel_residual for r in out.records], ref, rtol=1e-8)


@pytest.mark.slow
def test_spe10_shape_c3_kcycle_against_reference(gpu):
    """Config 3 with the K-cycle (nonlinear AMLI, FCG on the symmetric A_PP),
    against the unmodified reference's run recorded in tests/golden/c3_k0.json
    (make_golden.py --bigk): outer 2 / inner 5 with the explicit-residual
    restart reproduced, the Givens history of both cycles within 1e-8, the
    solution samples within 1e-6 and ||x - x*|| / ||x*|| = 4.78e-6."""
    ref = json.loads((GOLDEN / "c3_k0.json").read_text())
    (A, b), = P.generate_blackoil_like_sequence(60, 220, 85, 1, 0.01, 0).systems
    cfg = P.SolverConfig(theta=0.0, theta_amg=0.0, cycle="k")
    B = P.build_cpr(A, cfg)
    assert B.pressure_solver.symmetric
    res = P.gmres_solve(A, b, None, B, cfg.gmres_params(), history=True)
    assert (res.outer, res.inner, res.converged) == (ref["outer"], ref["inner"], True) == (2, 5, True)
    hist = np.array([hh if not isinstance(hh, tuple) else -hh[1] for hh in res.history])
    np.testing.assert_allclose(hist, ref["hist"], rtol=1e-8)
    assert abs(res.rel_residual - ref["rel"]) <= 1e-8 * ref["rel"]
    xs_ref = np.asarray(ref["x_sample"])
    assert np.linalg.norm(res.x[::ref["x_sample_stride"]] - xs_ref) <= 1e-6 * np.linalg.norm(xs_ref)
    xs = P.problems.manufactured_solution(60 * 220 * 85)
    err = np.linalg.norm(res.x - xs) / np.linalg.norm(xs)
    assert abs(err - 4.78e-6) <= 0.01e-6


@pytest.mark.slow
def test_c4_sequence_rebuild_mix_against_reference(gpu):
    """Config 4 with a reuse/rebuild MIX (tests/golden/c4_mix.json, made by
    the unmodified reference: make_golden.py --c4mix): ten SPE10-shaped
    Newton systems, drift 0.05, mu = 5.  The aging preconditioner crosses mu
    mid-sequence, so ascpr_decide must rebuild exactly where the reference
    did (src/cpr.py:204-212), with the reference's iteration counts, final
    residuals (1e-8) and solutions (1e-6)."""
    path = GOLDEN / "c4_mix.json"
    if not path.exists():
        pytest.skip("c4_mix fixture not generated")
    ref = json.loads(path.read_text())
    seq = P.generate_blackoil_like_sequence(*ref["grid"], ref["nsteps"], ref["drift"], ref["seed"])
    cfg = P.SolverConfig(theta=0.0, theta_amg=0.0, cycle="v")
    out = P.ascpr_gmres_sequence(seq.systems, ref["mu"], cfg, keep_solutions=True)
    assert out.setup_calls == ref["setup_calls"]
    assert [r.rebuilt for r in out.records] == ref["rebuilt"]
    assert any(ref["rebuilt"][1:]) and not all(ref["rebuilt"])
    assert [[r.outer, r.inner] for r in out.records] == ref["its"]
    np.testing.assert_allclose([r.rel_residual for r in out.records], ref["rel"], rtol=1e-8)
    st = ref["x_sample_stride"]
    for r, xs in zip(out.records, ref["x_sample"]):
        xs = np.asarray(xs)
        assert np.linalg.norm(r.x[::st] - xs) <= 1e-6 * np.linalg.norm(xs)


def test_c_abi_gmres_driver_matches_python_driver(gpu):
    """cprb_gmres_solve (the whole restarted GMRES driven in C++, for hosts
    without Python) takes the same steps as gmres_solve: equal iteration
    counts and convergence, x and the relative residual equal to rounding."""
    import ctypes as C
    import torch
    from paper_2201_01970_b200 import _native as N
    from paper_2201_01970_b200 import device as D
    (A, b), = P.generate_blackoil_like_sequence(16, 12, 9, 1, 0.01, 3).systems
    for cycle in ("v", "k"):
        cfg = P.SolverConfig(theta=0.0, theta_amg=0.0, cycle=cycle)
        B = P.build_cpr(A, cfg)
        ref = P.gmres_solve(A, b, None, B, cfg.gmres_params())
        Bd = B.device()
        M = D.device_matrix(A)
        prm = cfg.gmres_params()
        n = b.shape[0]
        m = prm.m
        work = torch.zeros((m + 1) * n + 3 * n + 2 * m + 3 + 1184, dtype=torch.float64,
                           device="cuda")
        iwork = torch.zeros(4, dtype=torch.int32, device="cuda")
        bd = torch.from_numpy(b).cuda()
        x = torch.zeros(n, dtype=torch.float64, device="cuda")
        res = (C.c_double * 4)()
        desc = Bd.kdesc if cycle == "k" else Bd.desc   # the K-cycle's descriptor (set by apply)
        N.check(N.lib().cprb_gmres_solve(C.addressof(M.sell.desc), 3, C.addressof(desc),
                                         Bd.graphs, n, D.ptr(bd), D.ptr(x), m, prm.max_restarts,
                                         prm.tol, D.ptr(work), D.ptr(iwork), res, D.stream()))
        torch.cuda.synchronize()
        assert (int(res[0]), int(res[1]), bool(res[2])) == (ref.outer, ref.inner, ref.converged)
        assert abs(res[3] - ref.rel_residual) <= 1e-9 * ref.rel_residual
        xr = np.asarray(ref.x)
        assert np.linalg.norm(x.cpu().numpy() - xr) <= 1e-10 * np.linalg.norm(xr)
    # unpreconditioned, and the dimension check
    x.zero_()
    N.check(N.lib().cprb_gmres_solve(C.addressof(M.sell.desc), 3, None, None, n, D.ptr(bd),
                                     D.ptr(x), m, 2, 1e-30, D.ptr(work), D.ptr(iwork), res,
                                     D.stream()))
    torch.cuda.synchronize()
    assert int(res[0]) == 2 and int(res[1]) == 2 * m and not bool(res[2])
    assert N.lib().cprb_gmres_solve(C.addressof(M.sell.desc), 3, None, None, n - 3, D.ptr(bd),
                                    D.ptr(x), m, 2, 1e-6, D.ptr(work), D.ptr(iwork), res,
                                    D.stream()) == N.EINVAL
