"""Host SETUP (C++ library) against the reference's fixtures: generator,
aggregation, colouring, Galerkin products, level schedules, BILU(0).
CPU only (the C ABI's setup entry points need no GPU)."""

import hashlib
import json
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, load_golden, orc, poisson_2d, random_block, random_sparse, tridiag

import paper_2201_01970_b200 as P
from paper_2201_01970_b200 import _native as N
from paper_2201_01970_b200.ilu import _strict

SUMMARY = json.loads((GOLDEN / "summary.json").read_text())


def _csr(o):
    return P.CsrMatrix(o.nrows, o.ncols, o.ptr, o.cols, o.vals)


def _bsr(o):
    return P.BlockCsrMatrix(o.b, o.nrows, o.ncols, o.ptr, o.cols, o.vals)


def test_abi_exports_every_header_symbol():
    header = (ROOT / "include" / "cpr_b200.h").read_text()
    declared = set(re.findall(r"\b(cprb_[a-z0-9_]+)\s*\(", header))
    lib = N.lib()
    for name in sorted(declared):
        assert hasattr(lib, name), name
    assert declared == set(N.EXPORTS), declared ^ set(N.EXPORTS)
    assert lib.cprb_version() >= 1


def test_library_has_no_unresolved_internal_symbols():
    """A shared library links with undefined symbols; a missing definition of
    one of the package's own C++ functions would only fail when loaded on the
    GPU box.  Every undefined symbol must come from the CUDA runtime / libc."""
    import shutil
    import subprocess
    nm = shutil.which("nm")
    if nm is None:
        pytest.skip("nm not available")
    out = subprocess.run([nm, "-D", "--undefined-only", str(N._LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    bad = [ln for ln in out.splitlines() if "cprb" in ln]
    assert not bad, bad


def test_generator_bitwise_c1_and_sequence():
    g = load_golden("gen_c1.npz")
    (A, b), = P.generate_blackoil_like_sequence(10, 10, 10, 1, 0.01, 0).systems
    assert np.array_equal(A.row_ptr, g["ptr"]) and np.array_equal(A.col_idx, g["cols"])
    assert np.array_equal(A.values, g["vals"]) and np.array_equal(b, g["b"])
    g3 = load_golden("gen_seq3.npz")
    seq = P.generate_blackoil_like_sequence(6, 5, 4, 3, 0.05, 11)
    for k, (Ak, bk) in enumerate(seq.systems):
        assert np.array_equal(Ak.values, g3[f"vals{k}"]) and np.array_equal(bk, g3[f"b{k}"])


def test_generator_matches_oracle_odd_shapes():
    for shape, drift, seed in (((1, 1, 1), 0.0, 1), ((7, 1, 3), 0.02, 2), ((1, 9, 2), 0.3, 3),
                               ((4, 3, 5), 0.01, 4)):
        seq = P.generate_blackoil_like_sequence(*shape, 2, drift, seed)
        ref = orc.generate_blackoil_like_sequence(*shape, 2, drift, seed)
        for (A, b), (Ao, bo) in zip(seq.systems, ref):
            assert np.array_equal(A.row_ptr, Ao.ptr) and np.array_equal(A.col_idx, Ao.cols)
            assert np.array_equal(A.values, Ao.vals) and np.array_equal(b, bo)


def test_random_scalar_setup_bitwise():
    g = load_golden("random_scalar.npz")
    for ci in range(int(g["ncases"])):
        p = f"c{ci}_"
        n = g[p + "ptr"].shape[0] - 1
        A = P.CsrMatrix(n, n, g[p + "ptr"], g[p + "cols"], g[p + "vals"])
        part = P.vertices_grouping(P.strong_connections(A, float(g[p + "theta"])))
        assert np.array_equal(part.perm(), g[p + "perm"]), ci
        assert [x.shape[0] for x in part.groups] == g[p + "gsz"].tolist()
        assert P.verify_partition(A, float(g[p + "theta"]), part).ok
        agg = P.pairwise_aggregate(A, 0.05)
        assert np.array_equal(agg.aggregate_of, g[p + "agg"]), ci


@pytest.mark.parametrize("tag,th_amg", [("v0", 0.0), ("k0", 0.0), ("vd", 0.08), ("kd", 0.08)])
def test_c1_hierarchy_and_bilu(tag, th_amg):
    g = load_golden(f"c1_{tag}.npz")
    gen = load_golden("gen_c1.npz")
    A = P.BlockCsrMatrix(3, 1000, 1000, gen["ptr"], gen["cols"], gen["vals"])
    B = P.build_cpr(A, P.SolverConfig(theta=0.0, theta_amg=th_amg, cycle=tag[0]))
    h = B.pressure_solver
    assert len(h.levels) == int(g["h_nlev"]) and h.symmetric == bool(g["h_sym"])
    for li, lvl in enumerate(h.levels):
        assert np.array_equal(lvl.A.row_ptr, g[f"h{li}_ptr"])
        assert np.array_equal(lvl.A.col_idx, g[f"h{li}_cols"])
        assert np.array_equal(lvl.A.values, g[f"h{li}_vals"])          # Galerkin: bitwise
        if lvl.aggregates is not None:
            assert np.array_equal(lvl.aggregates, g[f"h{li}_agg"])
            assert np.array_equal(lvl.partition.perm(), g[f"h{li}_perm"])
            assert [x.shape[0] for x in lvl.partition.groups] == g[f"h{li}_gsz"].tolist()
    # coarsest operator: inverse equals inv(LU) of the reference to rounding
    lu, piv = g["h_lu"], g["h_piv"]
    import scipy.linalg
    ref_inv = scipy.linalg.lu_solve((lu, piv), np.eye(lu.shape[0]))
    np.testing.assert_allclose(h.coarsest_lu[1], ref_inv, rtol=1e-10, atol=1e-13)
    F = B.relaxation
    assert np.array_equal(np.concatenate(F.l_schedule.levels), g["f_llev"])
    assert np.array_equal(np.concatenate(F.u_schedule.levels), g["f_ulev"])
    lp, lc, lv = _strict(F.L)
    up, uc, uv = _strict(F.U)
    assert np.array_equal(lp, g["f_lptr"]) and np.array_equal(lc, g["f_lcols"])
    assert np.array_equal(up, g["f_uptr"]) and np.array_equal(uc, g["f_ucols"])
    # factor values: OpenBLAS dgemm vs plain products -> agree to rounding
    scale = np.abs(g["f_lvals"]).max()
    assert np.abs(lv - g["f_lvals"]).max() <= 1e-13 * scale
    assert np.abs(uv - g["f_uvals"]).max() <= 1e-13 * np.abs(g["f_uvals"]).max()
    assert np.abs(F.u_diag_inv - g["f_uinv"]).max() <= 1e-13 * np.abs(g["f_uinv"]).max()


def test_pressure16_hierarchy_digests():
    s = SUMMARY["press16"]
    A = P.problems.pressure_operator(16, 16, 16)
    h = P.build_hierarchy(A, P.AmgParams(theta_amg=0.0, cycle="v"))
    dg = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    assert [l.A.nrows for l in h.levels] == s["sizes"]
    assert [l.A.nnz for l in h.levels] == s["nnz"]
    assert [l.partition.c if l.partition else None for l in h.levels] == s["colors"]
    for li, lvl in enumerate(h.levels):
        assert dg(lvl.A.values) == s["vals_digests"][li]
        if lvl.aggregates is not None:
            assert dg(lvl.aggregates) == s["digests"][li]
            assert dg(lvl.partition.perm()) == s["perm_digests"][li]


def test_poisson32_hierarchy_sizes():
    A = _csr(poisson_2d(32, 32))
    h = P.build_hierarchy(A, P.AmgParams(coarsest_size=256, cycle="v"))
    assert [l.A.nrows for l in h.levels] == SUMMARY["poisson32"]["sizes"]


def test_setup_random_against_oracle():
    rng = np.random.default_rng(77)
    for trial in range(25):
        n = int(rng.integers(3, 400))
        theta = float(rng.choice([0.0, 0.0, 0.02, 0.1, 0.4, 1.0]))
        A = random_sparse(rng, n, avg_nnz=int(rng.integers(2, 9)),
                          dominant=bool(rng.integers(0, 2)), symmetric=bool(rng.integers(0, 2)))
        Ap = _csr(A)
        S = P.strong_connections(Ap, theta)
        So = orc.strong_connections(A, theta)
        assert np.array_equal(S.row_ptr, So.ptr) and np.array_equal(S.col_idx, So.cols)
        part = P.vertices_grouping(S)
        assert np.array_equal(part.perm(), np.concatenate(orc.vertices_grouping(So)))
        agg = P.pairwise_aggregate(Ap, theta)
        ao, nao = orc.pairwise_aggregate(A, theta)
        assert np.array_equal(agg.aggregate_of, ao) and agg.n_aggregates == nao
        Ac = P.amg._galerkin(Ap, agg)
        Aco = orc.galerkin(A, ao, nao)
        assert np.array_equal(Ac.row_ptr, Aco.ptr) and np.array_equal(Ac.col_idx, Aco.cols)
        assert np.array_equal(Ac.values, Aco.vals)
        assert P.amg._is_symmetric(Ap) == orc.is_symmetric(A)


def test_bilu_random_block_against_oracle():
    rng = np.random.default_rng(78)
    for trial in range(12):
        n = int(rng.integers(2, 90))
        A = random_block(rng, n, b=3, avg_nnz=int(rng.integers(2, 7)))
        F = P.bilu0_factorize(_bsr(A))
        Fo = orc.bilu0_factorize_fast(A)
        lp, lc, lv = _strict(F.L)
        assert np.array_equal(lc, Fo.l_cols) and np.array_equal(lp, Fo.l_ptr)
        np.testing.assert_allclose(lv, Fo.l_vals, rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(F.u_diag_inv, Fo.u_diag_inv, rtol=1e-12, atol=1e-14)
        for a, b in zip(F.l_schedule.levels, Fo.l_levels):
            assert np.array_equal(a, b)


def test_error_conventions():
    with pytest.raises(ValueError, match="theta"):
        P.strong_connections(_csr(tridiag(4)), 1.5)
    with pytest.raises(ValueError, match="triangular"):
        P.level_schedule(P.CsrMatrix.from_dense([[1.0, 1.0], [1.0, 1.0]]))
    with pytest.raises(np.linalg.LinAlgError, match="row 1"):
        P.bilu0_factorize(P.CsrMatrix.from_dense([[1.0, 1.0], [1.0, 1.0]]))
    block = np.array([[[1.0, 0.0], [0.0, 0.0]]])
    A = P.BlockCsrMatrix.from_block_coo(2, [0], [0], block, (1, 1))
    with pytest.warns(RuntimeWarning, match="perturbing"):
        F = P.bilu0_factorize(A)
    assert np.isfinite(F.u_diag_inv).all()
    with pytest.raises(np.linalg.LinAlgError, match="row 1"):
        P.sparse.invert_small_blocks(np.stack([np.eye(2), np.zeros((2, 2))]))
    with pytest.raises(ValueError, match="diagonal block missing"):
        P.BlockCsrMatrix.from_block_coo(2, [0, 1], [1, 1], np.ones((2, 2, 2)), (2, 2))
    with pytest.raises(np.linalg.LinAlgError, match="zero diagonal"):
        A = P.CsrMatrix.from_coo([0, 0, 1], [0, 1, 0], [1.0, 1.0, 1.0], (2, 2))
        P.PgsScmSmoother(A, P.vertices_grouping(P.strong_connections(A, 0.0)))


def test_invert_small_blocks_bitwise_oracle(rng):
    blocks = rng.standard_normal((300, 3, 3)) + 2.0 * np.eye(3)
    assert np.array_equal(P.sparse.invert_small_blocks(blocks), orc.invert_small_blocks(blocks))


def test_config_api():
    cfg = P.SolverConfig(theta=0.05, mu=20, workers=4)
    assert P.SolverConfig.from_dict(cfg.to_dict()) == cfg
    with pytest.raises(ValueError, match="unknown solver config"):
        P.SolverConfig.from_dict({"bogus": 1})
    with pytest.raises(ValueError):
        P.GmresParams(m=0)
    with pytest.raises(ValueError):
        P.AmgParams(cycle="w")


@pytest.mark.slow
def test_c3_setup_digests_against_reference():
    """Config 3 (60x220x85): every structural digest the unmodified reference
    recorded in tests/golden/c3_v0.json (make_golden.py --big): the Jacobian
    values and rhs, and per pressure level the aggregates, the colour
    permutation, the Galerkin values and columns, plus the BILU(0) level
    counts.  Host setup only (reference: src/cpr.py:168-175,
    src/amg.py:143-174, src/coloring.py:171-256, src/ilu.py:38-59)."""
    ref = json.loads((GOLDEN / "c3_v0.json").read_text())
    dg = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    (A, b), = P.generate_blackoil_like_sequence(60, 220, 85, 1, 0.01, 0).systems
    assert dg(A.values) == ref["vals_digest"]
    assert dg(b) == ref["b_digest"]
    B = P.build_cpr(A, P.SolverConfig(theta=0.0, theta_amg=0.0, cycle="v"))
    h = B.pressure_solver
    assert [l.A.nrows for l in h.levels] == ref["sizes"]
    assert [l.A.nnz for l in h.levels] == ref["nnz"]
    assert [l.partition.c if l.partition else None for l in h.levels] == ref["colors"]
    for li, lvl in enumerate(h.levels):
        assert dg(lvl.A.values) == ref["lvl_vals_digests"][li], li
        assert dg(lvl.A.col_idx) == ref["lvl_cols_digests"][li], li
        if lvl.aggregates is not None:
            assert dg(lvl.aggregates) == ref["agg_digests"][li], li
            assert dg(lvl.partition.perm()) == ref["perm_digests"][li], li
        else:
            assert ref["agg_digests"][li] is None
    assert B.relaxation.l_schedule.n_levels == ref["bilu_llev"]
    assert B.relaxation.u_schedule.n_levels == ref["bilu_ulev"]


def _pack_sell_numpy(lane_row, lane_ptr, ent_cols, ent_vals, bs):
    """The per-entry numpy scatter the native fills replaced (layout spec)."""
    L = lane_row.shape[0]
    ns = L // 32
    lens = np.diff(lane_ptr)
    width = lens.reshape(ns, 32).max(axis=1)
    sp = np.zeros(ns + 1, dtype=np.int64)
    np.cumsum(width * 32, out=sp[1:])
    nnz = int(lens.sum())
    lane_of = np.repeat(np.arange(L), lens)
    m = np.arange(nnz) - lane_ptr[lane_of]
    lane = lane_of % 32
    d = sp[lane_of // 32] + m * 32 + lane
    cols = np.zeros(max(int(sp[-1]), 1), dtype=np.int32)
    cols[d] = ent_cols
    bb = bs * bs
    vals = np.zeros(max(int(sp[-1]) * bb, 1))
    if bb == 1:
        vals[d] = ent_vals
    else:
        idx = ((d - lane) * bb)[:, None] + np.arange(bb)[None, :] * 32 + lane[:, None]
        vals[idx.reshape(-1)] = ent_vals.reshape(-1)
    return sp, cols, vals


@pytest.mark.parametrize("bs", [1, 3])
def test_native_sell_fills_match_layout(rng, bs):
    from paper_2201_01970_b200 import device as D
    L = 32 * 7
    lens = rng.integers(0, 9, size=L)
    lens[rng.random(L) < 0.2] = 0
    lane_ptr = np.zeros(L + 1, dtype=np.int64)
    np.cumsum(lens, out=lane_ptr[1:])
    nnz = int(lane_ptr[-1])
    ec = rng.integers(0, 1000, size=nnz)
    ev = rng.standard_normal((nnz, bs, bs)) if bs > 1 else rng.standard_normal(nnz)
    lane_row = np.where(lens > 0, np.arange(L), -1).astype(np.int32)
    h = D.pack_sell(lane_row, lane_ptr, ec, ev, bs, L)
    sp, cols, vals = _pack_sell_numpy(lane_row, lane_ptr, ec, ev, bs)
    assert np.array_equal(h.slice_ptr, sp) and np.array_equal(h.cols, cols)
    assert np.array_equal(h.vals, vals)
    # rows of a CSR, columns renumbered: equal to the per-lane-list packing
    A = P.CsrMatrix.from_dense((rng.random((100, 100)) < 0.05) * rng.standard_normal((100, 100)))
    perm = rng.permutation(100)
    inv = np.empty(100, dtype=np.int64)
    inv[perm] = np.arange(100)
    src = D.pad_lanes(perm.astype(np.int64))
    got = D.sell_from_rows(src, A.row_ptr, A.col_idx, A.values, 100, colmap=inv)
    lp = np.zeros(src.shape[0] + 1, dtype=np.int64)
    ln = np.where(src >= 0, np.diff(A.row_ptr)[np.maximum(src, 0)], 0)
    np.cumsum(ln, out=lp[1:])
    ent = np.concatenate([np.arange(A.row_ptr[r], A.row_ptr[r + 1]) for r in src if r >= 0])
    sp, cols, vals = _pack_sell_numpy(got.lane_row, lp, inv[A.col_idx[ent]], A.values[ent], 1)
    assert np.array_equal(got.slice_ptr, sp) and np.array_equal(got.cols, cols)
    assert np.array_equal(got.vals, vals)
