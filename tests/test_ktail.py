"""Persistent K-cycle tail (csrc/ktail.cu) against the launched K-cycle
(csrc/kcycle.cu, itself bitwise equal to the host-driven K-cycle): the tail
runs the same arithmetic operation for operation, so every configuration must
agree BITWISE -- FCG and FGMRES flavours, snapshot colours (theta_amg > 0),
pre/post sweep counts, both CTA sizes, and tail starts from level 1 down to
the last Krylov level.  src/amg.py:177-225, :245-267."""

import numpy as np
import pytest

import paper_2201_01970_b200 as P

pytestmark = pytest.mark.gpu


def _kcycle(M, params, env, monkeypatch, r):
    from paper_2201_01970_b200 import device as D
    for k, v in env.items():
        monkeypatch.setenv(k, str(v))
    h = P.build_hierarchy(P.pressure_matrix(M), params)
    dev = h.device(1)
    assert dev.kdesc() is not None
    z = D.empty(M.nrows)
    dev.cycle(D.upload(r), z, "k")
    return z.cpu().numpy(), h


def _system(nx, ny, nz, seed=4):
    (M, _), = P.generate_blackoil_like_sequence(nx, ny, nz, 1, 0.01, seed).systems
    return M


CASES = [
    ("fcg", 0.0, 1, 1),
    ("fcg", 0.08, 1, 1),
    ("fcg", 0.0, 2, 1),
    ("fcg", 0.0, 0, 1),
    ("fcg", 0.0, 1, 2),
    ("fgmres", 0.0, 1, 1),
    ("fgmres", 0.08, 1, 1),
]


@pytest.mark.parametrize("krylov,theta_amg,pre,post", CASES)
@pytest.mark.parametrize("threads", [512, 1024])
def test_ktail_bitwise_equals_launched_kcycle(gpu, monkeypatch, krylov, theta_amg, pre, post,
                                              threads):
    M = _system(24, 20, 12)
    params = P.AmgParams(theta_amg=theta_amg, cycle="k", krylov=krylov, pre_sweeps=pre,
                         post_sweeps=post)
    r = np.random.default_rng(5).standard_normal(M.nrows)
    z_ref, h = _kcycle(M, params, {"CPRB_KTAIL_ROWS": 0}, monkeypatch, r)
    assert len(h.levels) >= 5
    for rows in (100_000, 2_000, 300):   # tail from level 1, a middle level, the last frames
        z, _ = _kcycle(M, params, {"CPRB_KTAIL_ROWS": rows, "CPRB_KTAIL_THREADS": threads},
                       monkeypatch, r)
        assert np.array_equal(z, z_ref), (rows, float(np.max(np.abs(z - z_ref))))


def test_ktail_zero_rhs_and_breakdowns(gpu, monkeypatch):
    """r = 0 takes FCG's "norm2(r) == 0" exit at every frame (z = 0); a
    residual living on a single row exercises the early-exit paths below."""
    M = _system(16, 12, 8)
    params = P.AmgParams(theta_amg=0.0, cycle="k")
    for r in (np.zeros(M.nrows), np.eye(1, M.nrows, 7)[0]):
        z_ref, _ = _kcycle(M, params, {"CPRB_KTAIL_ROWS": 0}, monkeypatch, r)
        z, _ = _kcycle(M, params, {"CPRB_KTAIL_ROWS": 100_000}, monkeypatch, r)
        assert np.array_equal(z, z_ref)


@pytest.mark.parametrize("tag", ["k0", "kd"])
def test_ktail_solve_c1_against_reference(gpu, monkeypatch, tag):
    """C1 K-cycle solves with the whole Krylov recursion in the tail (from
    level 1): the reference's iteration counts, Givens history (1e-8) and
    solution (tests/golden/c1_k0.npz, c1_kd.npz)."""
    import json
    from conftest import GOLDEN, load_golden
    g = load_golden("gen_c1.npz")
    A = P.BlockCsrMatrix(3, 1000, 1000, g["ptr"], g["cols"], g["vals"])
    ref = load_golden(f"c1_{tag}.npz")
    s = json.loads((GOLDEN / "summary.json").read_text())[tag]
    monkeypatch.setenv("CPRB_KTAIL_ROWS", "100000")
    cfg = P.SolverConfig(theta=0.0, theta_amg=0.0 if tag == "k0" else 0.08, cycle="k")
    B = P.build_cpr(A, cfg)
    res = P.gmres_solve(A, g["b"], None, B, cfg.gmres_params(), history=True)
    assert (res.outer, res.inner, res.converged) == (s["outer"], s["inner"], s["converged"])
    assert abs(res.rel_residual - s["rel"]) <= 1e-8 * s["rel"]
    hist = np.array([h if not isinstance(h, tuple) else -h[1] for h in res.history])
    np.testing.assert_allclose(hist, ref["hist"], rtol=1e-8)
    assert np.linalg.norm(res.x - ref["x"]) <= 1e-9 * np.linalg.norm(ref["x"])
