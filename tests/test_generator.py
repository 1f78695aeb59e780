"""Synthetic Jacobian generator (src/problems.py:74-155): the host
restatement and the device assembly (csrc/gen.cu) against the fixtures made
by the unmodified reference (tests/golden/gen_c1.npz, gen_seq3.npz) and
against each other -- bitwise."""

import numpy as np
import pytest

from conftest import load_golden

import paper_2201_01970_b200 as P
from paper_2201_01970_b200 import problems as PR


def _check_golden(seq_fn):
    g = load_golden("gen_c1.npz")
    (A, b), = seq_fn(10, 10, 10, 1, 0.01, 0).systems
    assert np.array_equal(A.row_ptr, g["ptr"]) and np.array_equal(A.col_idx, g["cols"])
    assert np.array_equal(A.values, g["vals"]) and np.array_equal(b, g["b"])
    g = load_golden("gen_seq3.npz")
    for k, (A, b) in enumerate(seq_fn(6, 5, 4, 3, 0.05, 11).systems):
        assert np.array_equal(A.row_ptr, g["ptr"])
        assert np.array_equal(A.values, g[f"vals{k}"]) and np.array_equal(b, g[f"b{k}"])


def test_host_generator_matches_reference_fixtures(monkeypatch):
    monkeypatch.setattr(PR, "_cuda_ok", lambda: False)
    _check_golden(P.generate_blackoil_like_sequence)


@pytest.mark.gpu
def test_device_generator_matches_reference_fixtures(gpu):
    assert PR._cuda_ok()
    _check_golden(P.generate_blackoil_like_sequence)


@pytest.mark.gpu
@pytest.mark.parametrize("dims,drift", [((23, 17, 9), 0.07), ((2, 3, 2), 0.0), ((1, 5, 7), 0.3),
                                        ((40, 1, 1), 0.02)])
def test_device_assembly_equals_host_restatement(gpu, monkeypatch, dims, drift):
    """Odd grids, degenerate axes and drift = 0 (signed zeros): every value
    and right-hand side bit-identical to the host restatement."""
    dev = P.generate_blackoil_like_sequence(*dims, 3, drift, 9).systems
    monkeypatch.setattr(PR, "_cuda_ok", lambda: False)
    host = P.generate_blackoil_like_sequence(*dims, 3, drift, 9).systems
    for (A, b), (Ah, bh) in zip(dev, host):
        assert np.array_equal(A.row_ptr, Ah.row_ptr) and np.array_equal(A.col_idx, Ah.col_idx)
        assert np.array_equal(A.values.view(np.uint64), Ah.values.view(np.uint64))
        assert np.array_equal(b.view(np.uint64), bh.view(np.uint64))


@pytest.mark.gpu
def test_device_generator_keeps_device_copy(gpu):
    """The generated matrix's device copy is the one the solve uses (no
    re-upload) and release_device() frees it."""
    from paper_2201_01970_b200 import device as D
    (A, b), = P.generate_blackoil_like_sequence(12, 10, 8, 1, 0.01, 3).systems
    M = getattr(A, "_cprb_dev", None)
    assert M is not None and D.device_matrix(A) is M
    x = np.random.default_rng(1).standard_normal(A.nrows * 3)
    assert np.array_equal(P.spmv(A, x), PR.bsr_matvec_reference_order(A, x))
    D.release_device(A)
    assert getattr(A, "_cprb_dev", None) is None
