"""MatrixMarket I/O and sequence manifests (src/mmio.py, src/problems.py:158-194)
against the behaviour recorded from the unmodified reference
(tests/golden/make_mmio_golden.py -> tests/golden/mmio.json): every reader
outcome (arrays or the exact line-numbered error), the written file bytes,
and save/load_sequence.  CPU only."""

import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN

import paper_2201_01970_b200 as P
from paper_2201_01970_b200 import mmio as M
from paper_2201_01970_b200 import problems as PR

G = json.loads((GOLDEN / "mmio.json").read_text())


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _outcome(fn, p):
    try:
        A = fn(p)
    except Exception as exc:  # noqa: BLE001
        return {"err": type(exc).__name__, "msg": str(exc).replace(str(p), "<path>")}
    d = {"nrows": int(A.nrows), "ncols": int(A.ncols), "ptr": _digest(A.row_ptr),
         "cols": _digest(A.col_idx), "vals": _digest(A.values)}
    if hasattr(A, "block_size"):
        d["block_size"] = int(A.block_size)
    return d


@pytest.mark.parametrize("name", sorted(G["cases"]))
def test_reader_matches_reference(tmp_path, name):
    case = G["cases"][name]
    p = tmp_path / f"{name}.mtx"
    p.write_text("\n".join(case["text"]) + ("\n" if case["text"] else ""))
    assert _outcome(M.read_matrix_market, p) == case["scalar"]
    assert _outcome(M.read_block_matrix_market, p) == case["block"]


def test_fast_path_and_python_fallback_agree(tmp_path):
    rng = np.random.default_rng(5)
    D = rng.standard_normal((60, 45)) * (rng.random((60, 45)) < 0.2)
    A = P.CsrMatrix.from_dense(D)
    p = tmp_path / "a.mtx"
    M.write_matrix_market(p, A)
    fast = M._read_entries(str(p))
    slow = M._read_entries_py(str(p))
    for a, b in zip(fast, slow):
        if isinstance(a, np.ndarray):
            assert np.array_equal(a, b)
        else:
            assert a == b


@pytest.mark.parametrize("k", [0, 1, 2])
def test_writer_bytes_match_reference(tmp_path, k):
    w = G["writes"][f"scalar{k}"]
    n, m = w["shape"]
    rng = np.random.default_rng(w["seed"])
    for kk in range(k + 1):      # replay the generator's draws up to case k
        nn, mm, dens = [(5, 5, 0.5), (40, 31, 0.1), (200, 200, 0.03)][kk]
        D = rng.standard_normal((nn, mm)) * (rng.random((nn, mm)) < dens)
        D[0, 0] = 1e-310
        if nn > 1:
            D[1, 0] = -0.0 if D[1, 0] == 0 else D[1, 0]
    assert _digest(D) == w["dense_digest"]
    p = tmp_path / "w.mtx"
    M.write_matrix_market(p, P.CsrMatrix.from_dense(D))
    assert _digest(np.frombuffer(p.read_bytes(), dtype=np.uint8)) == w["sha"]
    B = M.read_matrix_market(p)               # read -> write -> read is bitwise
    assert np.array_equal(B.to_dense(), D)


def test_sequence_manifest_round_trip(tmp_path, monkeypatch):
    s = G["sequence"]
    monkeypatch.setattr(PR, "_cuda_ok", lambda: False)
    seq = P.generate_blackoil_like_sequence(*s["args"])
    man = P.save_sequence(seq, tmp_path / "seq")
    files = {f.name: _digest(np.frombuffer(f.read_bytes(), dtype=np.uint8))
             for f in sorted((tmp_path / "seq").iterdir())}
    assert files == s["files"]
    assert json.loads(man.read_text()) == s["manifest"]
    back = P.load_sequence(man)
    assert [[_digest(A.values), _digest(b)] for A, b in back.systems] == s["reloaded"]
    for (A, b), (A2, b2) in zip(seq.systems, back.systems):
        assert np.array_equal(A.values, A2.values) and np.array_equal(b, b2)


def test_vector_round_trip(tmp_path):
    x = np.random.default_rng(2).standard_normal(33)
    x[3] = -0.0
    p = tmp_path / "v.mtx"
    M.write_vector(p, x)
    assert np.array_equal(M.read_vector(p).view(np.uint64), x.view(np.uint64))
