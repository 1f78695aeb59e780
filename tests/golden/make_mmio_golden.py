"""Golden behaviour of the reference's MatrixMarket I/O and sequence manifests
(cprkit.mmio, src/mmio.py; cprkit.problems save/load_sequence,
src/problems.py:158-194), recorded from the UNMODIFIED reference:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_mmio_golden.py

For every case text the reader's outcome (the CSR arrays, or the exception
type and message with the file path replaced by <path>) and, for written
matrices/vectors, the SHA-256 of the file bytes.  Output:
tests/golden/mmio.json.
"""
from __future__ import annotations

import hashlib
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent

H = "%%MatrixMarket matrix coordinate real general"
S = "%%MatrixMarket matrix coordinate real symmetric"
CASES = {
    "diag": [H, "2 2 2", "1 1 2.0", "2 2 2.0"],
    "sym": [S, "2 2 3", "1 1 2.0", "2 1 -1.0", "2 2 2.0"],
    "comments_blank": [H, "% a comment", "", "3 3 3", "% inside", "1 1 1e-300", "",
                       "3 3 -0.0", "2 3 +4.5E+2"],
    "specials": [H, "2 2 4", "1 1 inf", "1 2 -Infinity", "2 1 nan", "2 2 .5"],
    "count_mismatch": [H, "2 2 3", "1 1 1.0", "2 2 1.0"],
    "bad_header": ["%%MatrixMarket matrix array real general", "2 2 1", "1 1 1.0"],
    "bad_field": ["%%MatrixMarket matrix coordinate complex general", "1 1 1", "1 1 1 0"],
    "bad_symmetry": ["%%MatrixMarket matrix coordinate real hermitian", "1 1 1", "1 1 1.0"],
    "short_header": ["%%MatrixMarket matrix coordinate real", "1 1 1", "1 1 1.0"],
    "out_of_range": [H, "2 2 2", "1 1 1.0", "3 1 1.0"],
    "duplicate": [H, "2 2 3", "1 1 1.0", "2 2 1.0", "1 1 5.0"],
    "too_many": [H, "2 2 1", "1 1 1.0", "2 2 1.0"],
    "bad_entry_fields": [H, "2 2 1", "1 1"],
    "bad_entry_value": [H, "2 2 1", "1 1 x"],
    "bad_entry_index": [H, "2 2 1", "1.0 1 1.0"],
    "hex_value": [H, "1 1 1", "1 1 0x1p3"],
    "underscore": [H, "1 1 1", "1 1 1_000.5"],
    "bad_size_fields": [H, "2 2", "1 1 1.0"],
    "bad_size_int": [H, "2 2 a", "1 1 1.0"],
    "missing_size": [H, "% only comments", ""],
    "header_only": [H],
    "sym_nonsquare": [S, "2 3 1", "1 1 1.0"],
    "sym_mirror_dup": [S, "2 2 2", "1 2 1.0", "2 1 1.0"],
    "block_ok": [H, "% block_size: 2", "4 4 5", "1 1 1.0", "1 2 2.0", "2 1 3.0", "3 3 4.0",
                 "4 4 5.0"],
    "block_bad_sidecar": [H, "% block_size: two", "2 2 1", "1 1 1.0"],
    "block_missing": [H, "2 2 1", "1 1 1.0"],
    "block_indivisible": [H, "% block_size: 2", "3 3 1", "1 1 1.0"],
    "empty": [],
}


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def outcome(fn, p):
    try:
        M = fn(p)
    except Exception as exc:  # noqa: BLE001 - recording the reference's behaviour
        return {"err": type(exc).__name__, "msg": str(exc).replace(str(p), "<path>")}
    d = {"nrows": int(M.nrows), "ncols": int(M.ncols), "ptr": digest(M.row_ptr),
         "cols": digest(M.col_idx), "vals": digest(M.values)}
    if hasattr(M, "block_size"):
        d["block_size"] = int(M.block_size)
    return d


def main():
    sys.path.insert(0, REF)
    from cprkit import mmio
    from cprkit.problems import generate_blackoil_like_sequence, load_sequence, save_sequence
    from cprkit.sparse import CsrMatrix
    out = {"cases": {}, "writes": {}}
    with tempfile.TemporaryDirectory() as td:
        td = Path(td)
        for name, lines in CASES.items():
            p = td / f"{name}.mtx"
            p.write_text("\n".join(lines) + ("\n" if lines else ""))
            out["cases"][name] = {"text": lines,
                                  "scalar": outcome(mmio.read_matrix_market, p),
                                  "block": outcome(mmio.read_block_matrix_market, p)}
        rng = np.random.default_rng(7)
        for k, (n, m, dens) in enumerate([(5, 5, 0.5), (40, 31, 0.1), (200, 200, 0.03)]):
            D = rng.standard_normal((n, m)) * (rng.random((n, m)) < dens)
            D[0, 0] = 1e-310
            if n > 1:
                D[1, 0] = -0.0 if D[1, 0] == 0 else D[1, 0]
            A = CsrMatrix.from_dense(D)
            p = td / f"w{k}.mtx"
            mmio.write_matrix_market(p, A)
            out["writes"][f"scalar{k}"] = {"shape": [n, m], "seed": 7, "sha": digest(np.frombuffer(
                p.read_bytes(), dtype=np.uint8)), "dense_digest": digest(D)}
        seq = generate_blackoil_like_sequence(4, 3, 2, 2, 0.05, 3)
        man = save_sequence(seq, td / "seq")
        files = {f.name: digest(np.frombuffer(f.read_bytes(), dtype=np.uint8))
                 for f in sorted((td / "seq").iterdir())}
        back = load_sequence(man)
        out["sequence"] = {"args": [4, 3, 2, 2, 0.05, 3], "files": files,
                           "manifest": json.loads(man.read_text()),
                           "reloaded": [[digest(A.values), digest(b)] for A, b in back.systems]}
    (OUT / "mmio.json").write_text(json.dumps(out, indent=1) + "\n")
    print("wrote", OUT / "mmio.json")


if __name__ == "__main__":
    main()
