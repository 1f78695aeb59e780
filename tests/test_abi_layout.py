"""The ctypes mirrors in paper_2201_01970_b200/_native.py must match the C
structs of include/cpr_b200.h byte for byte (size and every field offset):
compiled here with gcc, no GPU needed."""

from __future__ import annotations

import ctypes as C
import shutil
import subprocess
from pathlib import Path

import pytest

from paper_2201_01970_b200 import _native as N

ROOT = Path(__file__).resolve().parents[1]
STRUCTS = {"cprb_sell": N.Sell, "cprb_amg_level": N.AmgLevel,
           "cprb_amg": N.Amg, "cprb_wave": N.Wave, "cprb_stencil": N.Stencil, "cprb_bilu": N.Bilu, "cprb_cpr": N.Cpr}


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_ctypes_layout_matches_header(tmp_path):
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "cpr_b200.h"', "int main(void) {"]
    for cname, py in STRUCTS.items():
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'  printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", f"-I{ROOT / 'include'}", str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {}
    for ln in out:
        if ln.strip():
            parts = ln.split()
            got[(parts[0], parts[1])] = int(parts[2])
    for cname, py in STRUCTS.items():
        assert got[(cname, "size")] == C.sizeof(py), cname
        for fname, _ in py._fields_:
            assert got[(cname, fname)] == getattr(py, fname).offset, (cname, fname)
