"""Build a variant of the native library with extra nvcc defines applied to
one source (diagnostics):  python tools/build_variant.py NAME SRC -DFOO ...
Output: tools/NAME/libcprb200.so (load it with CPRB_LIB=...)."""
import concurrent.futures as cf
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2201_01970_b200 import build_native as B  # noqa: E402

name, target, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
out = ROOT / "tools" / name
out.mkdir(exist_ok=True)
objd = Path("/tmp") / f"objs_{name}"
objd.mkdir(exist_ok=True)
nvcc = B._nvcc()
cmds, objs = [], []
for src in B._sources():
    obj = objd / (src.name + ".o")
    objs.append(obj)
    if src.suffix == ".cu":
        cmd = [nvcc, *B.ARCH, *B.NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
        if src.name == target:
            cmd += defs
    else:
        cmd = ["g++", *B.CXX_FLAGS, "-c", str(src), "-o", str(obj)]
    cmds.append(cmd)


def run(cmd):
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode:
        raise SystemExit(p.stderr)


with cf.ThreadPoolExecutor(8) as ex:
    list(ex.map(run, cmds))
run([nvcc, *B.ARCH, "-shared", "-o", str(out / "libcprb200.so"), *map(str, objs)])
print(out / "libcprb200.so")
