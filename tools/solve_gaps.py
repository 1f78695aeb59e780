"""GPU idle gaps inside one C3 solve (CUPTI kernel records via
torch.profiler): where the device waits for the host (Givens syncs,
launches)."""
import json
import sys
import tempfile
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile
import paper_2201_01970_b200 as P

(A, b), = P.generate_blackoil_like_sequence(60, 220, 85, 1, 0.01, 0).systems
cfg = P.SolverConfig(theta=0.0, theta_amg=0.0, cycle="v")
B = P.build_cpr(A, cfg)
bd = torch.from_numpy(b).cuda()
for _ in range(3):
    P.gmres_solve(A, bd, None, B, cfg.gmres_params())
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    P.gmres_solve(A, bd, None, B, cfg.gmres_params())
    torch.cuda.synchronize()
with tempfile.NamedTemporaryFile(suffix=".json") as f:
    prof.export_chrome_trace(f.name)
    tr = json.load(open(f.name))
ev = [e for e in tr["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
t0, t1 = ev[0]["ts"], max(e["ts"] + e["dur"] for e in ev)
busy_end = ev[0]["ts"]
gaps = []
for e in ev:
    if e["ts"] > busy_end:
        gaps.append((e["ts"] - busy_end, e["name"][:40]))
    busy_end = max(busy_end, e["ts"] + e["dur"])
g = np.array([x[0] for x in gaps])
print(f"span {t1 - t0:.0f} us, {len(ev)} device ops, idle {g.sum():.0f} us in {len(g)} gaps; "
      f"gaps > 5 us: {int((g > 5).sum())} totalling {g[g > 5].sum():.0f} us")
for d, n in sorted(gaps, reverse=True)[:15]:
    print(f"  {d:8.1f} us before {n}")
