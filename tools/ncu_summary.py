"""Summarise ncu --set full captures (gpurun_out/final_*.ncu-rep) into
profiles/<round>_ncu_summary.md and profiles/ncu_traffic.json (the DRAM
traffic per launch that bench.py reports as roofline.traffic).

    python tools/ncu_summary.py r01            # gpurun_out/final_*.ncu-rep
    python tools/ncu_summary.py r02            # gpurun_out/r02_*.ncu-rep

Families already in profiles/ncu_traffic.json that this round did not
re-capture are kept.
"""
import csv
import io
import json
import subprocess
import sys
from collections import Counter, defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "lts__t_sector_hit_rate.pct", "launch__grid_size", "launch__block_size"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "nsecond": 1e-9, "us": 1e-6, "ns": 1e-9, "ms": 1e-3,
         "msecond": 1e-3}


def raw(rep):
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"name": r[h.index("Kernel Name")].split("(")[0]}
        for m in METRICS:
            if m in h:
                i = h.index(m)
                try:
                    d[m] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)
                except ValueError:
                    d[m] = r[i]
        out.append(d)
    return out


lines = [f"# {tag}: ncu --set full captures of the committed kernels (C3, 1 B200)", "",
         "Command: `tools/ncu_round1_final.sh` under gpurun (`ncu --set full --clock-control none "
         "--import-source on -k regex:<kernel>` on `tools/profile_path.py`).  Times are ncu's "
         "(serialised, caches flushed): compare shares, not absolutes.", "",
         "| kernel | grid x block | time us | DRAM read MB | DRAM write MB | DRAM % of peak | warps active % | regs | L2 hit % |",
         "|---|---|---|---|---|---|---|---|---|"]
traffic = {}
FAMILY = {"bsr": "bsr_spmv", "sweep": "pgs_scm_sweep_l0", "rr": "resid_restrict_l0",
          "wave": "bilu_apply", "stencil": "bilu_apply", "ktail": "kcycle_tail"}
prefix = "final" if tag == "r01" else tag
for rep in sorted(OUT.glob(f"{prefix}_*.ncu-rep")):
    f = rep.stem[len(prefix) + 1:]
    if f not in FAMILY:
        continue
    for d in raw(rep):
        lines.append(f"| {d['name']} | {d.get('launch__grid_size'):.0f} x {d.get('launch__block_size'):.0f} | "
                     f"{d['gpu__time_duration.sum'] * 1e6:.1f} | {d['dram__bytes_read.sum'] / 1e6:.1f} | "
                     f"{d['dram__bytes_write.sum'] / 1e6:.1f} | "
                     f"{d['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']:.1f} | "
                     f"{d['sm__warps_active.avg.pct_of_peak_sustained_active']:.1f} | "
                     f"{d['launch__registers_per_thread']:.0f} | {d['lts__t_sector_hit_rate.pct']:.1f} |")
        fam = FAMILY[f]
        b = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
        traffic.setdefault(fam, {"dram_bytes": 0, "launches": 0})
        traffic[fam]["dram_bytes"] += b
        traffic[fam]["launches"] += 1
# the sweep capture holds the two level-0 colour launches of one pass; wave holds L + U
for fam in traffic:
    traffic[fam]["dram_bytes"] = int(traffic[fam]["dram_bytes"])
lst = OUT / ("launches_solve_final.csv" if tag == "r01" else f"launches_solve_{tag}.csv")
if lst.exists():
    rows = list(csv.reader(open(lst)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    tot, cnt = defaultdict(float), Counter()
    # SETUP kernels (device factorisation, packing, generator) run before the
    # solves in the same process; the table is about the SOLVE path
    setup = ("k_bilu_level", "k_stencil_pack", "k_pack_", "k_gen_", "k_fill", "k_sell_",
             "k_factor", "k_scatter_vals", "k_uinv")
    for r in rows[hi + 1:]:
        if len(r) <= vi or (mi is not None and r[mi] != "gpu__time_duration.sum"):
            continue
        v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1e-9) * 1e6
        nm = r[ki].split("(")[0].replace("void ", "").replace("cprb::", "")[:40]
        if nm.startswith(setup):
            continue
        tot[nm] += v
        cnt[nm] += 1
    T = sum(tot.values())
    lines += ["", "## Launch list: one warm-up + one timed C3 solve (`ncu --metrics gpu__time_duration.sum`; setup kernels excluded)",
              "", f"{sum(cnt.values())} launches, {T / 1e3:.2f} ms summed (serialised, cold caches).", "",
              "| kernel | launches | summed us | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:16]:
        lines.append(f"| {k} | {cnt[k]} | {v:.0f} | {v / T * 100:.1f}% |")
(ROOT / "profiles" / f"{tag}_ncu_summary.md").write_text("\n".join(lines) + "\n")
tj = ROOT / "profiles" / "ncu_traffic.json"
old = json.loads(tj.read_text()) if tj.exists() else {"kernels": {}}
for fam, v in traffic.items():
    v["source"] = f"profiles/{tag}_ncu_summary.md"
    old["kernels"][fam] = v
old.update({"source": "ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum per launch "
                      "group (per-family source file)", "grid": [60, 220, 85]})
tj.write_text(json.dumps(old, indent=1) + "\n")
print("\n".join(lines))
