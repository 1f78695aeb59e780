"""V-cycle critical path from the cprb_amg_set_log timeline
(tools/profile_path.py --what amgtl with AMGTL_OUT=...npy): block 0 of
launch i leaves griddepcontrol.wait when launch i-1 has completed, so the
completion-to-completion time of each launch is its cost on the dependent
chain (the block-0 start times only show how far PDL launched ahead).

    python tools/vcycle_critical_path.py gpurun_out/amgtl_r02b.npy > profiles/r02_vcycle_critical_path.txt
"""
import sys

import numpy as np

L = np.load(sys.argv[1]).astype(np.float64)
names = {1: "sweep", 2: "sweepZG", 3: "resid+restrict", 4: "prolong"}
t0 = L[0, 1]
rel = (L[:, 2] - t0) / 1e3          # block 0 past its wait = previous launch complete
kinds = [names[int(k)] for k in L[:, 0]]
cost = np.diff(rel)
print(f"{len(L)} launches, chain {rel[-1]:.1f} us to the last launch's release "
      f"(+ its own work {(L[-1, 3] - L[-1, 2]) / 1e3:.1f} us)")
tot = {}
for k, c in zip(kinds, cost):
    tot.setdefault(k, [0, 0.0])
    tot[k][0] += 1
    tot[k][1] += c
print("by kind: " + ", ".join(f"{k} {n} launches {v:.0f} us" for k, (n, v) in tot.items()))
small = cost[cost < 4.0]
print(f"launches costing < 4 us on the chain: {small.size}, median {np.median(small):.2f} us, "
      f"total {small.sum():.0f} us")
print("\nper launch (kind: completion-to-completion us), in launch order:")
for i in range(0, len(cost), 12):
    print("  " + " ".join(f"{kinds[j][:6]}:{cost[j]:.1f}" for j in range(i, min(i + 12, len(cost)))))
