"""Per-node cost of CUDA graph replay on this box (torch tiny kernels)."""
import os
import time

import torch

print({k: v for k, v in os.environ.items() if k.startswith(("CUDA", "NCCL", "TORCH", "PYTORCH"))})
x = torch.zeros(1, device="cuda")
s = torch.cuda.Stream()
for n in (10, 100, 1000):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        x.add_(1.0)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(n):
                x.add_(1.0)
    g.replay(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        g.replay()
    e1.record(); torch.cuda.synchronize()
    print(f"graph of {n:5d} tiny kernels: {e0.elapsed_time(e1) / 20 * 1e3 / n:.2f} us/node")
t0 = time.perf_counter()
for _ in range(2000):
    x.add_(1.0)
torch.cuda.synchronize()
print(f"eager launch: {(time.perf_counter() - t0) / 2000 * 1e6:.2f} us/launch")
print(torch.cuda.get_device_properties(0))
os.system("nvidia-smi -q | grep -iE 'persistence|compute mode|MIG|clocks event|Performance' | head -20; nproc; lscpu | grep -E 'Model name|MHz'")
