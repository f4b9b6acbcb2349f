"""H2D bandwidth of the 1.57 MB per-round dataset upload against the NUMA
placement of the page-locked buffer (debug helper): pages are first-touched by
the allocating thread, so the buffer lands on the node the process runs on."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
from paper_1806_02508_b200.hostio import gpu_local_cpus

NB = 1568000
local = gpu_local_cpus(0)
allc = os.sched_getaffinity(0)
remote = allc - local if local else set()
print("gpu-local cpus:", sorted(local)[:4], "...", len(local), "of", len(allc), flush=True)
dx = torch.empty(NB // 2, dtype=torch.bfloat16, device="cuda")
for name, cpus in (("all", allc), ("local", local), ("remote", remote), ("local", local)):
    if not cpus:
        continue
    os.sched_setaffinity(0, cpus)
    for b in range(3):
        x = torch.empty(NB // 2, dtype=torch.bfloat16, pin_memory=True)
        x.fill_(1.0)
        for _ in range(3):
            dx.copy_(x, non_blocking=True)
        torch.cuda.synchronize()
        ts = []
        for _ in range(30):
            s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
            s.record(); dx.copy_(x, non_blocking=True); e.record(); e.synchronize()
            ts.append(s.elapsed_time(e) * 1e3)
        ts.sort()
        print(f"{name:6s} buf{b}: median {ts[15]:6.1f} us  min {ts[0]:6.1f}  max {ts[-1]:6.1f}  "
              f"({NB / ts[15] / 1e3:5.1f} GB/s)", flush=True)
    os.sched_setaffinity(0, allc)
