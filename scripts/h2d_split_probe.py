"""Probe (GPU): host->device copy time of the C2 e2e step's 1.57 MB dataset
upload from NUMA-local page-locked memory, as one copy or split into 2/4
chunks on as many streams (copy engines), median over 300 copies after 300
warm copies; plus the PCIe link state from NVML. The buffer comes from
hostio.pinned_empty (huge pages when available)."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
from paper_1806_02508_b200.hostio import pinned_empty
nbytes = 1000 * 784 * 2 + 1000 * 4
h = pinned_empty((nbytes,), torch.uint8, 0)
d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
try:
    import pynvml
    pynvml.nvmlInit()
    hd = pynvml.nvmlDeviceGetHandleByIndex(0)
    print("PCIe gen %d x%d (max gen %d x%d)" % (pynvml.nvmlDeviceGetCurrPcieLinkGeneration(hd),
          pynvml.nvmlDeviceGetCurrPcieLinkWidth(hd), pynvml.nvmlDeviceGetMaxPcieLinkGeneration(hd),
          pynvml.nvmlDeviceGetMaxPcieLinkWidth(hd)))
except Exception as e:
    print("nvml:", e)
streams = [torch.cuda.Stream() for _ in range(4)]
main = torch.cuda.current_stream()
for parts in (1, 4, 1, 4, 2):
    ts = []
    for rep in range(600):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(main)
        ch = (nbytes + parts - 1) // parts
        for p in range(parts):
            st = streams[p]
            st.wait_stream(main)
            with torch.cuda.stream(st):
                d[p * ch:(p + 1) * ch].copy_(h[p * ch:(p + 1) * ch], non_blocking=True)
        for p in range(parts):
            main.wait_stream(streams[p])
        e.record(main)
        e.synchronize()
        if rep >= 300:
            ts.append(s.elapsed_time(e) * 1e3)
    ts.sort()
    med = ts[len(ts) // 2]
    print(f"{parts} chunk(s): median {med:.1f} us ({nbytes / med / 1e3:.1f} GB/s), p10 {ts[len(ts)//10]:.1f}, p90 {ts[9*len(ts)//10]:.1f}")
