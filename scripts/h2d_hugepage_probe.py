"""Probe (GPU): host->device copy rate of the C2 e2e step's 1.57 MB upload
from page-locked memory backed by 4 KB pages (torch pin_memory) vs a
2 MB-aligned transparent-huge-page mapping registered with cudaHostRegister
(fewer IOMMU translations per DMA). Each variant: 1500 copies, median of the
last 500, two passes in alternating order."""
import ctypes, mmap, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
from paper_1806_02508_b200.hostio import gpu_local_cpus
nbytes = 1000 * 784 * 2 + 1000 * 4
d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
local = gpu_local_cpus(0)
if local:
    os.sched_setaffinity(0, local)
# 4 KB pinned
h4 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True); h4.zero_()
# THP: 2 MB aligned anonymous mapping, madvise(HUGEPAGE), touched, registered
span = 4 << 20
mm = mmap.mmap(-1, span, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
base = ctypes.addressof(ctypes.c_char.from_buffer(mm))
off = (-base) % (2 << 20)
try:
    mm.madvise(mmap.MADV_HUGEPAGE, off, 2 << 20)
except Exception as e:
    print("madvise:", e)
buf = (ctypes.c_char * (2 << 20)).from_buffer(mm, off)
ctypes.memset(buf, 0, 2 << 20)
ptr = base + off
rt = torch.cuda.cudart()
err = rt.cudaHostRegister(ptr, 2 << 20, 0)
print("cudaHostRegister:", err)
try:
    with open("/proc/self/smaps") as f:
        txt = f.read()
    import re
    print("AnonHugePages total (kB):", sum(int(x) for x in re.findall(r"AnonHugePages:\s+(\d+)", txt)))
except Exception as e:
    print(e)
hthp = torch.frombuffer(buf, dtype=torch.uint8, count=nbytes)
main = torch.cuda.current_stream()
def run(h, name):
    ts = []
    for rep in range(1500):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(main)
        d.copy_(h, non_blocking=True)
        e.record(main)
        e.synchronize()
        if rep >= 1000:
            ts.append(s.elapsed_time(e) * 1e3)
    ts.sort()
    med = ts[len(ts) // 2]
    print(f"{name}: median {med:.1f} us ({nbytes / med / 1e3:.1f} GB/s), p10 {ts[len(ts)//10]:.1f}, p90 {ts[9*len(ts)//10]:.1f}", flush=True)
for h, name in ((hthp, "THP-registered"), (h4, "4KB pinned"), (hthp, "THP-registered"), (h4, "4KB pinned")):
    run(h, name)
