"""Probe (GPU): where the e2e step time goes -- isolated pinned H2D of the
dataset, the device round, the e2e step (lbbsp_mlp_step_e2e) and the host
time per e2e call."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
from paper_1806_02508_b200.mlp import MlpEngine, benchmark_trace
from paper_1806_02508_b200.hostio import pinned_empty

n, B = 8, 4096
eng = MlpEngine(dims=[784, 256, 10], global_batch=B, n_workers_local=n, predictor="narx",
                warmup_iterations=50, max_iterations=400, trace=benchmark_trace(n, 400, seed=3))
x, y = eng.dataset()
xb = pinned_empty(x.shape, torch.bfloat16, 0); xb.copy_(torch.from_numpy(x).to(torch.bfloat16))
yb = pinned_empty(y.shape, torch.int32, 0); yb.copy_(torch.from_numpy(y.astype(np.int32)))
osz = pinned_empty((n,), torch.int32, 0); ol = pinned_empty((1,), torch.float64, 0)
dx = torch.empty(xb.shape, dtype=xb.dtype, device="cuda")
s = torch.cuda.Stream()
for rep in range(3):
    ts = []
    for _ in range(100):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record(); dx.copy_(xb, non_blocking=True); b.record()
        b.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
    print(f"H2D 1.57 MB pinned: median {np.median(ts):.1f} us min {min(ts):.1f} "
          f"({x.size*2/np.median(ts)/1e3:.1f} GB/s)", flush=True)
st = torch.cuda.ExternalStream(eng.stream)
eng.run(100)
torch.cuda.synchronize()
for mode in ("run", "e2e", "run", "e2e"):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(st)
    t0 = time.perf_counter()
    for _ in range(40):
        if mode == "run":
            eng.run(1)
        else:
            eng.step_e2e(xb.data_ptr(), yb.data_ptr(), osz.data_ptr(), ol.data_ptr())
    host = (time.perf_counter() - t0) / 40 * 1e6
    b.record(st); b.synchronize()
    print(f"{mode}: device {a.elapsed_time(b)/40*1e3:.1f} us/step, host {host:.1f} us/call", flush=True)
