"""Probe (GPU): the bench's e2e section repeated on fresh engines (C2, NARX,
benchmark trace, huge-page host buffers, warm-up through step_e2e), with an
event after every step on the engine stream: is a slow e2e run slow in
every step or in a few? REPS repetitions."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
from paper_1806_02508_b200.mlp import MlpEngine, benchmark_trace
from paper_1806_02508_b200.hostio import pinned_empty
n, B, warm, steps = 8, 4096, 100, 100
trace = benchmark_trace(n, warm + steps + 12, seed=3)
for rep in range(int(os.environ.get("REPS", "6"))):
    eng = MlpEngine(dims=[784, 256, 10], global_batch=B, n_workers_local=n, predictor="narx",
                    warmup_iterations=50, learning_rate=0.05, seed=1, max_iterations=warm + steps + 8, trace=trace)
    x, y = eng.dataset()
    xb = pinned_empty(x.shape, torch.bfloat16, 0); xb.copy_(torch.from_numpy(x).to(torch.bfloat16))
    yb = pinned_empty(y.shape, torch.int32, 0); yb.copy_(torch.from_numpy(y.astype(np.int32)))
    osz = pinned_empty((n,), torch.int32, 0); ol = pinned_empty((1,), torch.float64, 0)
    st = torch.cuda.ExternalStream(eng.stream)
    # this rep's host buffer: standalone H2D copy time, and whether the
    # kernel granted it huge pages
    dx = torch.empty(xb.shape, dtype=xb.dtype, device="cuda")
    ts = []
    for _ in range(200):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); dx.copy_(xb, non_blocking=True); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    h2d = float(np.median(ts[100:]))
    addr = xb.data_ptr()
    thp = "?"
    try:
        cur = None
        for line in open("/proc/self/smaps"):
            if "-" in line.split()[0] and len(line.split()) >= 5 and all(c in "0123456789abcdef-" for c in line.split()[0]):
                lo, hi = (int(v, 16) for v in line.split()[0].split("-"))
                cur = lo <= addr < hi
            elif cur and line.startswith("AnonHugePages:"):
                thp = line.split()[1] + " kB"
                break
    except OSError:
        pass
    eng.run(warm - 5)
    for _ in range(5):
        eng.step_e2e(xb.data_ptr(), yb.data_ptr(), osz.data_ptr(), ol.data_ptr())
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    ev[0].record(st)
    t0 = time.perf_counter()
    for i in range(steps):
        eng.step_e2e(xb.data_ptr(), yb.data_ptr(), osz.data_ptr(), ol.data_ptr())
        ev[i + 1].record(st)
    th = (time.perf_counter() - t0) / steps * 1e6
    ev[-1].synchronize()
    d = np.array([ev[i].elapsed_time(ev[i + 1]) * 1e3 for i in range(steps)])
    p = np.percentile(d, [10, 50, 90, 99])
    print(f"rep {rep}: H2D {h2d:5.1f} us, THP {thp}; e2e {d.mean():6.1f} us/step (host {th:5.1f})  p10 {p[0]:6.1f} p50 {p[1]:6.1f} p90 {p[2]:6.1f} "
          f"p99 {p[3]:6.1f} max {d.max():7.1f}", flush=True)
    del eng
