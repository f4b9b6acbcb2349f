"""Per-round device time distribution of the e2e loop vs the device-resident
loop over the same rounds (debug helper): percentiles of event-to-event gaps."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
from paper_1806_02508_b200.mlp import MlpEngine, benchmark_trace
from paper_1806_02508_b200.hostio import pinned_empty
n = 8
scratch = None
for mode in ("run", "e2e", "run", "e2e", "load", "indep", "read"):
    eng = MlpEngine(dims=[784, 256, 10], global_batch=4096, n_workers_local=8, predictor="narx",
                    warmup_iterations=50, max_iterations=400, trace=benchmark_trace(n, 400, seed=3),
                    learning_rate=0.05, seed=1)
    x, y = eng.dataset()
    xb = pinned_empty(x.shape, torch.bfloat16); xb.copy_(torch.from_numpy(x).to(torch.bfloat16))
    yb = pinned_empty(y.shape, torch.int32); yb.copy_(torch.from_numpy(y.astype(np.int32)))
    osz = pinned_empty((n,), torch.int32); ol = pinned_empty((1,), torch.float64)
    st = torch.cuda.ExternalStream(eng.stream)
    eng.run(50)
    for _ in range(60):
        eng.load_data_async(xb.data_ptr(), yb.data_ptr()); eng.run(1)
        eng.read_result_async(osz.data_ptr(), ol.data_ptr())
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(101)]
    ev[0].record(st)
    cs = torch.cuda.Stream()
    scratch = torch.empty(x.shape, dtype=torch.bfloat16, device="cuda")
    for i in range(100):
        if mode == "indep":  # an unrelated H2D copy of the same bytes, no dependency on the engine
            with torch.cuda.stream(cs):
                scratch.copy_(xb, non_blocking=True)
        if mode in ("e2e", "load"):
            eng.load_data_async(xb.data_ptr(), yb.data_ptr())
        eng.run(1)
        if mode in ("e2e", "read"):
            eng.read_result_async(osz.data_ptr(), ol.data_ptr())
        ev[i + 1].record(st)
    ev[-1].synchronize()
    d = np.array([ev[i].elapsed_time(ev[i + 1]) * 1e3 for i in range(100)])
    p = np.percentile(d, [10, 50, 90, 99])
    print(f"{mode}: mean {d.mean():6.1f} us  p10 {p[0]:6.1f}  p50 {p[1]:6.1f}  p90 {p[2]:6.1f}  p99 {p[3]:6.1f}  "
          f"max {d.max():6.1f}  top5 rounds {np.argsort(d)[-5:].tolist()}", flush=True)
    del eng
