"""Probe (GPU): e2e step composition -- device time per step of run only,
load + run, run + read, and the full step_e2e, after the pinned buffers are
warm (C2, benchmark trace, rounds 100+)."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
from paper_1806_02508_b200.mlp import MlpEngine, benchmark_trace
from paper_1806_02508_b200.hostio import pinned_empty

n, B = 8, 4096
eng = MlpEngine(dims=[784, 256, 10], global_batch=B, n_workers_local=n, predictor=os.environ.get("PRED", "narx"),
                warmup_iterations=50, max_iterations=1200, trace=benchmark_trace(n, 1200, seed=3))
x, y = eng.dataset()
xb = pinned_empty(x.shape, torch.bfloat16, 0); xb.copy_(torch.from_numpy(x).to(torch.bfloat16))
yb = pinned_empty(y.shape, torch.int32, 0); yb.copy_(torch.from_numpy(y.astype(np.int32)))
osz = pinned_empty((n,), torch.int32, 0); ol = pinned_empty((1,), torch.float64, 0)
st = torch.cuda.ExternalStream(eng.stream)
eng.run(100)
eng.step_e2e(xb.data_ptr(), yb.data_ptr(), osz.data_ptr(), ol.data_ptr())  # warms the buffers
torch.cuda.synchronize()
for mode in ("run", "load+run", "run+read", "e2e") * 3:
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(st)
    t0 = time.perf_counter()
    for _ in range(40):
        if mode == "run":
            eng.run(1)
        elif mode == "load+run":
            eng.load_data_async(xb.data_ptr(), yb.data_ptr()); eng.run(1)
        elif mode == "run+read":
            eng.run(1); eng.read_result_async(osz.data_ptr(), ol.data_ptr())
        else:
            eng.step_e2e(xb.data_ptr(), yb.data_ptr(), osz.data_ptr(), ol.data_ptr())
    host = (time.perf_counter() - t0) / 40 * 1e6
    b.record(st); b.synchronize()
    print(f"{mode:9s}: device {a.elapsed_time(b)/40*1e3:6.1f} us/step, host {host:5.1f} us/call", flush=True)
