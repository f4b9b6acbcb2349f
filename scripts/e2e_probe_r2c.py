"""Probe (GPU): e2e step vs device round on the same engine, constant trace,
EMA predictor (no NARX tail): the cost the host I/O adds per round."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
from paper_1806_02508_b200.mlp import MlpEngine, constant_trace, benchmark_trace
from paper_1806_02508_b200.hostio import pinned_empty
n, B = 8, 4096
eng = MlpEngine(dims=[784, 256, 10], global_batch=B, n_workers_local=n, predictor=os.environ.get("PRED", "ema"),
                warmup_iterations=50, max_iterations=1200, trace=(benchmark_trace(n, 1200, seed=3) if os.environ.get("TRACE") == "bench" else constant_trace(n, 1200)))
x, y = eng.dataset()
xb = pinned_empty(x.shape, torch.bfloat16, 0); xb.copy_(torch.from_numpy(x).to(torch.bfloat16))
yb = pinned_empty(y.shape, torch.int32, 0); yb.copy_(torch.from_numpy(y.astype(np.int32)))
osz = pinned_empty((n,), torch.int32, 0); ol = pinned_empty((1,), torch.float64, 0)
st = torch.cuda.ExternalStream(eng.stream)
eng.run(100)
eng.step_e2e(xb.data_ptr(), yb.data_ptr(), osz.data_ptr(), ol.data_ptr())
torch.cuda.synchronize()
dx = torch.empty(xb.shape, dtype=xb.dtype, device="cuda")
cs = torch.cuda.Stream()
ts = []
for _ in range(50):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(cs):
        a.record(); dx.copy_(xb, non_blocking=True); b.record()
    b.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
print(f"H2D 1.57 MB: median {np.median(ts):.1f} us", flush=True)
for mode in ("run", "load+run", "run+read", "e2e") * 2:
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(50):
        if mode == "run":
            eng.run(1)
        elif mode == "load+run":
            eng.load_data_async(xb.data_ptr(), yb.data_ptr()); eng.run(1)
        elif mode == "run+read":
            eng.run(1); eng.read_result_async(osz.data_ptr(), ol.data_ptr())
        else:
            eng.step_e2e(xb.data_ptr(), yb.data_ptr(), osz.data_ptr(), ol.data_ptr())
    st.wait_stream(torch.cuda.ExternalStream(eng.result_stream))
    b.record(st); b.synchronize()
    print(f"{mode:9s}: {a.elapsed_time(b)/50*1e3:6.1f} us/step", flush=True)
