"""Host vs device time of the e2e loop at N=1 (debug helper): each mode on a
fresh engine over the same rounds 60..160 of the C2 trace."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
from paper_1806_02508_b200.mlp import MlpEngine, benchmark_trace
from paper_1806_02508_b200.hostio import pinned_empty
MODES = os.environ.get("MODES", "run only,e2e,load only,read only,run only,e2e,load only,read only").split(",")
LOCAL = os.environ.get("LOCAL", "0") == "1"
n = 8
for mode in MODES:
    eng = MlpEngine(dims=[784, 256, 10], global_batch=4096, n_workers_local=8,
                    predictor=os.environ.get("PRED", "narx"), warmup_iterations=50,
                    max_iterations=400, trace=benchmark_trace(n, 400, seed=3), learning_rate=0.05)
    x, y = eng.dataset()
    pe = pinned_empty if LOCAL else (lambda sh, dt: torch.empty(sh, dtype=dt, pin_memory=True))
    xb = pe(x.shape, torch.bfloat16); xb.copy_(torch.from_numpy(x).to(torch.bfloat16))
    yb = pe(y.shape, torch.int32); yb.copy_(torch.from_numpy(y.astype(np.int32)))
    osz = pe((n,), torch.int32); ol = pe((1,), torch.float64)
    st = torch.cuda.ExternalStream(eng.stream)
    eng.run(100); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        s.record(st)
    t0 = time.perf_counter()
    for i in range(100):
        if mode in ("e2e", "load only"):
            eng.load_data_async(xb.data_ptr(), yb.data_ptr())
        eng.run(1)
        if mode in ("e2e", "read only"):
            eng.read_result_async(osz.data_ptr(), ol.data_ptr())
    t1 = time.perf_counter()
    with torch.cuda.stream(st):
        e.record(st)
    e.synchronize()
    print(f"{mode}: host {1e6*(t1-t0)/100:.1f} us/step, device {s.elapsed_time(e)*10:.1f} us/step", flush=True)
    del eng
