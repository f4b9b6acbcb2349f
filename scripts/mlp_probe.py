"""Quick timing of MLP LB-BSP rounds (CUDA events on the engine stream)."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
from paper_1806_02508_b200.mlp import MlpEngine, benchmark_trace, constant_trace

def timed(eng, warm, iters):
    eng.run(warm); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    st = torch.cuda.ExternalStream(eng.stream)
    s.record(st); eng.run(iters); e.record(st); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters

for name, dims, B, n in [("C2", [784, 256, 10], 4096, 8), ("C3-1gpu", [4096]*5, 2048, 1)]:
    it = 60
    for scheme, tr in [("lb-bsp", benchmark_trace(n, 400, 3)), ("bsp", benchmark_trace(n, 400, 3)), ("ideal", constant_trace(n, 400))]:
        eng = MlpEngine(dims=dims, global_batch=B, n_workers_local=n, scheme="lb-bsp" if scheme != "bsp" else "bsp",
                        predictor="narx", warmup_iterations=50, max_iterations=400, trace=tr)
        ms = timed(eng, 60, it)
        rec = eng.records()
        print(f"{name} {scheme:6s}: {ms*1e3:9.1f} us/round  {B/ms*1e3:12.0f} samples/s  launches={eng.launches_per_iteration()} loss0={rec['loss'][0]:.4f} lossN={rec['loss'][rec['rows']-1]:.4f}")
        print("   last sizes", rec["sizes"][-1].tolist(), "caps", rec["caps"][-1].tolist(), "t_worker(us)", (rec["t_worker"][-1]*1e6).round(1).tolist())
        f, b = eng.work()
        print(f"   gemm flops/round {f/1e9:.2f} GF -> {f/ms/1e9:.1f} TF/s")
        del eng
