"""C2 steady state: per-worker sizes, SM caps and per-phase times (debug helper)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
from paper_1806_02508_b200.mlp import MlpEngine, benchmark_trace, constant_trace
n, B = 8, 4096
for name, tr in (("trace", benchmark_trace(n, 200, seed=3)), ("ideal", constant_trace(n, 200))):
    eng = MlpEngine(dims=[784, 256, 10], global_batch=B, n_workers_local=n, predictor="narx",
                    warmup_iterations=50, max_iterations=200, trace=tr)
    eng.run(100)
    torch.cuda.synchronize()
    r = eng.records()
    ph = eng.worker_phase_times() * 1e6
    np.set_printoptions(precision=1, suppress=True, linewidth=150)
    print(f"== {name}: sizes {r['sizes'][-1]} caps {r['caps'][-1]}")
    for p in range(ph.shape[0]):
        print(f"phase {p} us", ph[p])
    print("t_worker us", r["t_worker"][-1] * 1e6)
    del eng
