"""Runs a few C2 LB-BSP rounds after warm-up (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
from paper_1806_02508_b200.mlp import MlpEngine, benchmark_trace
n, B = 8, 4096
tr = benchmark_trace(n, 200, seed=3)
eng = MlpEngine(dims=[784, 256, 10], global_batch=B, n_workers_local=n, predictor="narx",
                warmup_iterations=50, max_iterations=200, trace=tr)
eng.run(int(sys.argv[1]) if len(sys.argv) > 1 else 100)
torch.cuda.synchronize()
print("launches/round", eng.launches_per_iteration())
