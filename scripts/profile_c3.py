"""One C3-shaped round on one GPU (b=2048, 4096x4 MLP) for ncu."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
from paper_1806_02508_b200.mlp import MlpEngine, constant_trace
eng = MlpEngine(dims=[4096] * 5, global_batch=2048, n_workers_local=1, predictor="narx",
                warmup_iterations=50, max_iterations=40, trace=constant_trace(1, 40))
eng.run(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
torch.cuda.synchronize()
print("launches/round", eng.launches_per_iteration())
