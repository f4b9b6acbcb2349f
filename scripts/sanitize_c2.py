"""Runs a few C2 rounds (fused worker kernel, NARX, interference) for
compute-sanitizer (racecheck / synccheck / memcheck). The beside-the-plan
gather is joined by a graph edge (LBBSP_GATHER_JOIN) because the tool
serialises kernels. NO_STRAGGLE=1: availability 1 (an ncu capture of the
worker kernel without injected interference traffic)."""
import os, sys
os.environ.setdefault("LBBSP_GATHER_JOIN", "1")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
from paper_1806_02508_b200.mlp import MlpEngine, benchmark_trace, constant_trace

n, R = 8, int(os.environ.get("ROUNDS", "6"))
eng = MlpEngine(dims=[784, 256, 10], global_batch=4096, n_workers_local=n, predictor="narx",
                warmup_iterations=3, max_iterations=R + 2, trace=(constant_trace(n, R + 2) if os.environ.get("NO_STRAGGLE")
                       else benchmark_trace(n, R + 2, seed=3)))
eng.run(R)
torch.cuda.synchronize()
rec = eng.records()
print("rounds", rec["rows"], "sizes", rec["sizes"][-1].tolist(), "loss", rec["loss"][-1])
