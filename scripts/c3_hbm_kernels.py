"""C3-shape engine on one GPU (4 x 4096x4096 MLP, B=4096) for profiling the
HBM-bound kernels of the round (reduce+apply over P=67M parameters, bias
gradient, softmax-CE head), in the graph (phase stamps of each worker) and
under ncu. N_WORKERS (default 2) emulated workers, AVAIL a comma list of
availabilities (default 1.0 for every worker: no interference in the
stamps)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
from paper_1806_02508_b200.mlp import MlpEngine, constant_trace
n = int(os.environ.get("N_WORKERS", "2"))
avail = [float(a) for a in os.environ.get("AVAIL", ",".join(["1.0"] * n)).split(",")]
B, iters = 4096, 12
eng = MlpEngine(dims=[4096] * 5, global_batch=B, n_workers_local=n, scheme="lb-bsp",
                predictor="ema", max_iterations=iters, trace=constant_trace(n, iters, avail),
                learning_rate=0.01)
eng.run(8)
torch.cuda.synchronize()
print("ok")
names = ["fwd0", "fwd1", "fwd2", "fwd3", "softmax_ce", "db3", "dW3", "dX3", "db2", "dW2", "dX2", "db1", "dW1",
         "dX1", "db0", "dW0"]
wp = eng.worker_phase_times() * 1e6
rows = eng.records()["sizes"][7]
print("rows per worker", rows.tolist())
for i, row in enumerate(wp):
    nm = names[i] if i < len(names) else f"ph{i}"
    extra = ""
    if nm.startswith("db") or nm == "softmax_ce":
        gbs = [r * 4096 * 2 / (t * 1e-6) / 1e9 for r, t in zip(rows, row) if t > 0]
        extra = "  dZ/logits read GB/s per worker " + " ".join(f"{x:.0f}" for x in gbs)
    print(f"{nm:>10s} us per worker " + " ".join(f"{t:7.1f}" for t in row) + extra)
