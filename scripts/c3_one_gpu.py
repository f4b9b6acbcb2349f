"""C3 per-GPU shape (MLP 4 x 4096^2 bf16, one worker, 2048 rows) for ncu:
a few rounds of the worker phases (CTA-pair tcgen05 GEMMs, bias, softmax-CE,
apply, dataset loss)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
from paper_1806_02508_b200.mlp import MlpEngine, constant_trace

R = int(os.environ.get("ROUNDS", "4"))
eng = MlpEngine(dims=[4096] * 5, global_batch=2048, n_workers_local=1, predictor="ema",
                learning_rate=0.01, max_iterations=R + 2, trace=constant_trace(1, R + 2))
eng.run(R)
torch.cuda.synchronize()
ph = eng.phase_times()
print("phases_us", [round(x * 1e6, 1) for x in ph], "worker_ms", float(eng.records()["t_worker"][-1][0]) * 1e3)
