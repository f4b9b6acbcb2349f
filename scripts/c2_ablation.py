"""C2 round-time ablation: which branch is on the critical path (debug helper).
Per-step device time (CUDA events on the engine stream, L2 flushed between
steps like bench.py) for NARX vs EMA predictor and loss on/off."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
from paper_1806_02508_b200.mlp import MlpEngine, benchmark_trace, constant_trace

n, B = 8, 4096
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")


def per_step(eng, steps=60, warmup=60):
    st = torch.cuda.ExternalStream(eng.stream)
    eng.run(warmup)
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        flush.zero_()
        torch.cuda.synchronize()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(st); eng.run(1); e.record(st); e.synchronize()
        ts.append(s.elapsed_time(e))
    return np.median(ts) * 1e3, np.mean(ts) * 1e3


for pred in ("narx", "ema"):
    for loss_every in (1, 100000):
        for trname, tr in (("trace", benchmark_trace(n, 300, seed=3)), ("ideal", constant_trace(n, 300))):
            eng = MlpEngine(dims=[784, 256, 10], global_batch=B, n_workers_local=n, predictor=pred,
                            warmup_iterations=50, max_iterations=300, trace=tr, loss_every=loss_every,
                            learning_rate=0.05)
            med, mean = per_step(eng)
            print(f"{pred:5s} loss_every={loss_every:6d} {trname:5s}: median {med:7.1f} us  mean {mean:7.1f} us")
            del eng
