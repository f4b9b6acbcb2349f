"""C3-shape engine on one GPU (4 x 4096x4096 MLP, 2 emulated workers, B=4096)
for profiling the HBM-bound kernels of the round (reduce+apply over P=67M
parameters, bias gradient, softmax-CE head) under ncu."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
from paper_1806_02508_b200.mlp import MlpEngine, constant_trace
n, B, iters = 2, 4096, 12
eng = MlpEngine(dims=[4096] * 5, global_batch=B, n_workers_local=n, scheme="lb-bsp",
                predictor="ema", max_iterations=iters, trace=constant_trace(n, iters, [1.0, 0.5]),
                learning_rate=0.01)
eng.run(8)
torch.cuda.synchronize()
print("ok")
ph = eng.phase_times()
print("phase times (ms) per phase x worker:")
print(ph)
