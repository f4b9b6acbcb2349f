"""Multi-rank LB-BSP with dynamic sizes (VERDICT r1 next-round
1(c)). Launched by tests/test_gpu_multi.py through torch.distributed.run with
2 ranks -- on 2 GPUs, or with --same-device as two processes sharing cuda:0
(the peer buffers are CUDA-IPC mappings either way, so the single-GPU tier
runs the same exchange code). No NCCL: the control plane is gloo (handle
exchange only); speeds and gradients move through the peer-memory kernels /
copy engines.

Each rank writes its records and final weights to --out; the pytest side
compares them with the reference replay and the restatement.
  --mode c2: several workers per GPU (4 per rank, MLP 784-256-10), NARX
  --mode c3: one worker per GPU (MLP 1024^4), bf16 copy-engine buckets, EMA
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
import torch.distributed as dist

from paper_1806_02508_b200.mlp import MlpEngine, benchmark_trace, connect

ap = argparse.ArgumentParser()
ap.add_argument("--mode", default="c2", choices=["c2", "c3"])
ap.add_argument("--same-device", action="store_true")
ap.add_argument("--rounds", type=int, default=24)
ap.add_argument("--out", required=True)
a = ap.parse_args()

world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(0 if a.same_device else local)
dist.init_process_group("gloo", init_method="env://")
R = a.rounds
if a.mode == "c2":
    dims, n_local, B, pred, lr = [784, 256, 10], 4, 2048 * world, "narx", 0.05
else:
    dims, n_local, B, pred, lr = [1024] * 4, 1, 1024 * world, "ema", 0.02
n = n_local * world
trace = benchmark_trace(n, R + 4, seed=3)
eng = MlpEngine(dims=dims, global_batch=B, n_workers_local=n_local, world=world, rank=rank,
                scheme="lb-bsp", predictor=pred, warmup_iterations=8, learning_rate=lr, seed=1,
                max_iterations=R + 4, trace=trace,
                sm_budget=0)
connect(eng, world, rank, nccl=False)  # peer-memory exchange only (gloo group)
p0 = eng.params()
eng.run(R)
torch.cuda.synchronize()
rec = eng.records()
flat = lambda ps: np.concatenate([np.concatenate([w.ravel(), b]) for w, b in ps])
out = dict(sizes=rec["sizes"], v_obs=rec["v_obs"], v_pred=rec["v_pred"], loss=rec["loss"],
           params=flat(eng.params()), p0=flat(p0), trace_c=trace[0], trace_m=trace[1],
           dims=np.asarray(dims), n_local=n_local, world=world, B=B, lr=lr, rounds=R)
if rank == 0:
    x, y = eng.dataset()
    out.update(x=x, y=y)
os.makedirs(a.out, exist_ok=True)
np.savez(os.path.join(a.out, f"rank{rank}.npz"), **out)
dist.barrier()
del eng
dist.destroy_process_group()
print(f"rank {rank}: {R} rounds, last sizes {rec['sizes'][-1].tolist()}", flush=True)
