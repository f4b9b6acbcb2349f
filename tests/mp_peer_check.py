"""Multi-GPU check (run with torchrun on >= 2 GPUs): the NVLink peer exchange
(speeds all-gather + gradient all-reduce) gives the same parameters as the
NCCL path after several LB-BSP rounds with static sizes."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
import torch.distributed as dist
from paper_1806_02508_b200.mlp import MlpEngine, connect, constant_trace

world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", local))
n = 8 * world
out = {}
for mode in ("nccl", "peers"):
    eng = MlpEngine(dims=[784, 256, 10], global_batch=4096 * world, n_workers_local=8, world=world, rank=rank,
                    predictor="ema", max_iterations=40, trace=constant_trace(n, 40),
                    static_sizes=[4096 // 8] * n)
    connect(eng, world, rank, peers=mode == "peers")
    eng.run(20)
    torch.cuda.synchronize()
    flat = np.concatenate([np.concatenate([w.ravel(), b]) for w, b in eng.params()])
    out[mode] = (flat, eng.records()["loss"][:19])
    del eng
p0, l0 = out["nccl"]
p1, l1 = out["peers"]
diff = float(np.max(np.abs(p0 - p1)))
print(f"rank {rank}: max |params nccl - peers| = {diff:.3e}, losses equal: {np.array_equal(l0, l1)}", flush=True)
assert diff <= 1e-5 * max(1.0, float(np.max(np.abs(p0)))), diff
dist.destroy_process_group()
