"""Per-round device time distribution, LB-BSP vs BSP, multi-GPU C2 (debug helper)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
import torch.distributed as dist
from paper_1806_02508_b200.mlp import MlpEngine, benchmark_trace
world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", local))
n = 8 * world
for scheme in ("lb-bsp", "bsp"):
    for pred in ("narx", "ema"):
        eng = MlpEngine(dims=[784, 256, 10], global_batch=4096 * world, n_workers_local=8, world=world, rank=rank,
                        scheme=scheme, predictor=pred, warmup_iterations=50, max_iterations=300,
                        trace=benchmark_trace(n, 300, seed=3), learning_rate=0.05)
        uid = [MlpEngine.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        eng.init_comm(uid[0])
        hs = [None] * world
        dist.all_gather_object(hs, eng.peer_handle())
        eng.init_peers(hs)
        st = torch.cuda.ExternalStream(eng.stream)
        eng.run(60)
        torch.cuda.synchronize(); dist.barrier()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(101)]
        with torch.cuda.stream(st):
            evs[0].record(st)
        for i in range(100):
            eng.run(1)
            with torch.cuda.stream(st):
                evs[i + 1].record(st)
        evs[-1].synchronize()
        t = np.array([evs[i].elapsed_time(evs[i + 1]) * 1e3 for i in range(100)])
        rec = eng.records()
        sz = rec["sizes"][-1]
        if rank == 0:
            print(f"{scheme:6s} {pred}: mean {t.mean():.1f} median {np.median(t):.1f} p90 {np.percentile(t,90):.1f} max {t.max():.1f}  "
                  f"sizes per GPU {[int(sz[g*8:(g+1)*8].sum()) for g in range(world)]} caps {rec['caps'][-1].tolist()[:8]}", flush=True)
        del eng
dist.destroy_process_group()
