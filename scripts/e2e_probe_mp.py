"""Per-step e2e times (H2D + round + D2H) on a multi-GPU C2 run (debug helper)."""
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
eng = MlpEngine(dims=[784, 256, 10], global_batch=4096 * world, n_workers_local=8, world=world, rank=rank,
                predictor="narx", warmup_iterations=50, max_iterations=300, trace=benchmark_trace(n, 300, seed=3),
                learning_rate=0.05)
uid = [MlpEngine.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(uid, src=0)
eng.init_comm(uid[0])
if not os.environ.get("LBBSP_NO_PEERS"):
    hs = [None] * world
    dist.all_gather_object(hs, eng.peer_handle())
    eng.init_peers(hs)
x, y = eng.dataset()
xb = torch.empty(x.shape, dtype=torch.bfloat16, pin_memory=True); xb.copy_(torch.from_numpy(x).to(torch.bfloat16))
yb = torch.empty(y.shape, dtype=torch.int32, pin_memory=True); yb.copy_(torch.from_numpy(y.astype(np.int32)))
osz = torch.zeros(n, dtype=torch.int32, pin_memory=True); ol = torch.zeros(1, dtype=torch.float64, pin_memory=True)
st = torch.cuda.ExternalStream(eng.stream)
eng.run(60)
torch.cuda.synchronize(); dist.barrier()
evs = [torch.cuda.Event(enable_timing=True) for _ in range(101)]
with torch.cuda.stream(st):
    evs[0].record(st)
for i in range(100):
    eng.load_data_async(xb.data_ptr(), yb.data_ptr())
    eng.run(1)
    eng.read_result_async(osz.data_ptr(), ol.data_ptr())
    with torch.cuda.stream(st):
        evs[i + 1].record(st)
evs[-1].synchronize()
t = np.array([evs[i].elapsed_time(evs[i + 1]) * 1e3 for i in range(100)])
print(f"rank {rank}: e2e per step us: mean {t.mean():.1f} median {np.median(t):.1f} max {t.max():.1f} "
      f"p90 {np.percentile(t, 90):.1f}; steps > 500us: {int((t > 500).sum())}", flush=True)
dist.destroy_process_group()
