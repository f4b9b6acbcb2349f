"""C5 records per round (caps, sizes, measured speeds) for BSP and LB-BSP (debug helper)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
import torch.distributed as dist
from paper_1806_02508_b200.mlp import MlpEngine, benchmark_trace
world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", local))
iters, period = 130, 100
raw = benchmark_trace(world, iters + period, seed=3)
trace = tuple(np.stack([a[i, (i * period) // world:(i * period) // world + iters] for i in range(world)]) for a in raw)
for scheme in ("bsp", "lb-bsp"):
    eng = MlpEngine(dims=[4096] * 5, global_batch=2048 * world, n_workers_local=1, world=world, rank=rank,
                    scheme=scheme, predictor="narx", warmup_iterations=50, max_iterations=iters, trace=trace,
                    learning_rate=0.01)
    uid = [MlpEngine.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    eng.init_comm(uid[0])
    st = torch.cuda.ExternalStream(eng.stream)
    eng.run(2)
    torch.cuda.synchronize(); dist.barrier()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(121)]
    with torch.cuda.stream(st):
        evs[0].record(st)
    for i in range(120):
        eng.run(1)
        with torch.cuda.stream(st):
            evs[i + 1].record(st)
    evs[-1].synchronize()
    t = [evs[i].elapsed_time(evs[i + 1]) for i in range(120)]
    rec = eng.records()
    if rank == 0:
        for r in (10, 30, 60, 80, 100, 115):
            print(f"{scheme} round {r+2}: {t[r]*1e3:.0f} us caps {rec['caps'][r+2].tolist()} sizes {rec['sizes'][r+2].tolist()} "
                  f"v_obs {np.round(rec['v_obs'][r+2]).tolist()} avail {[round(float(min(1, trace[0][i][r+2]*trace[2][i][r+2])),2) for i in range(world)]}", flush=True)
    del eng
dist.destroy_process_group()
