"""C5 diagnostic (torchrun, N GPUs): per-round sizes, SM caps, measured
worker times and observed/predicted speeds of every worker for BSP and
LB-BSP on the C5 trace, gathered to rank 0 and written to
gpurun_out/c5_diag_<scheme>.npz. Not a bench number."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1806_02508_b200.mlp import MlpEngine, benchmark_trace  # noqa: E402


def main():
    world, rank, local = bench.dist_env()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", local))
    rounds = int(os.environ.get("ROUNDS", "150"))
    dims = [4096] * 5
    B = 2048 * world
    iters = rounds + 8
    period = 100
    raw = benchmark_trace(world, iters + period, seed=bench.TRACE_SEED)
    trace = tuple(np.stack([a[i, (i * period) // world:(i * period) // world + iters] for i in range(world)])
                  for a in raw)
    for scheme in ("bsp", "lb-bsp"):
        eng = MlpEngine(dims=dims, global_batch=B, n_workers_local=1, world=world, rank=rank,
                        scheme=scheme, predictor="narx", warmup_iterations=bench.WARMUP_NARX,
                        learning_rate=0.01, seed=1, max_iterations=iters, trace=trace,
                        sm_budget=bench.comm_sm_budget(world))
        uid = [MlpEngine.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        eng.init_comm(uid[0])
        st = torch.cuda.ExternalStream(eng.stream)
        times = []
        for _ in range(rounds):
            s = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            s.record(st)
            eng.run(1)
            e.record(st)
            e.synchronize()
            times.append(s.elapsed_time(e))
        rec = eng.records()
        mine = {k: (v[:, rank] if getattr(v, "ndim", 0) == 2 else v) for k, v in rec.items()
                if k in ("caps", "t_worker", "v_obs", "v_pred", "sizes")}
        mine["round_ms"] = np.array(times)
        allr = [None] * world
        dist.all_gather_object(allr, mine)
        if rank == 0:
            out = {k: np.stack([a[k] for a in allr], axis=1) for k in mine}
            out["trace_c"] = trace[0].T[:rounds]
            np.savez(f"gpurun_out/c5_diag_{scheme}.npz", **out)
            rt = out["round_ms"].max(axis=1)
            print(scheme, "mean round ms", rt.mean(), "median", np.median(rt), flush=True)
            for k in range(0, rounds, 5):
                print(k, "c", np.round(out["trace_c"][k], 2), "cap", out["caps"][k], "b", out["sizes"][k],
                      "t", np.round(out["t_worker"][k], 3), "round", np.round(out["round_ms"][k], 3), flush=True)
        del eng
        dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
