"""Device timeline of a steady-state multi-GPU C2 round, rank 0 (debug helper).
torchrun --nproc-per-node N scripts/c2_timeline_mp.py"""
import os, sys, ctypes as C
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
import torch.distributed as dist
from paper_1806_02508_b200.mlp import MlpEngine, benchmark_trace, constant_trace, connect
from paper_1806_02508_b200._lib import lib
world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", local))
n = 8 * world
for pred in ("narx", "ema"):
    eng = MlpEngine(dims=[784, 256, 10], global_batch=4096 * world, n_workers_local=8, world=world, rank=rank,
                    predictor=pred, warmup_iterations=50, max_iterations=300,
                    trace=constant_trace(n, 300) if os.environ.get("TRACE") == "const" else benchmark_trace(n, 300, seed=3))
    connect(eng, world, rank, peers=not os.environ.get("LBBSP_NO_PEERS"))
    st = torch.cuda.ExternalStream(eng.stream)
    eng.run(100)
    for rep in range(5):
        torch.cuda.synchronize(); dist.barrier()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            s.record(st)
        eng.run(1)
        with torch.cuda.stream(st):
            e.record(st)
        e.synchronize()
        buf = np.zeros(16 + 2 * 28 * 8, np.uint64); nph = C.c_int()
        lib().lbbsp_mlp_debug_timeline(C.c_void_p(eng._h.value if hasattr(eng._h, "value") else eng._h),
                                       buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), C.byref(nph))
        if rank == 0:
            t0 = int(buf[0])
            names = ["plan_in", "plan_ready", "gather_in", "obs_in", "obs_out", "reduce_in", "losshead_in", "losshead_out",
                     "plan_computed", "gather_out", "pred_done", "solve_or_dry_done", "slices_done", "train_out", "train_in",
                     "obs_kernel_in"]
            stt = {k: round((int(buf[i]) - t0) / 1e3, 1) for i, k in enumerate(names) if buf[i] not in (0, 2**64 - 1)}
            tim = buf[16:16 + 2 * nph.value * 8].astype(np.int64).reshape(nph.value, 8, 2)
            ph = [(round((tim[p, :, 0].min() - t0) / 1e3, 1), round((tim[p, :, 1].max() - t0) / 1e3, 1)) for p in range(nph.value)]
            print(f"{pred} round {s.elapsed_time(e)*1e3:.1f} us stamps {stt} phases {ph}", flush=True)
    del eng
dist.destroy_process_group()
