"""Per-rank device timeline of a steady-state C3 round (one worker per GPU,
last GPU at half its SMs) for LB-BSP and BSP (debug helper)."""
import os, sys, ctypes as C
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
import torch.distributed as dist
from paper_1806_02508_b200.mlp import MlpEngine, constant_trace
from paper_1806_02508_b200._lib import lib
world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", local))
avail = [1.0] * world
avail[-1] = 0.5
for scheme in ("lb-bsp", "bsp"):
    eng = MlpEngine(dims=[4096] * 5, global_batch=2048 * world, n_workers_local=1, world=world, rank=rank,
                    scheme=scheme, predictor="ema", max_iterations=100, trace=constant_trace(world, 100, avail),
                    learning_rate=0.01)
    uid = [MlpEngine.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    eng.init_comm(uid[0])
    st = torch.cuda.ExternalStream(eng.stream)
    eng.run(30)
    torch.cuda.synchronize(); dist.barrier()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        s.record(st)
    eng.run(1)
    with torch.cuda.stream(st):
        e.record(st)
    e.synchronize()
    buf = np.zeros(16 + 2 * 28, np.uint64); nph = C.c_int()
    lib().lbbsp_mlp_debug_timeline(C.c_void_p(eng._h.value if hasattr(eng._h, "value") else eng._h),
                                   buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), C.byref(nph))
    t0 = int(buf[0])
    names = ["plan_in", "plan_out", "gather_in", "obs_in", "obs_out", "reduce_in", "losshead_in", "losshead_out"]
    stt = {k: round((int(buf[i]) - t0) / 1e3, 1) for i, k in enumerate(names) if buf[i] not in (0, 2**64 - 1)}
    tim = buf[16:16 + 2 * nph.value].astype(np.int64).reshape(nph.value, 2)
    ph = [(round((a - t0) / 1e3), round((b - t0) / 1e3)) for a, b in tim]
    rec = eng.records()
    for r in range(world):
        if r == rank:
            print(f"{scheme} rank {rank}: round {s.elapsed_time(e)*1e3:.0f} us sizes {rec['sizes'][-1].tolist()} stamps {stt}\n   phases {ph}", flush=True)
        dist.barrier()
    del eng
dist.destroy_process_group()
