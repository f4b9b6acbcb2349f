"""Multi-GPU check (run with torchrun on >= 2 GPUs), one worker per GPU: the
copy-engine bucket exchange (bf16 layer buckets pushed into the peers' IPC
slots, rank-ordered fp32 sum + apply; one-shot, and the reduce-scatter +
all-gather of bf16-rounded slice sums) gives the same parameters on every rank
and matches the NCCL bf16 bucket all-reduce (LBBSP_NCCL_BUCKETS=1) within the
bf16 rounding of the summed gradient, after several rounds with static sizes
(the exchange step of the sharded path)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
import torch.distributed as dist
from paper_1806_02508_b200.mlp import MlpEngine, constant_trace

world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", local))
dims = [1024, 1024, 1024, 1024]
rounds = 12
out = {}
os.environ["LBBSP_CE_BUCKETS"] = "1"  # the copy-engine path also at N > 2 (default: NCCL there)
for mode in ("nccl", "ce", "ce_two_shot"):
    os.environ.pop("LBBSP_NCCL_BUCKETS", None)
    os.environ.pop("LBBSP_CE_TWO_SHOT", None)
    if mode == "nccl":
        os.environ["LBBSP_NCCL_BUCKETS"] = "1"
    elif mode == "ce_two_shot":
        os.environ["LBBSP_CE_TWO_SHOT"] = "1"
    sizes = [1024 + 256 * (i % 2) - 128 for i in range(world)]  # ragged per-GPU batches
    eng = MlpEngine(dims=dims, global_batch=sum(sizes), n_workers_local=1, world=world, rank=rank,
                    scheme="lb-bsp", predictor="ema", learning_rate=0.05, max_iterations=rounds + 4,
                    trace=constant_trace(world, rounds + 4), static_sizes=sizes)
    uid = [MlpEngine.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    eng.init_comm(uid[0])
    hs = [None] * world
    dist.all_gather_object(hs, eng.peer_handle())
    eng.init_peers(hs)
    eng.run(rounds)
    torch.cuda.synchronize()
    flat = np.concatenate([np.concatenate([w.ravel(), b]) for w, b in eng.params()])
    out[mode] = (flat, eng.records()["loss"][:rounds])
    del eng
p0, l0 = out["nccl"]
p1, l1 = out["ce"]
# every rank holds bitwise the same parameters on the copy-engine path
allp = [None] * world
dist.all_gather_object(allp, p1)
same = all(np.array_equal(allp[0], a) for a in allp)
diff = float(np.max(np.abs(p0 - p1)))
moved = float(np.max(np.abs(p0 - allp[0]))) if rank else 0.0
ldiff = float(np.max(np.abs(l0 - l1) / np.maximum(1e-12, np.abs(l0))))
print(f"rank {rank}: ranks bitwise equal {same}, max |params nccl - ce| = {diff:.3e} "
      f"(max |p| {float(np.max(np.abs(p0))):.3e}), max rel loss diff {ldiff:.3e}", flush=True)
assert same
# two-shot (reduce-scatter + all-gather of the bf16-rounded slice sums):
# bitwise equal on every rank, within the bf16 rounding of the NCCL path
p2 = out["ce_two_shot"][0]
allp2 = [None] * world
dist.all_gather_object(allp2, p2)
same2 = all(np.array_equal(allp2[0], a) for a in allp2)
diff2 = float(np.max(np.abs(p0 - p2)))
print(f"rank {rank}: two-shot ranks bitwise equal {same2}, max |params nccl - two-shot| = {diff2:.3e}",
      flush=True)
assert same2
assert diff2 <= 2e-3 * max(1.0, float(np.max(np.abs(p0)))), diff2
assert diff <= 2e-3 * max(1.0, float(np.max(np.abs(p0)))), diff  # bf16 rounding of the bucket sum
assert ldiff <= 1e-2, ldiff
dist.destroy_process_group()
