"""Multi-GPU check (run with torchrun on >= 2 GPUs), one worker per GPU: the
copy-engine bucket exchange (bf16 layer buckets pushed into the peers' IPC
slots, rank-ordered fp32 sum + apply; one-shot, and the reduce-scatter +
all-gather of bf16-rounded slice sums) against the NCCL bf16 bucket
all-reduce (LBBSP_NCCL_BUCKETS=1), after several rounds with static sizes.

Bars: every variant leaves bitwise-equal weights on every rank;
a second copy-engine run is bitwise equal to the first (determinism); the
variants differ from NCCL by at most 1% of the weights' total update
max|p_N - p_0| (the bf16 rounding of the summed buckets differs by order of
summation; a stale or dropped bucket moves the update by ~1/world)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
import torch.distributed as dist
from paper_1806_02508_b200.mlp import MlpEngine, connect, constant_trace

world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", local))
dims = [1024, 1024, 1024, 1024]
rounds = 12
out = {}
os.environ["LBBSP_CE_BUCKETS"] = "1"  # the copy-engine path also at N > 2 (default: NCCL there)
flat = lambda ps: np.concatenate([np.concatenate([w.ravel(), b]) for w, b in ps])
p_init = None
for mode in ("nccl", "ce", "ce_again", "ce_two_shot"):
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
    if p_init is None:
        p_init = flat(eng.params())
    connect(eng, world, rank)
    eng.run(rounds)
    torch.cuda.synchronize()
    out[mode] = (flat(eng.params()), eng.records()["loss"][:rounds])
    del eng
upd = float(np.max(np.abs(out["nccl"][0] - p_init)))
for mode in ("ce", "ce_two_shot"):
    p = out[mode][0]
    allp = [None] * world
    dist.all_gather_object(allp, p)
    same = all(np.array_equal(allp[0], a) for a in allp)
    diff = float(np.max(np.abs(out["nccl"][0] - p)))
    print(f"rank {rank}: {mode}: ranks bitwise equal {same}, max |p_nccl - p| = {diff:.3e} "
          f"({diff / upd:.2e} of the update {upd:.3e})", flush=True)
    assert same, mode
    assert diff <= 1e-2 * upd, (mode, diff, upd)
assert np.array_equal(out["ce"][0], out["ce_again"][0]), "copy-engine exchange is not deterministic"
ldiff = float(np.max(np.abs(out["nccl"][1] - out["ce"][1]) / np.maximum(1e-12, np.abs(out["nccl"][1]))))
assert ldiff <= 1e-3, ldiff
dist.destroy_process_group()
