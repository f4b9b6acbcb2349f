"""Probe (2+ GPUs, torchrun): NVLink traffic of the gradient exchange, read
from the NVML hardware throughput counters (NVML_FI_DEV_NVLINK_THROUGHPUT_
DATA_TX/RX, KiB, summed over links) around a timed window of rounds.
  MODE=c3: one worker per GPU, MLP 4 x 4096^2, copy-engine bf16 buckets
  MODE=c2: 8 workers per GPU, MLP 784-256-10, peer-memory kernels
Prints per rank: rounds, ms/round, NVLink TX/RX bytes per round, the
algorithmic exchange bytes per round and the achieved bus GB/s."""
import os, sys, json
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
import torch.distributed as dist
import pynvml as nv
from paper_1806_02508_b200.mlp import MlpEngine, constant_trace

world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
# gloo for the host-side handshakes: no NCCL communicator in this process
# unless the exchange needs one (C3), so rank 0 can run under ncu
dist.init_process_group("gloo", init_method="env://")
mode = os.environ.get("MODE", "c3")
R = int(os.environ.get("ROUNDS", "50"))
if mode == "c3":
    dims, nl, B = [4096] * 5, 1, 2048 * world
else:
    dims, nl, B = [784, 256, 10], 8, 4096 * world
eng = MlpEngine(dims=dims, global_batch=B, n_workers_local=nl, world=world, rank=rank, predictor="ema",
                learning_rate=0.01, max_iterations=R + 20, trace=constant_trace(nl * world, R + 20))
if mode == "c3":
    uid = [MlpEngine.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    eng.init_comm(uid[0])
hs = [None] * world
dist.all_gather_object(hs, eng.peer_handle())
eng.init_peers(hs)
st = torch.cuda.ExternalStream(eng.stream)
eng.run(10)
torch.cuda.synchronize()
nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(local)
TX, RX = 138, 139  # NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX (KiB)
XB, RB = 202, 204  # NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES / _RCV_BYTES, per link (scope = link)
NL = 18            # NVLink 5 links per B200


def counters():
    """[tx, rx] bytes: the per-link byte counters summed over links when the
    driver serves them, else the throughput counters (KiB)"""
    ids = [(XB, l) for l in range(NL)] + [(RB, l) for l in range(NL)]
    try:
        vals = nv.nvmlDeviceGetFieldValues(h, ids)
        ok = [int(v.nvmlReturn) == 0 for v in vals]
        if rank == 0 and not getattr(counters, "said", False):
            print("per-link byte counters ok:", sum(ok), "of", len(ok), flush=True)
            counters.said = True
        if all(ok):
            tx = sum(int(v.value.ullVal) for v in vals[:NL])
            rx = sum(int(v.value.ullVal) for v in vals[NL:])
            return [tx, rx]
    except Exception as ex:  # noqa: BLE001
        if rank == 0:
            print("per-link counters unavailable:", ex, flush=True)
    vals = nv.nvmlDeviceGetFieldValues(h, [TX, RX])
    return [int(v.value.ullVal) * 1024 for v in vals]


def smi():
    import subprocess
    return subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", str(local)], capture_output=True,
                          text=True).stdout


dist.barrier()
smi0 = smi() if rank == 0 else ""
c0 = counters()
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record(st)
eng.run(R)
e.record(st)
e.synchronize()
c1 = counters()
if rank == 0:
    print("nvidia-smi nvlink -gt d before:\n" + smi0[:1500] + "\nafter:\n" + smi()[:1500], flush=True)
ms = s.elapsed_time(e) / R
P = sum(dims[l] * dims[l + 1] + dims[l + 1] for l in range(len(dims) - 1))
# algorithmic exchange per GPU per round (one direction): c3 one-shot push of
# the bf16 buckets to every peer; c2 fp32 gradient to every peer
alg = (world - 1) * P * (2 if mode == "c3" else 4)
tx = (c1[0] - c0[0]) / R
rx = (c1[1] - c0[1]) / R
out = dict(rank=rank, mode=mode, world=world, rounds=R, ms_per_round=ms, nvlink_tx_bytes_per_round=tx,
           nvlink_rx_bytes_per_round=rx, algorithmic_tx_bytes_per_round=alg,
           tx_over_algorithmic=tx / alg if alg else None,
           tx_gbs_over_round=tx / (ms * 1e-3) / 1e9)
print(json.dumps(out), flush=True)
dist.barrier()
dist.destroy_process_group()
