"""NVLink bus bandwidth of the C3/C5 gradient all-reduce (torchrun, N GPUs).

The engine's one-worker-per-GPU exchange is one bf16 ncclAllReduce per layer
bucket (W_l | b_l contiguous, 4096*4096 + 4096 elements) on the
comm stream, through the same libnccl.so.2 torch loads. This times exactly
those four buckets back to back, standalone, with CUDA events on the stream
they run on, max over ranks, and reports NCCL's bus bandwidth convention
busbw = 2(N-1)/N * bytes / t (SURVEY 8(d) "Allreduce"). One JSON line from
rank 0. Not a bench number.
"""
import json
import os

import torch
import torch.distributed as dist


def main():
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", local))
    width, layers = 4096, 4
    bucket = width * width + width
    bufs = [torch.randn(bucket, device="cuda", dtype=torch.bfloat16) for _ in range(layers)]
    one = torch.randn(bucket * layers, device="cuda", dtype=torch.bfloat16)
    res = {}
    for name, tensors in (("4_layer_buckets", bufs), ("one_flat_buffer", [one])):
        for _ in range(5):
            for t in tensors:
                dist.all_reduce(t)
        torch.cuda.synchronize()
        dist.barrier()
        iters = 20
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters):
            for t in tensors:
                dist.all_reduce(t)
        e.record()
        e.synchronize()
        ms = torch.tensor([s.elapsed_time(e) / iters], device="cuda", dtype=torch.float64)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        ms = float(ms.item())
        nbytes = sum(t.numel() for t in tensors) * 2
        res[name] = {"ms": ms, "bytes": nbytes, "algbw_GBps": nbytes / (ms * 1e-3) / 1e9,
                     "busbw_GBps": 2 * (world - 1) / world * nbytes / (ms * 1e-3) / 1e9}
    if rank == 0:
        print(json.dumps({"what": "bf16 ncclAllReduce of the C3 gradient (67,125,248 params)",
                          "n_gpus": world, "nccl": ".".join(map(str, torch.cuda.nccl.version())),
                          **res}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
