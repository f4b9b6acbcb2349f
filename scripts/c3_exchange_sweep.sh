#!/bin/bash
# C3 at N GPUs (one worker per GPU): the gradient-bucket exchange variants
# against the backward GEMMs -- NCCL buckets with the default / capped CTA
# count, copy-engine one-shot and two-shot pushes.
N=$(python -c "import torch; print(torch.cuda.device_count())")
O=${OUT:-gpurun_out/c3x}_n$N; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
run() { name=$1; shift; env "$@" timeout 600 $TR --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N --config c3 --steps 20 --warmup 5 > $O/$name.json 2> $O/$name.err; echo "$name rc=$?" >> $O/status; }
run nccl_default X=1
run nccl_ctas8 NCCL_MAX_CTAS=8
run nccl_ctas4 NCCL_MAX_CTAS=4
run nccl_ctas16 NCCL_MAX_CTAS=16
run ce_one_shot LBBSP_CE_BUCKETS=1
run ce_two_shot LBBSP_CE_BUCKETS=1 LBBSP_CE_TWO_SHOT=1
cat $O/status
