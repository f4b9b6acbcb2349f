#!/bin/bash
# Round-2 multi-GPU sweep on one box (N = number of visible GPUs): C2/C3/C5
# bench lines, NVLink counters of the exchanges, the multi-rank tests.
N=$(python -c "import torch; print(torch.cuda.device_count())")
O=gpurun_out/r02_n$N; mkdir -p $O
st() { echo "$1 rc=$2" >> $O/status; }
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29561"
timeout 900 $TR bench.py --gpus $N --steps 20 --warmup 5 > $O/c2.json 2> $O/c2.err; st c2 $?
timeout 900 $TR bench.py --gpus $N --config c3 --steps 20 --warmup 5 > $O/c3.json 2> $O/c3.err; st c3 $?
timeout 1200 $TR bench.py --gpus $N --config c5 --steps 300 > $O/c5.json 2> $O/c5.err; st c5 $?
MODE=c3 timeout 600 $TR scripts/nvlink_probe.py > $O/nvlink_c3.log 2>&1; st nvl_c3 $?
MODE=c2 timeout 600 $TR scripts/nvlink_probe.py > $O/nvlink_c2.log 2>&1; st nvl_c2 $?
LBBSP_NCCL_BUCKETS=1 MODE=c3 timeout 600 $TR scripts/nvlink_probe.py > $O/nvlink_c3_nccl.log 2>&1; st nvl_c3_nccl $?
timeout 900 python -m pytest tests/test_gpu_multi.py -q -rA > $O/multi_tests.log 2>&1; st multi $?
cat $O/status
