#!/bin/bash
# Round-2 multi-GPU sweep on one box (N = number of visible GPUs): C2/C3/C5
# bench lines, the reference arm, the multi-rank tests and exchange checks.
N=$(python -c "import torch; print(torch.cuda.device_count())")
O=${OUT:-gpurun_out/r02b}_n$N; mkdir -p $O
st() { echo "$1 rc=$2" >> $O/status; }
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 $TR --master-port 29561 bench.py --gpus $N --steps 20 --warmup 5 > $O/c2.json 2> $O/c2.err; st c2 $?
timeout 600 $TR --master-port 29562 bench.py --impl reference --gpus $N --steps 20 --warmup 5 > $O/ref.json 2> $O/ref.err; st ref $?
timeout 900 $TR --master-port 29563 bench.py --gpus $N --config c3 --steps 20 --warmup 5 > $O/c3.json 2> $O/c3.err; st c3 $?
timeout 1200 $TR --master-port 29564 bench.py --gpus $N --config c5 --steps 300 > $O/c5.json 2> $O/c5.err; st c5 $?
timeout 900 python -m pytest tests/test_gpu_multi.py -q -rA > $O/multi_tests.log 2>&1; st multi $?
for s in mp_bucket_check mp_peer_check; do
  timeout 300 $TR --master-port 2957$N tests/$s.py > $O/$s.log 2>&1; st $s $?
done
cat $O/status
