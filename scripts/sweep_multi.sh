#!/bin/bash
# Multi-GPU measurement sweep on one box: bench.py at N=2 and N=4 for the
# configs given as arguments (default c2), our arm then the reference arm.
O=gpurun_out/sweep; mkdir -p $O
CFGS=${@:-c2}
for C in $CFGS; do
  for N in 2 4; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29500 + N)) bench.py --gpus $N --config $C > $O/${C}_n$N.json 2> $O/${C}_n$N.err
    echo "$C n$N rc=$?" >> $O/status_multi
  done
done
[ -n "$NO_REF" ] || for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29600 + N)) bench.py --gpus $N --impl reference > $O/ref_n$N.json 2> $O/ref_n$N.err
  echo "ref n$N rc=$?" >> $O/status_multi
done
cat $O/status_multi
