# final multi-GPU pass (4-GPU box): exchange parity checks at N=2/4, then C3
# and C5 bench lines at N=2/4 with the default exchange
mkdir -p gpurun_out/final
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do
  timeout 300 $T --nproc-per-node $N --master-port $((29700+N)) tests/mp_bucket_check.py > gpurun_out/final/bucket_check_n$N.log 2>&1; echo bucket_check n$N rc=$?
  timeout 300 $T --nproc-per-node $N --master-port $((29710+N)) tests/mp_peer_check.py > gpurun_out/final/peer_check_n$N.log 2>&1; echo peer_check n$N rc=$?
done
grep -h "rank 0" gpurun_out/final/*_check_n*.log
rm -f gpurun_out/sweep/status_multi
NO_REF=1 bash scripts/sweep_multi.sh c3 c5
