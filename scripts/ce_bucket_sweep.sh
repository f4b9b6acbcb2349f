# one worker per GPU at N GPUs: parity of the copy-engine bucket exchange, then
# C3 and C5 with it (default) and with NCCL buckets (LBBSP_NCCL_BUCKETS=1)
N=${N:-2}
mkdir -p gpurun_out/ce
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port"
timeout 300 $T 29611 tests/mp_bucket_check.py > gpurun_out/ce/check_n$N.log 2>&1; echo check rc=$?
grep "rank " gpurun_out/ce/check_n$N.log
for mode in ce nccl; do
  if [ $mode = nccl ]; then export LBBSP_NCCL_BUCKETS=1; else unset LBBSP_NCCL_BUCKETS; fi
  timeout 300 $T 29621 bench.py --gpus $N --config c3 --steps 100 --warmup 10 > gpurun_out/ce/c3_${mode}_n$N.json 2> gpurun_out/ce/c3_${mode}_n$N.err; echo c3 $mode rc=$?
  timeout 300 $T 29631 bench.py --gpus $N --config c5 --steps 300 --warmup 0 > gpurun_out/ce/c5_${mode}_n$N.json 2> gpurun_out/ce/c5_${mode}_n$N.err; echo c5 $mode rc=$?
done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/ce/c*_n*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    if "schemes" in d:
        print(f, {k:round(v["ms_per_round"],3) for k,v in d["schemes"].items()}, "lb/bsp", round(d["lbbsp_over_bsp_speedup"],3))
    else:
        print(f, "lbbsp", round(d["ms_per_step"],3), "bsp", round(d["bsp"]["ms_per_step"],3), "ideal", round(d["ideal_no_straggler"]["ms_per_step"],3), d["lbbsp"]["sizes_last"], "roofline", round(d["roofline"]["achieved"]), "e2e" , d.get("e2e",{}).get("value"))
P
