mkdir -p gpurun_out/c3var
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port"
timeout 120 $T 29521 scripts/allreduce_busbw.py > gpurun_out/c3var/busbw_n2.json 2> gpurun_out/c3var/busbw.err; echo busbw rc=$?
for cs in 0 8 16 32; do
  LBBSP_COMM_SMS=$cs timeout 300 $T $((29530+cs)) bench.py --gpus 2 --config c3 --steps 50 --warmup 10 > gpurun_out/c3var/c3_cs$cs.json 2> gpurun_out/c3var/c3_cs$cs.err; echo cs=$cs rc=$?
done
for cs in 0 16; do
  LBBSP_COMM_SMS=$cs timeout 300 $T $((29560+cs)) bench.py --gpus 2 --config c5 --steps 100 --warmup 0 > gpurun_out/c3var/c5_cs$cs.json 2> gpurun_out/c3var/c5_cs$cs.err; echo c5 cs=$cs rc=$?
done
cat gpurun_out/c3var/busbw_n2.json
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/c3var/c*_cs*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    if "schemes" in d:
        print(f, {k:round(v["ms_per_round"],3) for k,v in d["schemes"].items()})
    else:
        print(f, "lbbsp", round(d["ms_per_step"],3), "bsp", round(d["bsp"]["ms_per_step"],3), "ideal", round(d["ideal_no_straggler"]["ms_per_step"],3), d["lbbsp"]["worker_ms_last"], d["bsp"]["worker_ms_last"], d["ideal_no_straggler"]["worker_ms_last"])
P
