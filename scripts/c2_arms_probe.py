"""Probe (GPU): C2 round time of every allocation / predictor / observation
combination over the bench's 100-round window (rounds 100..199, benchmark
trace seed 3), timed like bench.py (events per round, L2 flushed between)."""
import json, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
from paper_1806_02508_b200.mlp import MlpEngine, benchmark_trace, calibrate_gamma, constant_trace

n, B, warm, window = 8, 4096, 100, 100
iters = warm + window + 8
trace = benchmark_trace(n, iters, seed=3)
prof = calibrate_gamma([784, 256, 10], B, n)
print("profiles", [(round(m * 1e9, 3), round(b * 1e6, 2), xo) for m, b, _, xo in prof], flush=True)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
out = {}
arms = [("bsp_narx", "bsp", "narx", "proportional", "rate", trace),
        ("bsp_ema", "bsp", "ema", "proportional", "rate", trace),
        ("lbbsp_narx_rate", "lb-bsp", "narx", "proportional", "rate", trace),
        ("lbbsp_narx_capacity", "lb-bsp", "narx", "proportional", "capacity", trace),
        ("lbbsp_ema_rate", "lb-bsp", "ema", "proportional", "rate", trace),
        ("lbbsp_ema_capacity", "lb-bsp", "ema", "proportional", "capacity", trace),
        ("lbbsp_narx_gamma", "lb-bsp", "narx", "gamma", "rate", trace),
        ("lbbsp_ema_gamma", "lb-bsp", "ema", "gamma", "rate", trace),
        ("perfect", "lb-bsp", "perfect", "proportional", "rate", trace),
        ("perfect_gamma", "lb-bsp", "perfect", "gamma", "rate", trace),
        ("nostrag_narx", "lb-bsp", "narx", "proportional", "rate", constant_trace(n, iters)),
        ("nostrag_ema", "lb-bsp", "ema", "proportional", "rate", constant_trace(n, iters))]
only = os.environ.get("ARMS")
for name, scheme, pred, solver, obs, tr in arms:
    if only and name not in only.split(","):
        continue
    eng = MlpEngine(dims=[784, 256, 10], global_batch=B, n_workers_local=n, scheme=scheme, predictor=pred,
                    warmup_iterations=50, learning_rate=0.05, seed=1, max_iterations=iters + 4, trace=tr,
                    solver=solver, observe=obs,
                    gamma_profiles=prof if (solver == "gamma" or obs == "capacity") else None)
    st = torch.cuda.ExternalStream(eng.stream)
    eng.run(warm)
    torch.cuda.synchronize()
    ev = []
    for _ in range(window):
        with torch.cuda.stream(st):
            flush.zero_()
            s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
            s.record(st)
        eng.run(1)
        with torch.cuda.stream(st):
            e.record(st)
        ev.append((s, e))
    torch.cuda.synchronize()
    ms = np.array([s.elapsed_time(e) for s, e in ev]) * 1e3
    rec = eng.records()
    sz = rec["sizes"][warm:warm + window]
    tw = rec["t_worker"][warm:warm + window] * 1e6
    out[name] = dict(mean=float(ms.mean()), median=float(np.median(ms)), p90=float(np.percentile(ms, 90)),
                     min_batch=int(sz.min()), max_batch=int(sz.max()),
                     crit_worker_us=float(tw.max(axis=1).mean()),
                     mean_worker_us=float(tw.mean()))
    print(name, json.dumps({k: round(v, 2) if isinstance(v, float) else v for k, v in out[name].items()}), flush=True)
    if os.environ.get("DUMP"):
        np.savez(f"gpurun_out/arms_{name}.npz", ms=ms, sizes=sz, t=tw, v_obs=rec["v_obs"][warm:warm + window],
                 v_pred=rec["v_pred"][warm:warm + window])
    del eng
json.dump(out, open("gpurun_out/c2_arms.json", "w"), indent=1)
