"""Probe (GPU): multi-round weight drift of the MLP engine against the
bf16-aware restatement iterated with the device's sizes. Prints, per
checkpoint, the teacher-forced one-round update error and the free-running
trajectory error, to size the bounds of tests/test_gpu_parity_rounds.py."""
import sys, os, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
from oracle import mlp_oracle as MO
from oracle import oracle as O
from paper_1806_02508_b200.mlp import MlpEngine, benchmark_trace, constant_trace

orc = O.restatement()


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def run(name, dims, B, n, rounds, predictor, trace, lr, seed=1, every=1):
    eng = MlpEngine(dims=dims, global_batch=B, n_workers_local=n, predictor=predictor,
                    warmup_iterations=50, learning_rate=lr, seed=seed, max_iterations=rounds + 2,
                    trace=trace)
    x, y = eng.dataset()
    p0 = eng.params()
    porc = [(W.astype(np.float64), b.astype(np.float64)) for W, b in p0]
    prev = p0
    t0 = time.time()
    worst_tf = 0.0
    for k in range(rounds):
        eng.run(1)
        rec = eng.records()
        sizes = rec["sizes"][k].tolist()
        stream = orc.sample_stream(seed, k, B, 1000)
        cur = eng.params()
        if k % every == 0:
            exp, _ = MO.lbbsp_round_bf16(prev, x, y, stream, sizes, lr)
            e = max(rel(W1.astype(np.float64) - W0, We - W0) for (W0, _), (W1, _), (We, _) in zip(prev, cur, exp))
            worst_tf = max(worst_tf, e)
        # free-running oracle (fp64 master weights) with the device sizes
        porc, _ = MO.lbbsp_round_bf16([(W.astype(np.float32), b.astype(np.float32)) for W, b in porc],
                                      x, y, stream, sizes, lr)
        if (k + 1) % 10 == 0 or k == rounds - 1:
            tr = max(rel(W1.astype(np.float64) - W0, Wo - W0) for (W0, _), (W1, _), (Wo, _) in zip(p0, cur, porc))
            tb = max(rel(b1.astype(np.float64) - b0, bo - b0) for (_, b0), (_, b1), (_, bo) in zip(p0, cur, porc))
            lo = MO.full_loss(cur, x, y)
            print(f"{name} k={k+1} teacher-forced worst={worst_tf:.3e} traj W={tr:.3e} b={tb:.3e} "
                  f"loss dev={rec['loss'][k]:.6f} orc(dev params)={lo:.6f} t={time.time()-t0:.1f}s", flush=True)
        prev = cur
    del eng


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("all", "c2"):
        run("C2-narx", [784, 256, 10], 4096, 8, 110, "narx", benchmark_trace(8, 112, seed=3), 0.05)
    if which in ("all", "c2ema"):
        run("C2-ema-lr.1", [784, 256, 10], 4096, 8, 60, "ema", benchmark_trace(8, 62, seed=3), 0.1)
    if which in ("all", "c3"):
        run("C3", [4096] * 5, 2048, 1, 10, "ema", constant_trace(1, 12), 0.01)
