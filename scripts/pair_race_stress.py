"""Stress (GPU): the fused pair worker kernel under injected interference with
static ragged sizes -- two runs of the same inputs must end bitwise equal
(a race between the TMA ring, the phase-W prefetch and the DSMEM exchange
would show up as a mismatch); each run is also compared with the separate
kernels (LBBSP_NO_FUSE) within the split-sum bar."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
from paper_1806_02508_b200.mlp import MlpEngine, benchmark_trace

R = int(os.environ.get("ROUNDS", "120"))
rng = np.random.default_rng(int(os.environ.get("SEED", "5")))


def sizes_case(i):
    if i == 0:
        return [1, 1, 2, 3, 1000, 1030, 1029, 1030]
    if i == 1:
        return [3000, 200, 200, 200, 200, 200, 48, 48]
    w = rng.dirichlet(np.full(8, 0.4))
    s = np.maximum(1, np.floor(w * 4096)).astype(int)
    s[np.argmax(s)] += 4096 - s.sum()
    return s.tolist()


def run(static, env=None, predictor="ema"):
    saved = {}
    for k, v in (env or {}).items():
        saved[k] = os.environ.get(k)
        os.environ[k] = v
    try:
        eng = MlpEngine(dims=[784, 256, 10], global_batch=4096, n_workers_local=8, predictor=predictor,
                        learning_rate=0.05, seed=3, max_iterations=R + 2,
                        trace=benchmark_trace(8, R + 2, seed=3), static_sizes=static)
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    flat = lambda ps: np.concatenate([np.concatenate([w.ravel(), b]) for w, b in ps])
    p0 = flat(eng.params())
    eng.run(R)
    p = flat(eng.params())
    loss = eng.records()["loss"][:R].copy()
    del eng
    return p0, p, loss


bad = 0
for i in range(int(os.environ.get("CASES", "6"))):
    st = sizes_case(i)
    p0, a, la = run(st)
    _, b, lb = run(st)
    _, c, _ = run(st, {"LBBSP_NO_FUSE": "1"})
    upd = float(np.max(np.abs(c - p0)))
    same = np.array_equal(a, b) and np.array_equal(la, lb)
    dev = float(np.max(np.abs(a - c))) / upd
    first = int(np.argmax(la != lb)) if not np.array_equal(la, lb) else -1
    print(f"case {i} sizes {st}: pair run-to-run bitwise {same} (first differing loss round {first}), "
          f"pair vs separate {dev:.2e} of the update", flush=True)
    bad += not same
# dynamic LB-BSP sizes from the Perfect predictor (deterministic) through the
# plan fast path, the gather and the pair kernel
for rep in range(int(os.environ.get("DYN", "3"))):
    _, a, la = run(None, predictor="perfect")
    _, b, lb = run(None, predictor="perfect")
    same = np.array_equal(a, b) and np.array_equal(la, lb)
    first = int(np.argmax(la != lb)) if not np.array_equal(la, lb) else -1
    print(f"dynamic rep {rep}: run-to-run bitwise {same} (first differing loss round {first})", flush=True)
    bad += not same
print("FAIL" if bad else "OK", bad)
