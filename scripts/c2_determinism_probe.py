"""Probe (GPU): is the C2 engine's weight path deterministic? Two fresh engines
with the same static sizes (and optionally env toggles) are run round by
round; the first round whose weights differ bitwise is reported, plus the
teacher-forced error vs the bf16 restatement on every round."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
from oracle import mlp_oracle as MO
from oracle import oracle as O
from paper_1806_02508_b200.mlp import MlpEngine, benchmark_trace, constant_trace

orc = O.restatement()
R = int(os.environ.get("ROUNDS", "80"))
sizes_kind = os.environ.get("SIZES", "ragged")
n, B = 8, 4096
if sizes_kind == "tiny":
    static = [1, 7, 1, 1, 1020, 1022, 1022, 1022]
elif sizes_kind == "equal":
    static = [512] * 8
else:
    static = [300, 700, 100, 900, 500, 600, 400, 596]


def flat(ps):
    return np.concatenate([np.concatenate([w.ravel(), b]) for w, b in ps])


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


engs = [MlpEngine(dims=[784, 256, 10], global_batch=B, n_workers_local=n, predictor="narx",
                  warmup_iterations=50, learning_rate=0.05, seed=1, max_iterations=R + 2,
                  trace=benchmark_trace(n, R + 2, seed=3), static_sizes=static) for _ in range(2)]
x, y = engs[0].dataset()
prev = engs[0].params()
first_div = None
worst = []
for k in range(R):
    for e in engs:
        e.run(1)
    p = [e.params() for e in engs]
    if first_div is None and not np.array_equal(flat(p[0]), flat(p[1])):
        first_div = k
        d = np.abs(flat(p[0]) - flat(p[1]))
        print(f"first divergence at round {k}: max diff {d.max():.3e}, n diff {int((d > 0).sum())}", flush=True)
    stream = orc.sample_stream(1, k, B, 1000)
    exp, _ = MO.lbbsp_round_bf16(prev, x, y, stream, static, 0.05)
    errs = [(rel(W1.astype(np.float64) - W0, We - W0), rel(b1.astype(np.float64) - b0, be - b0))
            for (W0, b0), (W1, b1), (We, be) in zip(prev, p[0], exp)]
    e2 = [(rel(W1.astype(np.float64) - W0, We - W0), rel(b1.astype(np.float64) - b0, be - b0))
          for (W0, b0), (W1, b1), (We, be) in zip(prev, p[1], exp)]
    worst.append((max(max(a) for a in errs), k, errs, e2))
    prev = p[0]
worst.sort(key=lambda t: -t[0])
print(f"sizes={sizes_kind} env NO_PDL={os.environ.get('LBBSP_NO_PDL')} NO_FORK={os.environ.get('LBBSP_NO_FORK')} "
      f"first_div={first_div}", flush=True)
for w in worst[:6]:
    print(f"  k={w[1]} eng0 {[(round(a, 7), round(b, 7)) for a, b in w[2]]} eng1 {[(round(a, 7), round(b, 7)) for a, b in w[3]]}")
