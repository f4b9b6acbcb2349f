"""Probe: how many step halvings the NARX rotation's trainings take on the C2
bench workload. GPU part (MODE=gpu): run the engine (LB-BSP + NARX, capacity
observation, benchmark trace) for 200 rounds and dump the observed speeds and
the trace. CPU part (MODE=cpu): replay train_rotation on those histories with
a restatement of narx_train_online (predictor.cpp:155-196) that counts
evaluations, epochs and halvings per training."""
import os, sys, json
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np

OUT = "gpurun_out/narx_hist.npz"
if os.environ.get("MODE", "gpu") == "gpu":
    from paper_1806_02508_b200.mlp import MlpEngine, benchmark_trace, calibrate_gamma
    n, R = 8, 200
    tr = benchmark_trace(n, R + 4, seed=3)
    prof = calibrate_gamma([784, 256, 10], 4096, n)
    eng = MlpEngine(dims=[784, 256, 10], global_batch=4096, n_workers_local=n, predictor="narx",
                    warmup_iterations=50, max_iterations=R + 4, trace=tr, observe="capacity",
                    gamma_profiles=prof)
    eng.run(R)
    rec = eng.records()
    np.savez(OUT, v=rec["v_obs"], c=tr[0][:, :R].T, m=tr[1][:, :R].T)
    print("saved", rec["v_obs"].shape)
    sys.exit(0)

d = np.load(OUT)
V, Cc, Mm = d["v"], d["c"], d["m"]  # [rounds][n]
R, n = V.shape


def scaler(x):
    mu = np.mean(x)
    var = np.mean((x - mu) ** 2)
    return mu, (np.sqrt(var) if var > 1e-18 else 1.0)


def train(w, v, c, m, max_epochs=500, step0=0.05, delta=1e-4, patience=4):
    L = len(v)
    sv, sc, sm = scaler(v), scaler(c), scaler(m)
    t = np.arange(2, L)
    Z = np.stack([(v[t - 1] - sv[0]) / sv[1], (v[t - 2] - sv[0]) / sv[1], (c[t] - sc[0]) / sc[1],
                  (c[t - 1] - sc[0]) / sc[1], (c[t - 2] - sc[0]) / sc[1], (m[t] - sm[0]) / sm[1],
                  (m[t - 1] - sm[0]) / sm[1], (m[t - 2] - sm[0]) / sm[1]], axis=1)
    T = (v[t] - sv[0]) / sv[1]

    def mse(w):
        h = np.tanh(Z @ w[:8] + w[8])
        return float(np.mean((w[9] * h + w[10] - T) ** 2)), h

    def grad(w):
        cur, h = mse(w)
        e = w[9] * h + w[10] - T
        dy = 2.0 / len(T) * e
        dz = dy * w[9] * (1 - h * h)
        return np.concatenate([Z.T @ dz, [dz.sum(), dy @ h, dy.sum()]])

    current, _ = mse(w)
    evals, epochs, hv = 1, 0, []
    stall = 0
    for _ in range(max_epochs):
        g = grad(w)
        step = step0
        nxt, _ = mse(w - step * g); evals += 1
        h = 0
        while nxt > current and h < 20:
            step *= 0.5; nxt, _ = mse(w - step * g); evals += 1; h += 1
        hv.append(h)
        if nxt > current:
            break
        w = w - step * g
        epochs += 1
        stall = stall + 1 if current - nxt < delta else 0
        current = nxt
        if stall >= patience:
            break
    return w, evals, epochs, hv


rng = np.random.default_rng(0)
models = [np.concatenate([rng.uniform(-0.3, 0.3, 8), rng.uniform(-0.1, 0.1, 1), rng.uniform(-0.3, 0.3, 1), [0.0]])
          for _ in range(n)]
cursor, stats = 0, []
for k in range(R):
    L = k + 1
    if L >= 50:  # warm-up 50
        for j in range((n + 1) // 2):
            wi = (cursor + j) % n
            models[wi], ev, ep, hv = train(models[wi], V[:L, wi], Cc[:L, wi], Mm[:L, wi])
            if k >= 100:
                stats.append((ev, ep, hv))
    cursor = (cursor + (n + 1) // 2) % n
ev = np.array([s[0] for s in stats]); ep = np.array([s[1] for s in stats])
hs = np.concatenate([s[2] for s in stats])
print(json.dumps({"trainings": len(stats), "evals_mean": float(ev.mean()), "evals_p90": float(np.percentile(ev, 90)),
                  "evals_max": int(ev.max()), "epochs_mean": float(ep.mean()),
                  "halvings_per_epoch_mean": float(hs.mean()),
                  "halvings_hist": np.bincount(hs, minlength=6)[:8].tolist(),
                  "max_evals_per_round": None}))
