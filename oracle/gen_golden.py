"""ORACLE / TEST INFRASTRUCTURE ONLY.

Generates the golden vectors under tests/golden/ by running the UNMODIFIED
reference (oracle/_ref/liblbbsp_ref.so, built from /root/reference by
oracle/Makefile). Floats are stored as hex strings (float.hex) so the files
pin bits, not 9-significant-digit text.

    python oracle/gen_golden.py          # rewrites tests/golden/*.json
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)

from oracle import oracle as O  # noqa: E402
from paper_1806_02508_b200 import abi  # noqa: E402

GOLDEN = os.path.join(REPO, "tests", "golden")


def hexs(a):
    return [float(x).hex() for x in np.ravel(a)]


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# Scenario table shared with the tests (tests/scenarios.py imports this).
SIM_SCENARIOS = {
    # C1-shaped reference run: 4 workers, B=512, Hetero-L3, NARX warm-up 50
    "c1_hetero_l3_narx": dict(preset="hetero-l3", workers=4, total_budget=512, predictor="narx",
                              warmup_iterations=50, max_updates=300, convergence_loss=1e-4),
    # configs/hetero_l3_lbbsp.json
    "hetero_l3_lbbsp": dict(preset="hetero-l3", workers=8, total_budget=1024, predictor="ema",
                            warmup_iterations=50, max_updates=300, convergence_loss=0.30),
    # configs/hetero_l3_bsp.json
    "hetero_l3_bsp": dict(scheme="bsp", preset="hetero-l3", workers=8, total_budget=1024,
                          predictor="ema", warmup_iterations=50, max_updates=300,
                          convergence_loss=0.30),
    # configs/bench_predictors.json (benchmark dynamics, NARX)
    "bench_predictors_narx": dict(preset=None, dynamics=abi.DYN_BENCHMARK, workers=8,
                                  total_budget=1024, predictor="narx", warmup_iterations=50,
                                  max_updates=200, convergence_loss=1e-4, seed=3),
    # configs/gpu_cluster.json
    "gpu_cluster": dict(preset=None, workers=8, total_budget=3040,
                        gpu_profiles=[(0.002, 0.05, 58, 384)] * 4 + [(0.0007, 0.05, 92, 1184)] * 2
                        + [(0.0005, 0.05, 103, 788)] * 2, base_comm_s=0.1,
                        bandwidth_drop=(0, 150, 3.0), max_updates=300, convergence_loss=1e-4),
    # test_cluster_sim.cpp:192-217 (straggler dynamics, seed 12)
    "replay_stragglers": dict(preset=None, dynamics=abi.DYN_STRAGGLER, workers=4,
                              total_budget=256, predictor="ema", warmup_iterations=1 << 20,
                              stragglers=[(0.0, 0.0, 0.0, 10), (0.5, 0.3, 0.0, 10),
                                          (0.75, 0.5, 0.1, 10), (0.75, 0.66, 0.2, 10)],
                              seed=12, max_updates=100, convergence_loss=1e-9, dataset_size=200,
                              dataset_dim=4),
    # memoryless + perfect predictors on static speeds
    "static_perfect": dict(preset=None, dynamics=abi.DYN_STATIC, workers=4, total_budget=512,
                           static_cpu=[1.0, 0.75, 0.5, 0.25], predictor="perfect",
                           max_updates=40, convergence_loss=1e-9, dataset_size=200,
                           dataset_dim=4),
    "static_memoryless": dict(preset=None, dynamics=abi.DYN_STATIC, workers=4, total_budget=512,
                              static_cpu=[1.0, 0.9, 0.4, 0.2], static_mem=[1.0, 0.3, 0.6, 0.2],
                              predictor="memoryless", max_updates=40, convergence_loss=1e-9,
                              dataset_size=200, dataset_dim=4),
}


def gen_solver(ref):
    cases = []
    rng = np.random.default_rng(20261018)
    fixed = [([4, 2, 1, 1], 512), ([1, 1, 1, 1], 512), ([1e-9, 5.0, 5.0], 100), ([3, 2, 2], 10),
             ([1.0], 1), ([2.0, 1.0], 3)]
    for v, b in fixed:
        cases.append({"speeds": hexs(v), "budget": b, "sizes": ref.cpu_allocate(v, b).tolist()})
    for _ in range(300):
        n = int(rng.integers(1, 65))
        v = rng.uniform(1e-3, 50.0, n)
        if rng.random() < 0.2:
            v[rng.integers(0, n)] = 1e-9
        b = int(rng.integers(n, 5000))
        cases.append({"speeds": hexs(v), "budget": b, "sizes": ref.cpu_allocate(v, b).tolist()})
    errors = []
    for v, b in [([1.0, 0.0], 10), ([1.0, 1.0, 1.0], 2), ([], 5), ([1.0, -2.0], 4)]:
        try:
            ref.cpu_allocate(v, b)
        except Exception as e:  # noqa: BLE001
            errors.append({"speeds": hexs(v), "budget": b, "type": type(e).__name__,
                           "message": str(e)})
    gpu = []
    fixed_g = [
        ([(0.01, 0.1, 1, 1 << 20), (0.005, 0.1, 1, 1 << 20)], [0, 0], 759),
        ([(0.01, 0.1, 1, 1 << 20), (0.005, 0.1, 1, 1 << 20)], [0, 0], 200),
        ([(0.002, 0.05, 58, 384)], [0.0], 380),
        ([(0.002, 0.05, 58, 384)] * 2, [0.1, 0.1], 400),
        ([(0.002, 0.05, 58, 384)] * 4 + [(0.0007, 0.05, 92, 1184)] * 2
         + [(0.0005, 0.05, 103, 788)] * 2, [0.1] * 8, 3040),
    ]
    for p, c, b in fixed_g:
        gpu.append({"profiles": [[float(x[0]).hex(), float(x[1]).hex(), x[2], x[3]] for x in p],
                    "comm": hexs(c), "budget": b, "sizes": ref.gpu_allocate(p, c, b).tolist()})
    for _ in range(200):
        n = int(rng.integers(1, 33))
        prof = []
        lo = hi = 0
        for _i in range(n):
            sat = int(rng.integers(1, 128))
            oom = sat + int(rng.integers(0, 1024))
            prof.append((float(rng.uniform(5e-4, 0.02)), float(rng.uniform(0.0, 0.3)), sat, oom))
            lo += sat
            hi += oom
        comm = rng.uniform(0.0, 0.3, n)
        b = int(rng.integers(lo, hi + 1))
        gpu.append({"profiles": [[float(x[0]).hex(), float(x[1]).hex(), x[2], x[3]] for x in prof],
                    "comm": hexs(comm), "budget": b, "sizes": ref.gpu_allocate(prof, comm, b).tolist()})
    gpu_err = []
    p2 = [(0.002, 0.05, 58, 384), (0.0008, 0.08, 92, 1184)]
    for b in (100, 2000):
        try:
            ref.gpu_allocate(p2, [0.0, 0.0], b)
        except Exception as e:  # noqa: BLE001
            gpu_err.append({"profiles": [[float(x[0]).hex(), float(x[1]).hex(), x[2], x[3]] for x in p2],
                            "comm": hexs([0, 0]), "budget": b, "type": type(e).__name__,
                            "message": str(e)})
    return {"cpu": cases, "cpu_errors": errors, "gpu": gpu, "gpu_errors": gpu_err}


def gen_predictor(ref):
    out = {"ema": [], "narx_predict": [], "narx_train": [], "tanh": {}}
    rng = np.random.default_rng(7)
    for n in (1, 2, 5, 50, 1000):
        s = rng.uniform(0.5, 20.0, n)
        for a in (0.2, 1.0, 0.05):
            out["ema"].append({"series": hexs(s), "alpha": float(a).hex(), "value": ref.ema(s, a).hex()})
    for seed in (1, 5, 31, 77):
        m = ref.narx_init(seed)
        m.speed_mean, m.speed_stddev = 6.5, 2.25
        m.cpu_mean, m.cpu_stddev = 0.7, 0.2
        for _ in range(10):
            v = rng.uniform(1, 12, 2); c = rng.uniform(0.2, 1, 3); mm = rng.uniform(0.2, 1, 3)
            out["narx_predict"].append({"model": [float(x).hex() for x in m.as_tuple()],
                                        "v": hexs(v), "c": hexs(c), "m": hexs(mm),
                                        "value": ref.narx_predict(m, v, c, mm).hex()})
    # training on reference-test-shaped histories (test_predictor.cpp:105-179)
    hist = []
    L = 60
    hist.append(("constant", np.full(L, 7.5), np.full(L, 0.8), np.full(L, 0.9), 20, 5))
    k = np.arange(200)
    c = 0.5 + 0.4 * np.sin(k / 10.0)
    noise = rng.uniform(-0.1, 0.1, 200)
    hist.append(("sine", 10.0 * c + noise, c, np.ones(200), 30, 3))
    c2 = rng.uniform(0.3, 1.0, 400)
    hist.append(("linear", 10.0 * c2, c2, np.ones(400), 50, 9))
    series = ref.benchmark_series(3, 1000)
    vb = 10.0 * series[0] * series[2]
    hist.append(("benchmark", vb, series[0], series[1], 50, 12))
    for name, v, c, m, minh, seed in hist:
        model = ref.narx_init(seed)
        cfg = abi.NarxTrainConfig.default(min_history=minh)
        before = [float(x).hex() for x in model.as_tuple()]
        rep, log = ref.narx_train(model, v, c, m, cfg)
        out["narx_train"].append({"name": name, "v": hexs(v), "c": hexs(c), "m": hexs(m),
                                  "min_history": minh, "model_in": before,
                                  "model_out": [float(x).hex() for x in model.as_tuple()],
                                  "ran": rep.ran, "epochs": rep.epochs,
                                  "final_loss": float(rep.final_loss).hex(),
                                  "loss_log": hexs(log)})
    import math
    xs = np.concatenate([rng.uniform(-30, 30, 2000), rng.uniform(-1.2, 1.2, 2000),
                         [0.0, -0.0, 1e-300, 2.0 ** -60, 22.0, -22.0, 0.5 * math.log(3)]])
    out["tanh"] = {"x": hexs(xs), "y": [math.tanh(float(x)).hex() for x in xs]}
    return out


def gen_sim(ref):
    out = {}
    for name, kw in SIM_SCENARIOS.items():
        cfg, keep = abi.make_sim_config(**kw)
        r = ref.sim_run(cfg)
        out[name] = {"rows": int(len(r["loss"])), "converged": r["converged"],
                     "batch": r["batch"].tolist(),
                     "sha_v_pred": digest(r["v_pred"]), "sha_v_actual": digest(r["v_actual"]),
                     "sha_wall": digest(r["wall"]), "sha_params": digest(r["params"]),
                     "sha_loss": digest(r["loss"]),
                     "v_pred_last": hexs(r["v_pred"][-1]), "wall_last": float(r["wall"][-1]).hex(),
                     "loss_last": float(r["loss"][-1]).hex(),
                     "params_last": hexs(r["params"][-1])}
    return out


def gen_stream(ref):
    out = []
    for seed, k, b, n in [(1, 0, 512, 1000), (1, 7, 4096, 1000), (3, 123, 1024, 1000),
                          (21, 2, 300, 17)]:
        s = ref.sample_stream(seed, k, b, n)
        out.append({"seed": seed, "k": k, "budget": b, "N": n, "sha": digest(s.astype(np.int32)),
                    "head": s[:16].tolist()})
    return out


def main():
    if not O.reference_available():
        raise SystemExit("oracle/_ref/liblbbsp_ref.so missing: run `make -C oracle` where "
                         "/root/reference exists")
    ref = O.reference()
    os.makedirs(GOLDEN, exist_ok=True)
    for name, fn in (("solver", gen_solver), ("predictor", gen_predictor), ("sim", gen_sim),
                     ("stream", gen_stream)):
        with open(os.path.join(GOLDEN, name + ".json"), "w") as f:
            json.dump(fn(ref), f, separators=(",", ":"))
        print("wrote", name)


if __name__ == "__main__":
    main()
