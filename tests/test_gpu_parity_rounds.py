"""Multi-round parity of the benchmarked MLP path (north_star: "gradients,
NARX predictions and weights after N iterations must match within a stated
fp32/bf16 tolerance"; the reference's own bar is the trajectory test
test_cluster_sim.cpp:219-240).

Each test runs the engine one round at a time and checks, every round:
  * batch sizes: BIT-EXACT against the reference (oracle/_ref) replaying the
    device's measured speed stream (cluster_sim.cpp:355-402, 458-464);
  * the round's update (teacher-forced: restatement started from the device's
    weights of the previous round): relative L2 error of every layer's
    dW and db against oracle/mlp_oracle.lbbsp_round_bf16;
and at the end
  * the weight trajectory: the restatement iterated on its own from the
    initial weights with the device's sizes, relative L2 error of
    (W_N - W_0) per layer;
  * the recorded full-dataset loss against the restatement's loss of the
    device's weights (cluster_sim.cpp:445).

Why these bars. The device and the restatement round to bf16 at the same
points (activations, dZ, GEMM operands) but accumulate in a different order
(fp32 tensor-core tiles vs fp64), and the device is deterministic
(test_*_two_runs_bitwise_equal), so every difference is one of two
order-dependent events, both measured on B200 (profiles/r02_parity_rounds.txt):
  * a pre-activation within accumulation error of 0 flips its ReLU mask: one
    flip moves dW_l by one sample's outer product, ~ 1/sqrt(B * width) of the
    update (1e-3 for C2's first layer); rounds with a few flips reach 5e-3;
  * a bf16 rounding of an activation flips by one ulp (2^-8): hundreds per
    layer per round at C3 widths, compounding through 4 layers.
The second is also what two CPU restatements that differ only in summation
order (fp32 sgemm vs fp64) disagree by -- the "floor" measured here every
checked round; the device sits at 3-5x that floor (tensor-core fp32
accumulation is less accurate than sgemm's FMA chains).
Bars: C2 1e-2 per round (at most two rounds of the 110 up to 3e-2: clusters
of mask flips, measured up to 1.16e-2) and 1e-2 over the 110-round
trajectory (a sample dropped in every round, 1/sqrt(B) = 1.6e-2, fails it; a
dropped worker, ~0.35, fails it by far); C3 max(8 x floor, 1e-2) per round, 5e-2 over the trajectory.
"""
import json
import os

import numpy as np
import pytest

from oracle import mlp_oracle as MO
from paper_1806_02508_b200 import abi

pytestmark = pytest.mark.gpu

REPORT = os.environ.get("LBBSP_PARITY_REPORT")


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _checker():
    from oracle import oracle as O
    return O.reference() if O.reference_available() else O.restatement()


def _update_errors(prev, cur, exp):
    """per layer (dW, db) relative error of the device update vs expected"""
    out = []
    for (W0, b0), (W1, b1), (We, be) in zip(prev, cur, exp):
        out.append((rel(W1.astype(np.float64) - W0, We - W0), rel(b1.astype(np.float64) - b0, be - b0)))
    return out


def run_parity(orc, name, dims, B, n, rounds, predictor, trace, lr, seed=1, tf_rounds=None,
               traj_acc32=False, warmup=50):
    from paper_1806_02508_b200.mlp import MlpEngine
    eng = MlpEngine(dims=dims, global_batch=B, n_workers_local=n, predictor=predictor,
                    warmup_iterations=warmup, learning_rate=lr, seed=seed,
                    max_iterations=rounds + 2, trace=trace)
    x, y = eng.dataset()
    p0 = eng.params()
    porc = [(W.astype(np.float32), b.astype(np.float32)) for W, b in p0]
    prev = p0
    per_round = []
    for k in range(rounds):
        eng.run(1)
        rec = eng.records()
        sizes = rec["sizes"][k].tolist()
        assert sum(sizes) == B and min(sizes) >= 1
        stream = orc.sample_stream(seed, k, B, 1000)
        cur = eng.params()
        if tf_rounds is None or k in tf_rounds:
            exp, _ = MO.lbbsp_round_bf16(prev, x, y, stream, sizes, lr)
            alt, _ = MO.lbbsp_round_bf16(prev, x, y, stream, sizes, lr, acc32=True)
            dev = _update_errors(prev, cur, exp)
            floor = _update_errors([(W.astype(np.float64), b.astype(np.float64)) for W, b in prev],
                                   [(W, b) for W, b in alt], exp)
            per_round.append({"k": k, "sizes_min": min(sizes), "dev": dev, "floor": floor})
        nxt, _ = MO.lbbsp_round_bf16(porc, x, y, stream, sizes, lr, acc32=traj_acc32)
        porc = [(W.astype(np.float32), b.astype(np.float32)) for W, b in nxt]
        prev = cur
    rec = eng.records()
    traj = [(rel(W1.astype(np.float64) - W0, Wo.astype(np.float64) - W0),
             rel(b1.astype(np.float64) - b0, bo.astype(np.float64) - b0))
            for (W0, b0), (W1, b1), (Wo, bo) in zip(p0, cur, porc)]
    loss_dev = float(rec["loss"][rounds - 1])
    loss_orc = MO.full_loss(cur, x, y)
    out = {"name": name, "rounds": rounds, "per_round": per_round, "traj": traj,
           "loss_dev": loss_dev, "loss_orc": loss_orc, "rec": rec}
    if REPORT:
        os.makedirs(REPORT, exist_ok=True)
        with open(os.path.join(REPORT, f"parity_{name}.json"), "w") as f:
            json.dump({k: v for k, v in out.items() if k != "rec"}, f, indent=1)
    del eng
    return out


def check_bars(out, abs_bar, traj_bar, floor_mult=0.0, tail_rounds=0, tail_mult=1.0):
    """every checked round within the bar, except at most `tail_rounds`
    rounds within tail_mult x the bar (ReLU-mask flip clusters)"""
    worst, per_round = [], []
    for r in out["per_round"]:
        rw = []
        for l, ((dw, db), (fw, fb)) in enumerate(zip(r["dev"], r["floor"])):
            bw, bb = max(floor_mult * fw, abs_bar), max(floor_mult * fb, abs_bar)
            rw.append((dw / bw, r["k"], l, "W", dw, fw))
            rw.append((db / bb, r["k"], l, "b", db, fb))
        per_round.append(max(rw))
        worst += rw
    worst.sort(reverse=True)
    per_round.sort(reverse=True)
    over = [w for w in per_round if w[0] > 1.0]
    assert len(over) <= tail_rounds and (not over or over[0][0] <= tail_mult), \
        f"round update outside the bar: {worst[:3]} ({len(over)} rounds over)"
    for l, (tw, tb) in enumerate(out["traj"]):
        assert tw <= traj_bar and tb <= traj_bar, (out["name"], l, tw, tb)
    assert abs(out["loss_dev"] - out["loss_orc"]) <= 1e-3 * abs(out["loss_orc"]), \
        (out["loss_dev"], out["loss_orc"])


def test_c2_engine_110_rounds_sizes_and_weights(orc):
    """BASELINE configs[1] (the bench workload): MLP 784-256-10, 8 emulated
    workers, B=4096, LB-BSP + NARX (warm-up 50), benchmark-series straggler
    trace; 50 warm-up + 60 post-warm-up rounds."""
    from paper_1806_02508_b200.mlp import benchmark_trace
    n, B, R = 8, 4096, 110
    trace = benchmark_trace(n, R + 2, seed=3)
    out = run_parity(orc, "c2", [784, 256, 10], B, n, R, "narx", trace, 0.05)
    rec = out["rec"]
    # sizes: bit-exact vs the reference replaying the measured speeds
    chk = _checker()
    pcfg = abi.PredictorConfig.default(abi.PRED_NARX, warmup_iterations=50)
    seeds = [chk.mix_seed(1, 0x9ced1c70, i) for i in range(n)]
    c, m = trace[0][:, :R].T, trace[1][:, :R].T
    sizes, vpred = chk.replay_cpu(pcfg, seeds, B, rec["v_obs"], c, m)
    assert sizes.tolist() == rec["sizes"].tolist()
    assert np.array_equal(vpred, rec["v_pred"])
    # mask-flip clusters: measured per-round maxima 1.4e-3 .. 3.3e-3 in most
    # runs, 1.16e-2 in one of five (profiles/r02_parity_rounds.txt); a dropped
    # sample costs 1.6e-2 in every round it happens in
    check_bars(out, abs_bar=1e-2, traj_bar=1e-2, tail_rounds=2, tail_mult=3.0)


def test_c3_shape_10_rounds(orc):
    """BASELINE configs[2] per-GPU shape through the engine: MLP 4 x (4096 x
    4096) bf16, one worker, 2048 rows, 10 rounds (teacher-forced check on
    rounds 0, 4, 9; trajectory restated with fp32 accumulation)."""
    from paper_1806_02508_b200.mlp import constant_trace
    out = run_parity(orc, "c3", [4096] * 5, 2048, 1, 10, "ema", constant_trace(1, 12), 0.01,
                     tf_rounds={0, 4, 9}, traj_acc32=True)
    check_bars(out, abs_bar=1e-2, traj_bar=5e-2, floor_mult=8.0)


def test_c3_shape_two_runs_bitwise_equal():
    """Run-to-run determinism of the one-worker path (fixed reduction orders,
    no atomics in the weight path): two fresh engines, same seeds and sizes,
    bitwise-equal weights after 6 rounds."""
    from paper_1806_02508_b200.mlp import MlpEngine, constant_trace
    ps = []
    for _ in range(2):
        eng = MlpEngine(dims=[4096] * 5, global_batch=2048, n_workers_local=1, predictor="ema",
                        learning_rate=0.01, seed=1, max_iterations=8, trace=constant_trace(1, 8))
        eng.run(6)
        ps.append(np.concatenate([np.concatenate([w.ravel(), b]) for w, b in eng.params()]))
        del eng
    assert np.array_equal(ps[0], ps[1])


def test_c2_engine_two_runs_bitwise_equal():
    """Run-to-run determinism of the several-workers-per-GPU path (segmented
    reduction in worker order, CTA-ordered head partials, no float atomics in
    the weight path): two fresh engines with the same static ragged sizes,
    bitwise-equal weights after 40 rounds."""
    from paper_1806_02508_b200.mlp import MlpEngine, benchmark_trace
    n, B, R = 8, 4096, 40
    static = [300, 700, 100, 900, 500, 600, 400, 596]
    ps = []
    for _ in range(2):
        eng = MlpEngine(dims=[784, 256, 10], global_batch=B, n_workers_local=n, predictor="narx",
                        warmup_iterations=20, learning_rate=0.05, seed=1, max_iterations=R + 2,
                        trace=benchmark_trace(n, R + 2, seed=3), static_sizes=static)
        eng.run(R)
        ps.append(np.concatenate([np.concatenate([w.ravel(), b]) for w, b in eng.params()]))
        del eng
    assert np.array_equal(ps[0], ps[1])
