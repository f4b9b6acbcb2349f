"""The fused worker kernels (forward + head + dW0 of every emulated worker in
one persistent launch):
  * csrc/c2_fused.cuh (LBBSP_FUSE_SINGLE=1, one CTA per 128-row tile)
    computes bitwise what the three separate launches compute
    (LBBSP_NO_FUSE=1): same K order in every accumulation, same head
    arithmetic, same CTA-ordered combine;
  * csrc/c2_fused_pair.cuh (the default, a (2,1,1) cluster per tile split by
    hidden columns) sums the logits as two column halves, so it matches the
    separate kernels to the rounding of that sum: weights within 1e-3 of the
    total update after 6 rounds, bitwise deterministic run to run.
Ragged sizes cover one-row workers, a worker whose rows end inside a 16-row
head tile, and a worker with more 128-row tiles than CTA pairs."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(static, rounds, mode, predictor="ema", trace=None, sm_budget=0):
    """mode: 'pair' (default kernel), 'single' (LBBSP_FUSE_SINGLE), 'separate'
    (LBBSP_NO_FUSE). Returns (initial params, final params, records)."""
    from paper_1806_02508_b200.mlp import MlpEngine, constant_trace
    n = len(static)
    env = {"single": "LBBSP_FUSE_SINGLE", "separate": "LBBSP_NO_FUSE"}.get(mode)
    saved = {k: os.environ.pop(k, None) for k in ("LBBSP_FUSE_SINGLE", "LBBSP_NO_FUSE")}
    if env:
        os.environ[env] = "1"
    try:
        eng = MlpEngine(dims=[784, 256, 10], global_batch=int(sum(static)), n_workers_local=n,
                        predictor=predictor, learning_rate=0.05, seed=3, max_iterations=rounds + 2,
                        trace=trace if trace is not None else constant_trace(n, rounds + 2),
                        static_sizes=static, sm_budget=sm_budget)
    finally:
        for k, v in saved.items():
            os.environ.pop(k, None)
            if v is not None:
                os.environ[k] = v
    flat = lambda ps: np.concatenate([np.concatenate([w.ravel(), b]) for w, b in ps])
    p0 = flat(eng.params())
    eng.run(rounds)
    p = flat(eng.params())
    rec = eng.records()
    del eng
    return p0, p, rec


SIZES = [
    [512] * 8,
    [300, 700, 100, 900, 500, 600, 400, 596],
    [1, 7, 1, 1, 1020, 1022, 1022, 1022],
    [3000, 200, 200, 200, 200, 200, 48, 48],
    [4096],
]


@pytest.mark.parametrize("static", SIZES)
def test_single_cta_fused_equals_separate_kernels_bitwise(static):
    _, a, ra = _run(static, 6, "single")
    _, b, rb = _run(static, 6, "separate")
    assert np.array_equal(a, b), float(np.max(np.abs(a - b)))
    assert np.array_equal(ra["loss"], rb["loss"])


@pytest.mark.parametrize("static", SIZES)
def test_pair_fused_matches_separate_kernels(static):
    p0, a, _ = _run(static, 6, "pair")
    _, b, _ = _run(static, 6, "separate")
    upd = float(np.max(np.abs(b - p0)))
    assert float(np.max(np.abs(a - b))) <= 1e-3 * upd, (float(np.max(np.abs(a - b))), upd)
    _, a2, _ = _run(static, 6, "pair")
    assert np.array_equal(a, a2)


def test_fused_under_interference_and_small_budget():
    """Interference on, a reduced SM budget (fewer CTAs than 128-row tiles
    for the big worker), NARX predictor with LB-BSP dynamic sizes: the fused
    run completes, its sizes sum to B every round and its loss falls."""
    from paper_1806_02508_b200.mlp import MlpEngine, benchmark_trace
    n, B, R = 8, 4096, 70
    eng = MlpEngine(dims=[784, 256, 10], global_batch=B, n_workers_local=n, predictor="narx",
                    warmup_iterations=20, learning_rate=0.1, seed=1, max_iterations=R + 2,
                    trace=benchmark_trace(n, R + 2, seed=3), sm_budget=96)
    eng.run(R)
    rec = eng.records()
    assert (rec["sizes"].sum(axis=1) == B).all()
    assert rec["loss"][-1] < rec["loss"][0]
