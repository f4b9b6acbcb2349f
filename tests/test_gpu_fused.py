"""The fused worker kernel (csrc/c2_fused.cuh: forward + head + dW0 of every
emulated worker in one persistent launch) computes bitwise what the three
separate launches compute (same K order in every accumulation, same head
arithmetic, same CTA-ordered combine); LBBSP_NO_FUSE=1 selects the separate
kernels. Ragged sizes cover: one-row workers, a worker whose rows end inside
a 16-row head tile, and a worker with more 128-row tiles than CTAs."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(static, rounds, fuse, predictor="ema", trace=None, sm_budget=0):
    from paper_1806_02508_b200.mlp import MlpEngine, constant_trace
    n = len(static)
    old = os.environ.pop("LBBSP_NO_FUSE", None)
    if not fuse:
        os.environ["LBBSP_NO_FUSE"] = "1"
    try:
        eng = MlpEngine(dims=[784, 256, 10], global_batch=int(sum(static)), n_workers_local=n,
                        predictor=predictor, learning_rate=0.05, seed=3, max_iterations=rounds + 2,
                        trace=trace if trace is not None else constant_trace(n, rounds + 2),
                        static_sizes=static, sm_budget=sm_budget)
    finally:
        os.environ.pop("LBBSP_NO_FUSE", None)
        if old is not None:
            os.environ["LBBSP_NO_FUSE"] = old
    eng.run(rounds)
    p = np.concatenate([np.concatenate([w.ravel(), b]) for w, b in eng.params()])
    rec = eng.records()
    del eng
    return p, rec


@pytest.mark.parametrize("static", [
    [512] * 8,
    [300, 700, 100, 900, 500, 600, 400, 596],
    [1, 7, 1, 1, 1020, 1022, 1022, 1022],
    [3000, 200, 200, 200, 200, 200, 48, 48],
    [4096],
])
def test_fused_equals_separate_kernels_bitwise(static):
    a, ra = _run(static, 6, fuse=True)
    b, rb = _run(static, 6, fuse=False)
    assert np.array_equal(a, b), float(np.max(np.abs(a - b)))
    assert np.array_equal(ra["loss"], rb["loss"])


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
