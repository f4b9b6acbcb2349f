"""The fused worker kernels (forward + head + dW0 of every emulated worker in
one persistent launch):
  * csrc/c2_fused.cuh (LBBSP_FUSE_SINGLE=1, one CTA per 128-row tile)
    computes bitwise what the three separate launches compute
    (LBBSP_NO_FUSE=1): same K order in every accumulation, same head
    arithmetic, same CTA-ordered combine;
  * csrc/c2_fused_pair.cuh (the default, a (2,1,1) cluster per tile split by
    hidden columns) and csrc/c2_fused_quad.cuh (LBBSP_FUSE_QUAD=1, four CTAs)
    sum the logits as column partials, so they match the separate kernels to
    the rounding of that sum: weights within 1e-3 of the total update after
    6 rounds, bitwise deterministic run to run.
Ragged sizes cover one-row workers, a worker whose rows end inside a 16-row
head tile, and a worker with more 128-row tiles than CTA pairs."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(static, rounds, mode, predictor="ema", trace=None, sm_budget=0):
    """mode: 'pair' (default: two CTAs per tile), 'quad' (four,
    LBBSP_FUSE_QUAD), 'pair_kg' (pair kernel gathering the rows itself by
    tile::gather4, LBBSP_KGATHER), 'single' (LBBSP_FUSE_SINGLE), 'separate'
    (LBBSP_NO_FUSE). Returns (initial params, final params, records)."""
    from paper_1806_02508_b200.mlp import MlpEngine, constant_trace
    n = len(static)
    env = {"single": "LBBSP_FUSE_SINGLE", "separate": "LBBSP_NO_FUSE", "pair_kg": "LBBSP_KGATHER",
           "quad": "LBBSP_FUSE_QUAD"}.get(mode)
    saved = {k: os.environ.pop(k, None)
             for k in ("LBBSP_FUSE_SINGLE", "LBBSP_NO_FUSE", "LBBSP_KGATHER", "LBBSP_FUSE_QUAD")}
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


@pytest.mark.parametrize("mode", ["pair", "quad"])
@pytest.mark.parametrize("static", SIZES)
def test_split_fused_matches_separate_kernels(static, mode):
    p0, a, _ = _run(static, 6, mode)
    _, b, _ = _run(static, 6, "separate")
    upd = float(np.max(np.abs(b - p0)))
    assert float(np.max(np.abs(a - b))) <= 1e-3 * upd, (float(np.max(np.abs(a - b))), upd)
    _, a2, _ = _run(static, 6, mode)
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


@pytest.mark.parametrize("static", SIZES)
def test_pair_in_kernel_gather_equals_gather_kernel_bitwise(static):
    """tile::gather4 rows straight from the dataset land in shared memory in
    the same swizzled layout as the TMA tile of the gathered batch: weights
    and losses bitwise equal to the pair kernel fed by the gather kernel."""
    _, a, ra = _run(static, 6, "pair_kg")
    _, b, rb = _run(static, 6, "pair")
    assert np.array_equal(a, b), float(np.max(np.abs(a - b)))
    assert np.array_equal(ra["loss"], rb["loss"])


def test_pair_in_kernel_gather_dynamic_sizes_and_e2e_buffers():
    """LB-BSP sizes that change every round (Perfect predictor over the
    benchmark trace: deterministic, so both runs see the same sizes) under
    interference, then end-to-end steps that alternate the two dataset
    buffers (each graph gathers from its own): bitwise equal to the
    gather-kernel path over the same rounds."""
    import torch
    from paper_1806_02508_b200.mlp import MlpEngine, benchmark_trace
    from paper_1806_02508_b200.hostio import pinned_empty
    n, B, R = 8, 4096, 40
    out = []
    for kg in (True, False):
        saved = os.environ.pop("LBBSP_KGATHER", None)
        if kg:
            os.environ["LBBSP_KGATHER"] = "1"
        try:
            eng = MlpEngine(dims=[784, 256, 10], global_batch=B, n_workers_local=n, predictor="perfect",
                            learning_rate=0.05, seed=1, max_iterations=R + 12,
                            trace=benchmark_trace(n, R + 12, seed=3))
        finally:
            os.environ.pop("LBBSP_KGATHER", None)
            if saved is not None:
                os.environ["LBBSP_KGATHER"] = saved
        eng.run(R)
        x, y = eng.dataset()
        xb = pinned_empty(x.shape, torch.bfloat16, 0)
        xb.copy_(torch.from_numpy(x).to(torch.bfloat16))
        yb = pinned_empty(y.shape, torch.int32, 0)
        yb.copy_(torch.from_numpy(y.astype(np.int32)))
        osz = pinned_empty((n,), torch.int32, 0)
        ol = pinned_empty((1,), torch.float64, 0)
        for _ in range(8):
            eng.step_e2e(xb.data_ptr(), yb.data_ptr(), osz.data_ptr(), ol.data_ptr())
        torch.cuda.synchronize()
        rec = eng.records()
        # the host buffers hold the last round's sizes and loss
        assert osz.tolist() == rec["sizes"][rec["rows"] - 1].tolist()
        assert ol.item() == float(rec["loss"][rec["rows"] - 1])
        out.append((np.concatenate([np.concatenate([w.ravel(), b]) for w, b in eng.params()]),
                    rec["sizes"].copy(), rec["loss"].copy()))
        del eng
    assert np.array_equal(out[0][1], out[1][1])
    assert np.array_equal(out[0][0], out[1][0]), float(np.max(np.abs(out[0][0] - out[1][0])))
    assert np.array_equal(out[0][2], out[1][2])
