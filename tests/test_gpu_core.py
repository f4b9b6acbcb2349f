"""GPU parity tests for the fp64 hot-path kernels (K1-K10) and the fused
iteration, through the C-ABI (paper_1806_02508_b200/lbbsp.py mirrors the
reference API). Bars:
  * allocations (cpu_allocate / gpu_allocate, batch sizes of every round):
    bit-exact vs the reference;
  * EMA, NARX predict, NARX training, v_pred, v_actual, wall: bit-exact;
  * LR gradients / loss / parameter trajectory: the device exp/log1p are not
    glibc's, so within 1e-12 relative per call and 1e-9 relative over a run
    (the reference's own aggregation-order bar, test_cluster_sim.cpp:219-240).
"""
import hashlib

import numpy as np
import pytest

from oracle.gen_golden import SIM_SCENARIOS
from paper_1806_02508_b200 import abi
from paper_1806_02508_b200.errors import InvalidArgument, OutOfRange
from util import bits_equal, fromhex, profiles_fromhex

pytestmark = pytest.mark.gpu


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ------------------------------------------------------------------ K1 / K2
def test_cpu_allocate_known_answers(lb):
    # test_batch_sizer.cpp:21-27, 77-82
    assert lb.cpu_allocate([4, 2, 1, 1], 512).sizes == [256, 128, 64, 64]
    assert lb.cpu_allocate([1, 1, 1, 1], 512).sizes == [128] * 4
    a = lb.cpu_allocate([1e-9, 5.0, 5.0], 100)
    assert a.sizes[0] == 1 and sum(a.sizes) == 100


def test_cpu_allocate_golden(lb, golden):
    for case in golden("solver")["cpu"]:
        assert lb.cpu_allocate(fromhex(case["speeds"]), case["budget"]).sizes == case["sizes"]


def test_gpu_allocate_golden(lb, golden):
    for case in golden("solver")["gpu"]:
        got = lb.gpu_allocate(profiles_fromhex(case["profiles"]), fromhex(case["comm"]),
                              case["budget"])
        assert got.sizes == case["sizes"]


def test_solver_errors_keep_reference_wording(lb, golden):
    g = golden("solver")
    for case in g["cpu_errors"] + g["gpu_errors"]:
        with pytest.raises(InvalidArgument) as ei:
            if "profiles" in case:
                lb.gpu_allocate(profiles_fromhex(case["profiles"]), fromhex(case["comm"]),
                                case["budget"])
            else:
                lb.cpu_allocate(fromhex(case["speeds"]), case["budget"])
        assert str(ei.value) == case["message"]


def test_cpu_allocate_fuzz_vs_oracle(lb, orc):
    # budget conservation fuzz (test_batch_sizer.cpp:220-229) plus bit parity
    rng = np.random.default_rng(0xf0220)
    for _ in range(3000):
        n = int(rng.integers(1, 17)) if rng.random() < 0.8 else int(rng.integers(17, 1025))
        v = rng.uniform(1e-3, 50.0, n)
        b = int(rng.integers(n, 5000 if n < 17 else 1 << 17))
        got = lb.cpu_allocate(v, b).sizes
        assert sum(got) == b
        assert got == orc.cpu_allocate(v, b).tolist()


def test_gpu_allocate_fuzz_vs_oracle(lb, orc):
    rng = np.random.default_rng(4242)
    for trial in range(400):
        n = int(rng.integers(1, 9)) if trial < 300 else int(rng.integers(64, 513))
        prof, lo, hi = [], 0, 0
        for _ in range(n):
            sat = int(rng.integers(1, 128)); oom = sat + int(rng.integers(0, 1024))
            prof.append((float(rng.uniform(5e-4, 0.02)), float(rng.uniform(0, 0.2)), sat, oom))
            lo += sat; hi += oom
        comm = rng.uniform(0.0, 0.3, n)
        b = int(rng.integers(lo, hi + 1))
        assert lb.gpu_allocate(prof, comm, b).sizes == orc.gpu_allocate(prof, comm, b).tolist()


# ------------------------------------------------------------------ K3-K5
def test_ema_golden(lb, golden):
    for case in golden("predictor")["ema"]:
        got = lb.ema(fromhex(case["series"]), float.fromhex(case["alpha"]))
        assert got.hex() == case["value"]
    with pytest.raises(InvalidArgument):
        lb.ema([], 0.2)
    with pytest.raises(InvalidArgument):
        lb.ema([1.0], 0.0)


def _model(vals):
    m = lb_narx()
    for j in range(8):
        m.input_weights[j] = vals[j]
    (m.hidden_bias, m.output_weight, m.output_bias, m.speed_mean, m.speed_stddev, m.cpu_mean,
     m.cpu_stddev, m.mem_mean, m.mem_stddev) = vals[8:]
    return m


def lb_narx():
    from paper_1806_02508_b200.lbbsp import Narx
    return Narx()


def test_narx_predict_golden(lb, golden):
    for case in golden("predictor")["narx_predict"]:
        m = _model(fromhex(case["model"]))
        got = lb.narx_predict(m, fromhex(case["v"]), fromhex(case["c"]), fromhex(case["m"]))
        assert got.hex() == case["value"]
    # test_predictor.cpp:80-88
    m = lb_narx()
    m.output_bias = 6.5
    assert lb.narx_predict(m, [1, 2], [1, 1, 1], [1, 1, 1]) == pytest.approx(6.5)
    m.output_bias = -3.0
    assert lb.narx_predict(m, [1, 2], [1, 1, 1], [1, 1, 1]) == pytest.approx(1e-3)


def test_device_tanh_bit_exact_vs_glibc(lb, golden):
    # every NARX forward goes through glibc_tanh (exactmath.cuh); with zero
    # input weights and identity scalers the prediction is w_o*tanh(b_h) + b_o
    t = golden("predictor")["tanh"]
    xs, ys = fromhex(t["x"]), fromhex(t["y"])
    m = lb_narx()
    m.output_weight, m.output_bias = 1.0, 0.0
    bad = 0
    for x, y in zip(xs[::7], ys[::7]):
        m.hidden_bias = x
        got = lb.narx_predict(m, [0, 0], [0, 0, 0], [0, 0, 0], floor=-10.0)
        bad += got != y
    assert bad == 0


def test_device_tanh_batch_bit_exact_vs_host_libm(lb, golden):
    """glibc_tanh over ~1.2M inputs covering every expm1 reduction branch
    (k = 0, +-1, 2..19, 20..56, > 56), the range boundaries and the golden
    vectors, against the host libm (the reference's std::tanh)."""
    import math
    rng = np.random.default_rng(7)
    ln2 = math.log(2)  # expm1(+-2|x|) switches branch at |x| = (k + 0.5) ln2 / 2
    bounds = [0.0, 2.0 ** -55, 2.0 ** -28, 0.25 * ln2, 0.75 * ln2, 1.0, 1.25 * ln2,
              9.75 * ln2, 19.4, 28.25 * ln2, 22.0, 28.0]
    near = np.concatenate([np.nextafter(b, np.inf) + np.arange(-40, 40) * np.spacing(max(b, 1e-300))
                           for b in bounds])
    xs = np.concatenate([rng.uniform(-25, 25, 400000), rng.uniform(-1.2, 1.2, 400000),
                         rng.normal(0, 1e-3, 100000), rng.uniform(0.3, 0.4, 100000),
                         rng.uniform(0.5, 0.55, 100000), near, -near,
                         np.array([1e-310, -1e-310, 1e300, -1e300, np.inf, -np.inf]),
                         fromhex(golden("predictor")["tanh"]["x"])])
    got = lb.glibc_tanh(xs)
    want = np.array([math.tanh(x) for x in xs])
    bad = np.flatnonzero(got.view(np.uint64) != want.view(np.uint64))
    assert bad.size == 0, f"{bad.size} mismatches, e.g. {[(xs[i], got[i], want[i]) for i in bad[:3]]}"


def test_narx_train_golden(lb, golden):
    for case in golden("predictor")["narx_train"]:
        m = _model(fromhex(case["model_in"]))
        h = lb.SpeedHistory()
        for v, c, mm in zip(fromhex(case["v"]), fromhex(case["c"]), fromhex(case["m"])):
            h.push(v, c, mm)
        cfg = abi.NarxTrainConfig.default(min_history=case["min_history"])
        rep = lb.narx_train_online(m, h, cfg)
        assert rep.ran == bool(case["ran"]) and rep.epochs == case["epochs"], case["name"]
        assert rep.final_loss.hex() == case["final_loss"], case["name"]
        assert bits_equal(m.as_tuple(), fromhex(case["model_out"])), case["name"]
        assert bits_equal(m.training_loss, fromhex(case["loss_log"])), case["name"]


def test_narx_train_noop_below_warmup(lb):
    # test_predictor.cpp:122-130
    h = lb.SpeedHistory()
    for _ in range(100):
        h.push(5.0, 1.0, 1.0)
    m = lb.narx_init(1)
    before = m.as_tuple()
    rep = lb.narx_train_online(m, h, abi.NarxTrainConfig.default())
    assert not rep.ran and m.as_tuple() == before


def test_pipeline_returns_ema_before_warmup(lb, orc):
    # test_predictor.cpp:242-255
    cfg = abi.PredictorConfig.default(abi.PRED_NARX, warmup_iterations=50)
    p = lb.SpeedPredictor(cfg, 77)
    rng = np.random.default_rng(404)
    h = lb.SpeedHistory()
    for _ in range(49):
        h.push(rng.uniform(2, 12), rng.uniform(0.2, 1.0), 1.0)
        assert p.predict(h, 0.9, 1.0) == orc.ema(h.speed, 0.2)


# ------------------------------------------------------------------ K6-K10
def test_sample_stream_golden(lb, golden):
    import torch
    from paper_1806_02508_b200._lib import check, lib
    for case in golden("stream"):
        out = torch.zeros(case["budget"], dtype=torch.int32, device="cuda")
        check(lib().lbbsp_sample_stream(case["seed"], case["k"], case["budget"], case["N"],
                                        out.data_ptr(), None))
        torch.cuda.synchronize()
        s = out.cpu().numpy()
        assert s[:16].tolist() == case["head"]
        assert digest(s.astype(np.int32)) == case["sha"]


def test_lr_gradient_loss_aggregate_vs_oracle(lb, orc):
    feat, lab = orc.generate_dataset(17, 60, 5)
    data = lb.generate_dataset(17, 60, 5)
    params = [0.1, 0.2, -0.3, 0.4, -0.5]
    rng = np.random.default_rng(1234)
    for _ in range(50):
        idx = rng.integers(0, 60, int(rng.integers(1, 40)))
        g = lb.batch_gradient(lb.ModelState(params), data, idx).values
        e = orc.batch_gradient(feat, lab, params, idx)
        np.testing.assert_allclose(g, e, rtol=1e-12, atol=1e-15)
    assert lb.loss(lb.ModelState(params), data) == pytest.approx(orc.loss(feat, lab, params),
                                                                 rel=1e-12)
    with pytest.raises(OutOfRange):
        lb.batch_gradient(lb.ModelState(params), data, [60])
    with pytest.raises(InvalidArgument):
        lb.batch_gradient(lb.ModelState(params), data, [])
    grads = [lb.Gradient([4.0], 1), lb.Gradient([8.0], 3)]
    assert lb.aggregate_weighted(grads).values[0] == pytest.approx((4.0 + 24.0) / 4.0)
    G = rng.normal(size=(7, 11))
    S = rng.integers(1, 50, 7)
    for w in (True, False):
        got = (lb.aggregate_weighted if w else lb.aggregate_naive)(
            [lb.Gradient(list(G[i]), int(S[i])) for i in range(7)]).values
        assert bits_equal(got, orc.aggregate(G, S, w))


def test_ps_step_lbbsp_and_validation(lb):
    # test_coordination.cpp:86-124
    m = lb.ModelState([0.0], 1.0)
    ready = [lb.PendingUpdate(0, lb.Gradient([2.0], 1), 1),
             lb.PendingUpdate(1, lb.Gradient([6.0], 3), 1)]
    nxt = lb.ps_step(lb.SchemeConfig(abi.SCHEME_LBBSP, 0, 4), 2, m, ready)
    assert nxt.params[0] == pytest.approx(-(2.0 + 18.0) / 4.0) and nxt.clock == 1
    with pytest.raises(InvalidArgument):
        lb.ps_step(lb.SchemeConfig(abi.SCHEME_BSP, 0, 2), 2, m, ready[:1])
    with pytest.raises(InvalidArgument):
        lb.ps_step(lb.SchemeConfig(abi.SCHEME_LBBSP, 0, 2), 2, m, [ready[0], ready[0]])


# ------------------------------------------------------------------ A1 fused
@pytest.mark.parametrize("name", sorted(SIM_SCENARIOS))
def test_fused_iteration_vs_reference(lb, golden, name):
    g = golden("sim")[name]
    sim = lb.Simulation(**SIM_SCENARIOS[name])
    r = sim.run()
    assert len(r.loss) == g["rows"]
    # bit-exact allocations, predictions, realised speeds and wall times
    assert r.batch.tolist() == g["batch"]
    assert digest(r.v_pred) == g["sha_v_pred"]
    assert digest(r.v_actual) == g["sha_v_actual"]
    assert digest(r.wall) == g["sha_wall"]
    # workload numerics within the reference's own 1e-9 trajectory bar
    np.testing.assert_allclose(r.params[-1], fromhex(g["params_last"]), rtol=1e-9, atol=1e-12)
    assert r.loss[-1] == pytest.approx(float.fromhex(g["loss_last"]), rel=1e-9)
    assert int(r.batch.sum(axis=1).min()) == int(r.batch.sum(axis=1).max())


def test_fused_iteration_vs_oracle_full_arrays(lb, orc):
    kw = SIM_SCENARIOS["c1_hetero_l3_narx"]
    cfg, keep = abi.make_sim_config(**kw)
    e = orc.sim_run(cfg)
    r = lb.Simulation(**kw).run()
    assert bits_equal(r.v_pred, e["v_pred"])
    assert bits_equal(r.tp, e["tp"]) and bits_equal(r.tm, e["tm"])
    assert bits_equal(r.wait, e["wait"])
    np.testing.assert_allclose(r.params, e["params"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(r.grad_norm, e["grad_norm"], rtol=1e-9, atol=1e-14)


def test_bsp_lbbsp_share_parameter_trajectory(lb):
    # controlled sampling, test_cluster_sim.cpp:219-240
    base = dict(preset=None, dynamics=abi.DYN_STATIC, workers=4, total_budget=512,
                static_cpu=[1.0, 0.7, 0.5, 0.25], warmup_iterations=1 << 20, max_updates=60,
                convergence_loss=1e-9, dataset_size=200, dataset_dim=4)
    rb = lb.Simulation(scheme="bsp", **base).run()
    rl = lb.Simulation(scheme="lb-bsp", **base).run()
    assert (rl.batch != 128).any()
    np.testing.assert_allclose(rb.params, rl.params, rtol=1e-9, atol=1e-9)


def test_reference_signature_cpp_shim(lb):
    """include/lbbsp_b200.hpp (reference signatures + exception types) against
    the reference's known answers, as a compiled C++ program."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "test_shim")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
