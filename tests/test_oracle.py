"""Pin the oracle: the C restatement (oracle/lbbsp_oracle.c) must reproduce the
golden vectors produced by the unmodified reference (tests/golden/, made by
oracle/gen_golden.py from oracle/_ref) bit-for-bit, and, where oracle/_ref is
built, agree with it on fresh fuzzed inputs. CPU only."""
import hashlib
import math

import numpy as np
import pytest

from oracle.gen_golden import SIM_SCENARIOS
from paper_1806_02508_b200 import abi
from paper_1806_02508_b200.errors import InvalidArgument
from util import bits_equal, fromhex, profiles_fromhex


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_solver_golden(orc, golden):
    g = golden("solver")
    for case in g["cpu"]:
        got = orc.cpu_allocate(fromhex(case["speeds"]), case["budget"])
        assert got.tolist() == case["sizes"]
    for case in g["gpu"]:
        got = orc.gpu_allocate(profiles_fromhex(case["profiles"]), fromhex(case["comm"]),
                               case["budget"])
        assert got.tolist() == case["sizes"]


def test_solver_error_wording(orc, golden):
    g = golden("solver")
    for case in g["cpu_errors"] + g["gpu_errors"]:
        with pytest.raises(InvalidArgument) as ei:
            if "profiles" in case:
                orc.gpu_allocate(profiles_fromhex(case["profiles"]), fromhex(case["comm"]),
                                 case["budget"])
            else:
                orc.cpu_allocate(fromhex(case["speeds"]), case["budget"])
        assert str(ei.value) == case["message"]


def test_predictor_golden(orc, golden):
    g = golden("predictor")
    for case in g["ema"]:
        assert orc.ema(fromhex(case["series"]), float.fromhex(case["alpha"])).hex() == case["value"]
    for case in g["narx_predict"]:
        m = abi.NarxModel()
        vals = fromhex(case["model"])
        for j in range(8):
            m.input_weights[j] = vals[j]
        (m.hidden_bias, m.output_weight, m.output_bias, m.speed_mean, m.speed_stddev, m.cpu_mean,
         m.cpu_stddev, m.mem_mean, m.mem_stddev) = vals[8:]
        got = orc.narx_predict(m, fromhex(case["v"]), fromhex(case["c"]), fromhex(case["m"]))
        assert got.hex() == case["value"]


def _model_from(vals):
    m = abi.NarxModel()
    for j in range(8):
        m.input_weights[j] = vals[j]
    (m.hidden_bias, m.output_weight, m.output_bias, m.speed_mean, m.speed_stddev, m.cpu_mean,
     m.cpu_stddev, m.mem_mean, m.mem_stddev) = vals[8:]
    return m


def test_narx_train_golden(orc, golden):
    for case in golden("predictor")["narx_train"]:
        m = _model_from(fromhex(case["model_in"]))
        cfg = abi.NarxTrainConfig.default(min_history=case["min_history"])
        rep, log = orc.narx_train(m, fromhex(case["v"]), fromhex(case["c"]), fromhex(case["m"]), cfg)
        assert rep.ran == case["ran"] and rep.epochs == case["epochs"], case["name"]
        assert bits_equal(m.as_tuple(), fromhex(case["model_out"])), case["name"]
        assert bits_equal(log, fromhex(case["loss_log"])), case["name"]


def test_tanh_port_matches_glibc_golden(orc, golden):
    t = golden("predictor")["tanh"]
    xs, ys = fromhex(t["x"]), fromhex(t["y"])
    got = np.array([orc.tanh_port(x) for x in xs])
    assert bits_equal(got, ys)


def test_tanh_port_matches_host_libm(orc):
    rng = np.random.default_rng(99)
    xs = np.concatenate([rng.uniform(-25, 25, 50000), rng.uniform(-1, 1, 50000),
                         rng.normal(0, 1e-3, 5000), rng.uniform(0.9, 1.1, 5000)])
    bad = [x for x in xs if orc.tanh_port(x) != math.tanh(x)]
    assert not bad, f"{len(bad)} mismatches, e.g. {bad[:3]}"


@pytest.mark.parametrize("name", sorted(SIM_SCENARIOS))
def test_sim_golden(orc, golden, name):
    g = golden("sim")[name]
    cfg, keep = abi.make_sim_config(**SIM_SCENARIOS[name])
    r = orc.sim_run(cfg)
    assert len(r["loss"]) == g["rows"]
    assert r["batch"].tolist() == g["batch"]
    assert digest(r["v_pred"]) == g["sha_v_pred"]
    assert digest(r["v_actual"]) == g["sha_v_actual"]
    assert digest(r["wall"]) == g["sha_wall"]
    assert digest(r["params"]) == g["sha_params"]
    assert digest(r["loss"]) == g["sha_loss"]


def test_sample_stream_golden(orc, golden):
    for case in golden("stream"):
        s = orc.sample_stream(case["seed"], case["k"], case["budget"], case["N"])
        assert s[:16].tolist() == case["head"]
        assert digest(s.astype(np.int32)) == case["sha"]


# --- against the live reference build (fresh fuzz) -------------------------
def test_restatement_vs_reference_fuzz(orc, ref):
    rng = np.random.default_rng(12345)
    for _ in range(2000):
        n = int(rng.integers(1, 40))
        v = rng.uniform(1e-3, 50.0, n) * (10.0 ** rng.integers(-3, 4))
        b = int(rng.integers(n, 20000))
        assert orc.cpu_allocate(v, b).tolist() == ref.cpu_allocate(v, b).tolist()
    for _ in range(300):
        n = int(rng.integers(1, 20))
        prof, lo, hi = [], 0, 0
        for _i in range(n):
            sat = int(rng.integers(1, 64)); oom = sat + int(rng.integers(0, 500))
            prof.append((float(rng.uniform(1e-4, 0.05)), float(rng.uniform(0, 0.5)), sat, oom))
            lo += sat; hi += oom
        comm = rng.uniform(0, 0.5, n)
        b = int(rng.integers(lo, hi + 1))
        assert orc.gpu_allocate(prof, comm, b).tolist() == ref.gpu_allocate(prof, comm, b).tolist()


def test_replay_driver_vs_reference(orc, ref):
    rng = np.random.default_rng(5)
    iters, n = 120, 6
    c = rng.uniform(0.3, 1.0, (iters, n)); m = np.ones((iters, n))
    v = 10.0 * c * rng.uniform(0.9, 1.1, (iters, n))
    for kind in (abi.PRED_EMA, abi.PRED_NARX, abi.PRED_MEMORYLESS):
        p = abi.PredictorConfig.default(kind, warmup_iterations=40)
        seeds = [orc.mix_seed(1, 0x9ced1c70, i) for i in range(n)]
        s1, v1 = orc.replay_cpu(p, seeds, 1024, v, c, m)
        s2, v2 = ref.replay_cpu(p, seeds, 1024, v, c, m)
        assert s1.tolist() == s2.tolist()
        assert bits_equal(v1, v2)


def test_generalised_narx_reduces_to_reference_at_delay2_hidden1(orc, golden):
    """the (delay, hidden) generalisation used for the C4 sweep
    must reproduce the reference bit-for-bit at (2, 1) before it is trusted."""
    for case in golden("predictor")["narx_train"]:
        seed_model = fromhex(case["model_in"])
        p = np.zeros(orc.narxg_param_count(2, 1))
        p[:8] = seed_model[:8]
        p[8], p[9], p[10] = seed_model[8], seed_model[9], seed_model[10]
        p[11:] = [0.0, 1.0, 0.0, 1.0, 0.0, 1.0]
        cfg = abi.NarxTrainConfig.default(min_history=case["min_history"])
        rep, log = orc.narxg_train(p, 2, 1, fromhex(case["v"]), fromhex(case["c"]),
                                   fromhex(case["m"]), cfg)
        assert rep.epochs == case["epochs"], case["name"]
        out = fromhex(case["model_out"])
        assert bits_equal(p, out), case["name"]
        assert bits_equal(log, fromhex(case["loss_log"])), case["name"]
    # narx_init draw order
    m = orc.narx_init(31)
    p = orc.narxg_init(31, 2, 1)
    assert bits_equal(p[:11], m.weights())
