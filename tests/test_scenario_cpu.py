"""SURVEY 8(f) host path on CPU: the scenario loader, trace ingest, metrics and
exporters of the product library (host code, no kernels) against golden
fixtures made by the UNMODIFIED reference CLI (oracle/gen_scenario_golden.py).

The record streams here come from the C restatement (orc_sim_run) fed with
the config the product's loader built; the same files produced from the
device driver are checked in tests/test_gpu_scenario.py."""
import hashlib
import json
import os

import numpy as np
import pytest

from paper_1806_02508_b200 import abi
from paper_1806_02508_b200 import lbbsp as L
from paper_1806_02508_b200.errors import ConfigError, RuntimeFailure

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN_DIR = os.path.join(HERE, "golden")
TRACE_CSV = os.path.join(GOLDEN_DIR, "scenario_trace.csv")
NARX_CSV = os.path.join(GOLDEN_DIR, "scenario_narx_weights.csv")


@pytest.fixture(scope="module")
def sg():
    with open(os.path.join(GOLDEN_DIR, "scenario.json")) as f:
        return json.load(f)


def materialise(cfg):
    if not isinstance(cfg, dict):
        return cfg
    return {k: (TRACE_CSV if v == "@trace" else NARX_CSV if v == "@narx" else v)
            for k, v in cfg.items()}


def write_config(d, name, cfg):
    p = os.path.join(d, name + ".json")
    with open(p, "w") as f:
        if isinstance(cfg, str):
            f.write(cfg)
        else:
            json.dump(materialise(cfg), f, indent=2)
    return p


def sha(path):
    with open(path, "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


def result_from_oracle(r):
    return L.SimResult(k=r["k"], loss=r["loss"], grad_norm=r["grad_norm"], wall=r["wall"],
                       batch=r["batch"], tp=r["tp"], tm=r["tm"], wait=r["wait"],
                       v_pred=r["v_pred"], v_actual=r["v_actual"], params=r["params"],
                       converged=r["converged"], worker_id=r.get("worker_id"),
                       row_workers=r.get("row_workers"))


def test_config_errors_match_reference(sg, tmp_path):
    for name, case in sg["errors"].items():
        p = write_config(str(tmp_path), "bad_" + name, case["config"])
        with pytest.raises(ConfigError) as ei:
            L.load_scenario(p)
        assert str(ei.value) == case["message"].replace("@dir", str(tmp_path)), name
    assert issubclass(ConfigError, RuntimeError)  # ConfigError : std::runtime_error


def test_config_fields_and_defaults(sg, tmp_path):
    s = L.load_scenario(write_config(str(tmp_path), "gpu_cluster", sg["configs"]["gpu_cluster"]))
    i = s.info
    assert i.name == b"gpu_cluster" and i.workers == 8 and i.total_budget == 3040
    assert i.scheme == abi.SCHEME_LBBSP and i.predictor == abi.PRED_EMA
    c = s.sim_config()
    assert [c.gpu_profiles[k].oom_point for k in range(8)] == [384] * 4 + [1184] * 2 + [788] * 2
    assert (c.bw_worker, c.bw_at_iteration, c.bw_factor) == (0, 150, 3.0)
    assert c.base_comm_s == 0.1 and c.predictor.train.min_history == 50
    # defaults (scenario.cpp:112-141)
    s = L.load_scenario(write_config(str(tmp_path), "minimal", {"scheme": "bsp", "workers": 3}))
    i = s.info
    assert (i.total_budget, i.warmup_iterations, i.alpha, i.max_iterations, i.seed) == \
        (384, 500, 0.2, 500, 1)
    assert i.paired_sim == 1 and i.convergence_loss == 0.40
    # presets are resolved when the simulation is built, with the reference's wording
    s = L.load_scenario(write_config(str(tmp_path), "p", {"scheme": "bsp", "workers": 3,
                                                          "preset": "weird"}))
    with pytest.raises(ConfigError, match="config: field 'preset': unknown preset: weird"):
        s.sim_config()
    # ASP / SSP carry the staleness threshold into the simulation config
    s = L.load_scenario(write_config(str(tmp_path), "a", {"scheme": "ssp", "workers": 4,
                                                          "staleness_threshold": 3}))
    c = s.sim_config()
    assert (c.scheme, c.staleness_threshold) == (abi.SCHEME_SSP, 3)


def test_trace_errors_match_reference(sg, tmp_path):
    for name, case in sg["trace_errors"].items():
        p = tmp_path / f"trace_{name}.csv"
        p.write_text(case["text"])
        with pytest.raises(RuntimeFailure) as ei:
            L.parse_trace(p)
        assert str(ei.value) == case["message"].replace("@dir", str(tmp_path)), name


def test_trace_map_and_lookup_match_reference(sg):
    traces = L.parse_trace(TRACE_CSV)
    assert len(traces) == 10 and all(len(t.points) == 81 for t in traces)
    for key, want in sg["trace_map"].items():
        w, s = map(int, key.split("_"))
        assert L.map_traces(traces, w, s) == want, key
    for i, t, c, m in sg["trace_at"]:
        assert L.trace_at(traces[i], t) == (c, m)


def test_trace_write_roundtrip(tmp_path):
    traces = L.parse_trace(TRACE_CSV)
    out = tmp_path / "t.csv"
    L.write_trace(traces, out)
    back = L.parse_trace(out)
    assert [(t.machine_id, t.points) for t in back] == [(t.machine_id, t.points) for t in traces]


def test_narx_csv_roundtrip(tmp_path, orc):
    m = L.load_narx_csv(NARX_CSV)
    assert m.speed_mean == 6.5 and m.mem_stddev == 0.15
    p = tmp_path / "w.csv"
    L.save_narx_csv(m, p)
    m2 = L.load_narx_csv(p)
    assert m2.as_tuple() == m.as_tuple()
    (tmp_path / "bad.csv").write_text("hidden_bias,1.0\n")
    with pytest.raises(RuntimeFailure, match="missing parameter 'input_weight_0'"):
        L.load_narx_csv(tmp_path / "bad.csv")


@pytest.mark.parametrize("name", ["homo_smoke", "hetero_l3_bsp", "hetero_l3_lbbsp",
                                  "gpu_cluster", "bench_predictors", "trace_lbbsp_narx",
                                  "trace_bsp", "narx_warm_start", "benchmark_small",
                                  "asp_hetero_narx", "ssp_hetero", "ssp_gpu_cluster",
                                  "asp_trace"])
def test_exported_files_byte_identical(sg, orc, tmp_path, name):
    """cmd_run's outputs (records.csv, metrics.json) rebuilt from the product's
    loader + build_sim_config + exporters over the restatement's record stream
    must be byte-identical to the reference CLI's."""
    s = L.load_scenario(write_config(str(tmp_path), name, sg["configs"][name]))
    info = s.info
    r = result_from_oracle(orc.sim_run(s.sim_config()))
    L.write_records_csv(r, tmp_path / "records.csv")
    m = L.compute_metrics(r, r.converged, info.warmup_iterations, rounded=True)
    L.write_metrics_json(m, info.convergence_loss, info.convergence_consecutive,
                         info.warmup_iterations, tmp_path / "metrics.json")
    g = sg["run"][name]
    lines = (tmp_path / "records.csv").read_text().splitlines()
    assert lines[:4] == g["records_head"] and lines[-2:] == g["records_tail"]
    assert len(lines) == g["records_lines"]
    assert sha(tmp_path / "records.csv") == g["records_sha"]
    assert (tmp_path / "metrics.json").read_text() == g["metrics_json"]


def test_compare_rows_match_reference(sg, orc, tmp_path):
    """The reference's comparison.csv rows (cmd_compare, scenario.cpp:388-423)
    are the unrounded Simulation::run metrics, which compute_metrics gives."""
    rows = ["scenario,metric,value"]
    for name in sg["compare"]["configs"]:
        s = L.load_scenario(write_config(str(tmp_path), name, sg["configs"][name]))
        r = result_from_oracle(orc.sim_run(s.sim_config()))
        m = L.compute_metrics(r, r.converged, s.info.warmup_iterations)
        for key, v in (("updates_to_convergence", float(m.updates_to_convergence)),
                       ("mean_per_update_time", m.mean_per_update_time),
                       ("wastage", m.wastage), ("predictor_rmse", m.predictor_rmse),
                       ("converged", 1.0 if m.converged else 0.0)):
            rows.append(f"{name},{key},{v:.9g}")
    assert "\n".join(rows) + "\n" == sg["compare"]["csv"]


def test_metrics_recomputable_from_records(sg, orc, tmp_path):
    """test_scenario.cpp:135-172: metrics.json is recomputable from records.csv."""
    name = "trace_lbbsp_narx"
    s = L.load_scenario(write_config(str(tmp_path), name, sg["configs"][name]))
    r = result_from_oracle(orc.sim_run(s.sim_config()))
    L.write_records_csv(r, tmp_path / "records.csv")
    m = L.compute_metrics(r, r.converged, s.info.warmup_iterations, rounded=True)
    rows = np.genfromtxt(tmp_path / "records.csv", delimiter=",", names=True)
    walls = {}
    wf, sse, cnt = 0.0, 0.0, 0
    for row in rows:
        walls[int(row["k"])] = row["iter_wall_s"]
        wf += row["wait_s"] / row["iter_wall_s"] if row["iter_wall_s"] > 0 else 0.0
        if row["v_pred"] > 0 and row["k"] >= s.info.warmup_iterations:
            sse += (row["v_pred"] - row["v_actual"]) ** 2
            cnt += 1
    assert m.updates_to_convergence == len(walls)
    assert abs(m.mean_per_update_time - sum(walls.values()) / len(walls)) < 1e-9
    assert abs(m.wastage - wf / len(rows)) < 1e-9
    assert abs(m.predictor_rmse - (sse / cnt) ** 0.5) < 1e-9


def test_recorded_trace_drives_the_mlp_engine_schedule(sg):
    """The MLP engine's straggler input from a trace CSV (map_traces + trace_at
    at iteration-indexed times) matches the reference's mapping and lookup."""
    from paper_1806_02508_b200.mlp import recorded_trace
    c, m, x = recorded_trace(TRACE_CSV, 4, 30, seed=5, seconds_per_iteration=120.0)
    traces = L.parse_trace(TRACE_CSV)
    assign = sg["trace_map"]["4_5"]
    for i in range(4):
        for k in (0, 7, 29):
            assert (c[i, k], m[i, k]) == L.trace_at(traces[assign[i]], 120.0 * k)
    assert (x == 1.0).all() and c.shape == (4, 30)
