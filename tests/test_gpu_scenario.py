"""SURVEY 8(f) on the B200: cmd_run with every simulation executed by the
device driver must write files byte-identical to the reference CLI's (golden
fixtures from
oracle/gen_scenario_golden.py), and the device-side compute_metrics and
predictor_series_rmse must match the host / reference bit for bit."""
import hashlib
import json
import os

import numpy as np
import pytest

from paper_1806_02508_b200 import abi
from paper_1806_02508_b200 import lbbsp as L

from test_scenario_cpu import NARX_CSV, TRACE_CSV, materialise, sha, write_config  # noqa: F401

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def sg():
    with open(os.path.join(HERE, "golden", "scenario.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("name", ["homo_smoke", "hetero_l3_bsp", "hetero_l3_lbbsp",
                                  "gpu_cluster", "bench_predictors", "trace_lbbsp_narx",
                                  "trace_bsp", "narx_warm_start", "benchmark_small",
                                  "asp_hetero_narx", "ssp_hetero", "ssp_gpu_cluster",
                                  "asp_trace"])
def test_cmd_run_byte_identical(sg, tmp_path, name):
    cfg = write_config(str(tmp_path), name, sg["configs"][name])
    out = tmp_path / "out"
    assert L.cmd_run(cfg, out) == 0
    g = sg["run"][name]
    lines = (out / "records.csv").read_text().splitlines()
    assert lines[:4] == g["records_head"]
    assert len(lines) == g["records_lines"]
    assert sha(out / "records.csv") == g["records_sha"]
    assert (out / "metrics.json").read_text() == g["metrics_json"]


def test_cmd_run_seed_override(sg, tmp_path):
    g = sg["run_seed77"]
    cfg = write_config(str(tmp_path), g["config"], sg["configs"][g["config"]])
    assert L.cmd_run(cfg, tmp_path / "o", seed_override=77) == 0
    assert sha(tmp_path / "o" / "records.csv") == g["records_sha"]
    assert (tmp_path / "o" / "metrics.json").read_text() == g["metrics_json"]


def test_cmd_run_error_status(tmp_path, capfd):
    cfg = write_config(str(tmp_path), "bad", {"scheme": "bsp", "workers": 4, "colour": 1})
    assert L.cmd_run(cfg, tmp_path / "o") == 1
    assert "lbbsp run: config: unknown field 'colour'" in capfd.readouterr().err


@pytest.mark.parametrize("name", ["hetero_l3_lbbsp", "trace_lbbsp_narx", "gpu_cluster",
                                  "asp_hetero_narx", "ssp_hetero"])
def test_device_metrics_equal_host_compute_metrics(sg, tmp_path, name):
    s = L.load_scenario(write_config(str(tmp_path), name, sg["configs"][name]))
    sim = L.Simulation.from_scenario(s)
    r = sim.run()
    dev = sim.metrics()
    host = L.compute_metrics(r, r.converged, s.info.warmup_iterations)
    assert dev.as_dict() == host.as_dict()


def test_series_rmse_matches_reference(ref):
    """predictor_series_rmse (cluster_sim.cpp:645-672) on device vs the reference."""
    lb = L
    c, m, x = L.make_benchmark_series(21, iterations=600, regime_length=40)
    for kind in (abi.PRED_MEMORYLESS, abi.PRED_EMA, abi.PRED_NARX, abi.PRED_PERFECT):
        base = abi.PredictorConfig.default(kind, warmup_iterations=60)
        got = lb.predictor_series_rmse(kind, base, c, m, x, 10.0, 1234, 60)
        want = ref.series_rmse(kind, base, c, m, x, 10.0, 1234, 60)
        assert got.hex() == want.hex(), kind
