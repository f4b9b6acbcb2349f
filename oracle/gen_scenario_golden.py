"""ORACLE / TEST INFRASTRUCTURE ONLY -- golden fixtures for SURVEY 8(f).

Runs the UNMODIFIED reference CLI entry points (cmd_run / cmd_compare /
cmd_predict_bench, scenario.cpp:369-481, through oracle/_ref) on

  * the reference's own configs/*.json (their contents are embedded as data),
  * a recorded-trace scenario over tests/golden/scenario_trace.csv
    (synthetic, generated here with a fixed seed),
  * a NARX scenario warm-started from tests/golden/scenario_narx_weights.csv,

and records the exact bytes (records.csv as sha256 + row count, metrics.json,
comparison.csv and predict_bench.csv in full) in tests/golden/scenario.json,
together with the reference's error text for malformed configs and traces.

    python oracle/gen_scenario_golden.py      (needs /root/reference)
"""
import glob
import hashlib
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)

from oracle import oracle as O  # noqa: E402

GOLDEN = os.path.join(REPO, "tests", "golden")
TRACE_CSV = os.path.join(GOLDEN, "scenario_trace.csv")
NARX_CSV = os.path.join(GOLDEN, "scenario_narx_weights.csv")
REF_CONFIGS = "/root/reference/proj/configs"

# Extra scenarios (beyond the reference's configs). "@trace" / "@narx" are
# replaced by the absolute fixture paths when the config file is written.
EXTRA = {
    "trace_lbbsp_narx": {"scheme": "lb-bsp", "workers": 4, "total_budget": 512,
                         "trace_path": "@trace", "predictor": "narx", "warmup_iterations": 30,
                         "max_iterations": 200, "convergence_loss": 1e-4, "seed": 5,
                         "base_comm_s": 0.5},
    "trace_bsp": {"scheme": "bsp", "workers": 4, "total_budget": 512, "trace_path": "@trace",
                  "predictor": "ema", "warmup_iterations": 30, "max_iterations": 150,
                  "convergence_loss": 1e-4, "seed": 5},
    "narx_warm_start": {"scheme": "lb-bsp", "workers": 4, "total_budget": 512,
                        "preset": "hetero-l3", "predictor": "narx", "warmup_iterations": 20,
                        "narx_weights_path": "@narx", "max_iterations": 120,
                        "convergence_loss": 1e-4, "seed": 9},
    "benchmark_small": {"scheme": "lb-bsp", "workers": 6, "total_budget": 600,
                        "preset": "benchmark", "predictor": "narx", "warmup_iterations": 40,
                        "benchmark_iterations": 300, "benchmark_regime_length": 30,
                        "benchmark_high_band": [0.7, 0.95], "benchmark_low_band": [0.2, 0.5],
                        "max_iterations": 200, "convergence_loss": 1e-4, "seed": 11,
                        "paired_sim": True},
    # ASP / SSP (Simulation::step_async, cluster_sim.cpp:486-631)
    "asp_hetero_narx": {"scheme": "asp", "workers": 4, "total_budget": 512, "preset": "hetero-l3",
                        "predictor": "narx", "warmup_iterations": 20, "max_iterations": 300,
                        "convergence_loss": 1e-4, "seed": 4},
    "ssp_hetero": {"scheme": "ssp", "staleness_threshold": 2, "workers": 6, "total_budget": 600,
                   "preset": "hetero-l3", "predictor": "ema", "warmup_iterations": 30,
                   "max_iterations": 150, "convergence_loss": 1e-4, "seed": 6},
    "ssp_gpu_cluster": {"scheme": "ssp", "staleness_threshold": 1, "workers": 4,
                        "total_budget": 400, "gpu_profiles": [
                            {"sec_per_sample": 0.002, "base_time_s": 0.05, "saturation_point": 20,
                             "oom_point": 300, "count": 2},
                            {"sec_per_sample": 0.0007, "base_time_s": 0.05,
                             "saturation_point": 30, "oom_point": 400, "count": 2}],
                        "base_comm_s": 0.1,
                        "bandwidth_drop": {"worker": 1, "at_iteration": 40, "comm_factor": 4.0},
                        "max_iterations": 120, "convergence_loss": 1e-4, "seed": 2},
    "asp_trace": {"scheme": "asp", "workers": 4, "total_budget": 256, "trace_path": "@trace",
                  "predictor": "memoryless", "max_iterations": 250, "convergence_loss": 1e-4,
                  "seed": 8, "base_comm_s": 1.0},
}

# Malformed configs: (name, json text or dict); the expected text is the reference's.
BAD_CONFIGS = [
    ("unknown_key", {"scheme": "bsp", "workers": 4, "colour": "red"}),
    ("missing_scheme", {"workers": 4}),
    ("missing_workers", {"scheme": "bsp"}),
    ("bad_scheme", {"scheme": "fast", "workers": 4}),
    ("bad_predictor", {"scheme": "bsp", "workers": 4, "predictor": "oracle"}),
    ("bad_value", {"scheme": "bsp", "workers": "four"}),
    ("budget_small", {"scheme": "bsp", "workers": 4, "total_budget": 3}),
    ("alpha_range", {"scheme": "bsp", "workers": 4, "alpha": 1.5}),
    ("lr_zero", {"scheme": "bsp", "workers": 4, "learning_rate": 0.0}),
    ("consec_zero", {"scheme": "bsp", "workers": 4, "convergence_consecutive": 0}),
    ("max_iter_zero", {"scheme": "bsp", "workers": 4, "max_iterations": 0}),
    ("trace_missing", {"scheme": "bsp", "workers": 4, "trace_path": "/nonexistent/trace.csv"}),
    ("weights_missing", {"scheme": "bsp", "workers": 4,
                         "narx_weights_path": "/nonexistent/w.csv"}),
    ("gpu_counts", {"scheme": "lb-bsp", "workers": 4, "gpu_profiles": [
        {"sec_per_sample": 0.001, "base_time_s": 0.01, "saturation_point": 10,
         "oom_point": 500, "count": 3}]}),
    ("gpu_not_array", {"scheme": "lb-bsp", "workers": 4, "gpu_profiles": {"a": 1}}),
    ("band_len", {"scheme": "bsp", "workers": 4, "benchmark_high_band": [0.1]}),
    ("bw_worker", {"scheme": "bsp", "workers": 4,
                   "bandwidth_drop": {"worker": 7, "at_iteration": 3, "comm_factor": 2.0}}),
    ("not_object", [1, 2, 3]),
    ("invalid_json", "{\"scheme\": \"bsp\", \"workers\": 4,,}"),
]

BAD_TRACES = [
    ("empty", ""),
    ("missing_column", "machine_id,t_offset_s,cpu_avail\nm0,0,1\n"),
    ("column_order", "machine_id,cpu_avail,t_offset_s,mem_avail\nm0,1,0,1\n"),
    ("field_count", "machine_id,t_offset_s,cpu_avail,mem_avail\nm0,0,1\n"),
    ("bad_real", "machine_id,t_offset_s,cpu_avail,mem_avail\nm0,abc,1,1\n"),
    ("trailing_junk", "machine_id,t_offset_s,cpu_avail,mem_avail\nm0,1.5x,1,1\n"),
    ("fraction", "machine_id,t_offset_s,cpu_avail,mem_avail\nm0,0,1.5,1\n"),
    ("unsorted", "machine_id,t_offset_s,cpu_avail,mem_avail\nm0,5,1,1\nm0,2,1,1\n"),
]


def write_trace_fixture():
    """Synthetic leftover-resource traces: 10 machines, 81 points each over
    [0, 9600] s (one LB-BSP round is ~10-55 s of simulated time here)."""
    rng = np.random.default_rng(1806)
    lines = ["machine_id,t_offset_s,cpu_avail,mem_avail"]
    for m in range(10):
        level = rng.uniform(0.25, 1.0)
        for q in range(81):
            t = 120.0 * q
            c = float(np.clip(level + rng.normal(0, 0.12), 0.05, 1.0))
            mem = float(np.clip(rng.uniform(0.3, 1.1), 0.0, 1.0))
            lines.append(f"host-{m:02d},{t:g},{c:.4f},{mem:.4f}")
    # rows of different machines interleaved is legal; keep file order by machine
    with open(TRACE_CSV, "w") as f:
        f.write("\n".join(lines) + "\n")


def write_narx_fixture(orc):
    m = orc.narx_init(4242)
    vals = m.weights()
    names = [f"input_weight_{j}" for j in range(8)] + [
        "hidden_bias", "output_weight", "output_bias", "speed_mean", "speed_stddev",
        "cpu_mean", "cpu_stddev", "mem_mean", "mem_stddev"]
    # scalers from a plausible history so predictions are in range
    vals = list(vals[:11]) + [6.5, 2.0, 0.7, 0.2, 0.8, 0.15]
    with open(NARX_CSV, "w") as f:
        for n, v in zip(names, vals):
            f.write(f"{n},{v!r}\n")


def materialise(cfg):
    out = {}
    for k, v in cfg.items():
        if v == "@trace":
            v = TRACE_CSV
        elif v == "@narx":
            v = NARX_CSV
        out[k] = v
    return out


def write_config(d, name, cfg):
    path = os.path.join(d, name + ".json")
    with open(path, "w") as f:
        if isinstance(cfg, str):
            f.write(cfg)
        else:
            json.dump(materialise(cfg) if isinstance(cfg, dict) else cfg, f, indent=2)
    return path


def sha(path):
    with open(path, "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


def main():
    if not O.reference_available():
        raise SystemExit("oracle/_ref/liblbbsp_ref.so missing: run `make -C oracle`")
    ref, orc = O.reference(), O.restatement()
    write_trace_fixture()
    write_narx_fixture(orc)
    configs = {}
    for p in sorted(glob.glob(os.path.join(REF_CONFIGS, "*.json"))):
        with open(p) as f:
            configs[os.path.splitext(os.path.basename(p))[0]] = json.load(f)
    configs.update(EXTRA)
    out = {"configs": configs, "run": {}, "errors": {}, "trace_errors": {}}
    with tempfile.TemporaryDirectory() as d:
        paths = {name: write_config(d, name, cfg) for name, cfg in configs.items()}
        for name, path in paths.items():
            od = os.path.join(d, "out_" + name)
            rc = ref.cmd_run(path, od)
            assert rc == 0, name
            with open(os.path.join(od, "records.csv")) as f:
                lines = f.read().splitlines()
            with open(os.path.join(od, "metrics.json")) as f:
                metrics = f.read()
            out["run"][name] = {"records_sha": sha(os.path.join(od, "records.csv")),
                                "records_lines": len(lines), "records_head": lines[:4],
                                "records_tail": lines[-2:], "metrics_json": metrics}
            print(name, len(lines), json.loads(metrics)["updates_to_convergence"])
        # seed override
        od = os.path.join(d, "out_seed")
        assert ref.cmd_run(paths["hetero_l3_lbbsp"], od, seed=77) == 0
        out["run_seed77"] = {"config": "hetero_l3_lbbsp",
                             "records_sha": sha(os.path.join(od, "records.csv")),
                             "metrics_json": open(os.path.join(od, "metrics.json")).read()}
        # compare
        cmp_names = ["homo_smoke", "hetero_l3_bsp", "hetero_l3_lbbsp", "gpu_cluster", "trace_bsp",
                     "asp_hetero_narx", "ssp_hetero"]
        od = os.path.join(d, "out_cmp")
        assert ref.cmd_compare([paths[n] for n in cmp_names], od) == 0
        out["compare"] = {"configs": cmp_names,
                          "csv": open(os.path.join(od, "comparison.csv")).read()}
        # predict-bench
        out["predict_bench"] = {}
        for name in ("bench_predictors", "benchmark_small"):
            od = os.path.join(d, "out_pb_" + name)
            assert ref.cmd_predict_bench(paths[name], od) == 0
            out["predict_bench"][name] = open(os.path.join(od, "predict_bench.csv")).read()
            print(out["predict_bench"][name])
        # malformed configs
        for name, cfg in BAD_CONFIGS:
            p = write_config(d, "bad_" + name, cfg)
            msg = ref.scenario_error(p)
            assert msg is not None, name
            out["errors"][name] = {"config": cfg, "message": msg.replace(d, "@dir")}
        for name, text in BAD_TRACES:
            p = os.path.join(d, f"trace_{name}.csv")
            with open(p, "w") as f:
                f.write(text)
            try:
                ref.trace_map(p, 2, 1)
                raise AssertionError(name)
            except Exception as e:  # noqa: BLE001
                out["trace_errors"][name] = {"text": text, "message": str(e).replace(d, "@dir")}
        # map_traces / trace_at on the fixture
        out["trace_map"] = {f"{w}_{s}": ref.trace_map(TRACE_CSV, w, s)
                            for w in (1, 3, 4, 7, 10, 16) for s in (1, 5, 99)}
        out["trace_at"] = [[i, t, *ref.trace_at(TRACE_CSV, i, t)]
                           for i in (0, 3, 9) for t in (-5.0, 0.0, 119.9, 120.0, 1234.5, 99999.0)]
    with open(os.path.join(GOLDEN, "scenario.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("wrote", os.path.join(GOLDEN, "scenario.json"))


if __name__ == "__main__":
    main()
