"""ctypes mirror of the C-ABI data layouts in include/lbbsp_c.h.

Pure data layout (no compute). Shared by the product's Python host layer
(paper_1806_02508_b200.lbbsp) and by the test-only oracle bindings
(oracle/oracle.py) so both speak the exact same structs.
"""
import ctypes as C

OK = 0
INVALID_ARGUMENT = -1
OUT_OF_RANGE = -2
RUNTIME = -3
LOGIC = -4
CUDA = -5
NCCL = -6
CONFIG = -7

PRED_MEMORYLESS, PRED_EMA, PRED_NARX, PRED_PERFECT = 0, 1, 2, 3
SCHEME_BSP, SCHEME_ASP, SCHEME_SSP, SCHEME_LBBSP = 0, 1, 2, 3
DYN_STATIC, DYN_STRAGGLER, DYN_BENCHMARK, DYN_TRACE = 0, 1, 2, 3
PRESET_NONE, PRESET_HOMO, PRESET_HETERO_L2, PRESET_HETERO_L3 = -1, 0, 1, 2
PRESET_HETERO_L2_STATIC, PRESET_HETERO_L3_STATIC = 3, 4

PREDICTORS = {"memoryless": PRED_MEMORYLESS, "ema": PRED_EMA, "narx": PRED_NARX,
              "perfect": PRED_PERFECT}
SCHEMES = {"bsp": SCHEME_BSP, "asp": SCHEME_ASP, "ssp": SCHEME_SSP, "lb-bsp": SCHEME_LBBSP,
           "lbbsp": SCHEME_LBBSP}
PRESETS = {"homo": PRESET_HOMO, "hetero-l2": PRESET_HETERO_L2, "hetero-l3": PRESET_HETERO_L3,
           "hetero-l2-static": PRESET_HETERO_L2_STATIC,
           "hetero-l3-static": PRESET_HETERO_L3_STATIC}


class DevStatus(C.Structure):
    _fields_ = [("code", C.c_int), ("what", C.c_int), ("a", C.c_int64), ("b", C.c_int64)]


class GpuProfile(C.Structure):
    """GpuProfile, batch_sizer.hpp:10-15"""
    _fields_ = [("sec_per_sample", C.c_double), ("base_time_s", C.c_double),
                ("saturation_point", C.c_int), ("oom_point", C.c_int)]


class NarxModel(C.Structure):
    """NarxModel, predictor.hpp:49-67 (weights + scalers)"""
    _fields_ = [("input_weights", C.c_double * 8), ("hidden_bias", C.c_double),
                ("output_weight", C.c_double), ("output_bias", C.c_double),
                ("speed_mean", C.c_double), ("speed_stddev", C.c_double),
                ("cpu_mean", C.c_double), ("cpu_stddev", C.c_double),
                ("mem_mean", C.c_double), ("mem_stddev", C.c_double)]

    def weights(self):
        return list(self.input_weights) + [self.hidden_bias, self.output_weight, self.output_bias]

    def as_tuple(self):
        return tuple(self.weights()) + (self.speed_mean, self.speed_stddev, self.cpu_mean,
                                        self.cpu_stddev, self.mem_mean, self.mem_stddev)


class NarxTrainConfig(C.Structure):
    """NarxTrainConfig, predictor.hpp:69-75"""
    _fields_ = [("step", C.c_double), ("max_epochs", C.c_int), ("early_stop_delta", C.c_double),
                ("early_stop_patience", C.c_int), ("min_history", C.c_int)]

    @classmethod
    def default(cls, **kw):
        c = cls(0.05, 500, 1e-4, 4, 500)
        for k, v in kw.items():
            setattr(c, k, v)
        return c


class NarxReport(C.Structure):
    _fields_ = [("ran", C.c_int), ("epochs", C.c_int), ("final_loss", C.c_double)]


class PredictorConfig(C.Structure):
    """PredictorConfig, predictor.hpp:107-114"""
    _fields_ = [("kind", C.c_int), ("alpha", C.c_double), ("warmup_iterations", C.c_int),
                ("speed_floor", C.c_double), ("train", NarxTrainConfig)]

    @classmethod
    def default(cls, kind=PRED_EMA, **kw):
        c = cls(kind, 0.2, 500, 1e-3, NarxTrainConfig.default())
        for k, v in kw.items():
            setattr(c, k, v)
        return c


class Straggler(C.Structure):
    _fields_ = [("on_probability", C.c_double), ("cpu_consumed", C.c_double),
                ("mem_consumed", C.c_double), ("period", C.c_int)]


class SimConfig(C.Structure):
    """lbbsp_sim_cfg == SimConfig (cluster_sim.hpp:165-180) flattened."""
    _fields_ = [
        ("scheme", C.c_int), ("n_workers", C.c_int), ("total_budget", C.c_int),
        ("preset", C.c_int), ("base_speed", C.c_double), ("dynamics", C.c_int),
        ("static_cpu", C.POINTER(C.c_double)), ("static_mem", C.POINTER(C.c_double)),
        ("stragglers", C.POINTER(Straggler)),
        ("bench_iterations", C.c_int), ("bench_regime_length", C.c_int),
        ("bench_high_lo", C.c_double), ("bench_high_hi", C.c_double),
        ("bench_low_lo", C.c_double), ("bench_low_hi", C.c_double),
        ("bench_spike_mult", C.c_double), ("bench_spike_prob", C.c_double),
        ("predictor", PredictorConfig),
        ("gpu_profiles", C.POINTER(GpuProfile)),
        ("base_comm_s", C.c_double), ("bw_worker", C.c_int), ("bw_at_iteration", C.c_int64),
        ("bw_factor", C.c_double),
        ("learning_rate", C.c_double), ("dataset_seed", C.c_uint64), ("dataset_size", C.c_int),
        ("dataset_dim", C.c_int), ("dataset_noise", C.c_double),
        ("convergence_loss", C.c_double), ("convergence_consecutive", C.c_int),
        ("max_updates", C.c_int64), ("seed", C.c_uint64),
        ("trace_offsets", C.POINTER(C.c_int)), ("trace_t", C.POINTER(C.c_double)),
        ("trace_cpu", C.POINTER(C.c_double)), ("trace_mem", C.POINTER(C.c_double)),
        ("narx_weights_path", C.c_char_p), ("staleness_threshold", C.c_int),
    ]


class IterScalars(C.Structure):
    _fields_ = [("k", C.c_int64), ("grad_norm", C.c_double), ("loss", C.c_double),
                ("wall_s", C.c_double)]


class RecordsView(C.Structure):
    """lbbsp_records_view: a host record stream ([rows] scalars, [rows*n] rows)."""
    _fields_ = [("rows", C.c_int), ("n", C.c_int), ("scalars", C.POINTER(IterScalars)),
                ("batch", C.POINTER(C.c_int)), ("tp", C.POINTER(C.c_double)),
                ("tm", C.POINTER(C.c_double)), ("wait", C.POINTER(C.c_double)),
                ("v_pred", C.POINTER(C.c_double)), ("v_actual", C.POINTER(C.c_double)),
                ("worker_id", C.POINTER(C.c_int)), ("row_workers", C.POINTER(C.c_int))]


class Metrics(C.Structure):
    """Metrics, cluster_sim.hpp:157-163"""
    _fields_ = [("updates_to_convergence", C.c_int64), ("mean_per_update_time", C.c_double),
                ("wastage", C.c_double), ("predictor_rmse", C.c_double), ("converged", C.c_int)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class ScenarioInfo(C.Structure):
    """lbbsp_scenario_info: ScenarioConfig scalars (scenario.hpp:33-64)"""
    _fields_ = [("name", C.c_char * 256), ("scheme", C.c_int), ("staleness_threshold", C.c_int),
                ("workers", C.c_int), ("total_budget", C.c_int), ("predictor", C.c_int),
                ("alpha", C.c_double), ("warmup_iterations", C.c_int),
                ("speed_floor", C.c_double), ("base_speed", C.c_double),
                ("base_comm_s", C.c_double), ("learning_rate", C.c_double),
                ("convergence_loss", C.c_double), ("convergence_consecutive", C.c_int),
                ("max_iterations", C.c_int64), ("seed", C.c_uint64), ("paired_sim", C.c_int)]


def make_sim_config(scheme="lb-bsp", workers=4, total_budget=512, preset="hetero-l3",
                    base_speed=10.0, dynamics=DYN_STATIC, static_cpu=None, static_mem=None,
                    stragglers=None, predictor="ema", alpha=0.2, warmup_iterations=500,
                    speed_floor=1e-3, train=None, gpu_profiles=None, base_comm_s=0.0,
                    bandwidth_drop=None, learning_rate=0.5, dataset_seed=7, dataset_size=1000,
                    dataset_dim=10, dataset_noise=0.1, convergence_loss=0.40,
                    convergence_consecutive=10, max_updates=500, seed=1, benchmark=None,
                    traces=None, narx_weights_path=None, staleness_threshold=0):
    """Defaults follow SimConfig (cluster_sim.hpp:165-180) and PredictorConfig
    (predictor.hpp:107-114). Returns (cfg, keepalive) -- keep the second value
    alive while cfg is in use (it owns the pointed-to arrays).
    traces: per-worker list of (t, cpu, mem) point lists (DYN_TRACE)."""
    keep = []
    c = SimConfig()
    c.scheme = SCHEMES[scheme] if isinstance(scheme, str) else scheme
    c.n_workers = workers
    c.total_budget = total_budget
    c.preset = PRESETS[preset] if isinstance(preset, str) else (PRESET_NONE if preset is None else preset)
    c.base_speed = base_speed
    c.dynamics = dynamics
    if static_cpu is not None:
        a = (C.c_double * workers)(*static_cpu); keep.append(a); c.static_cpu = a
    if static_mem is not None:
        a = (C.c_double * workers)(*static_mem); keep.append(a); c.static_mem = a
    if stragglers is not None:
        a = (Straggler * workers)(*[Straggler(*s) for s in stragglers]); keep.append(a)
        c.stragglers = a
    b = dict(iterations=1200, regime_length=50, high_lo=0.75, high_hi=1.0, low_lo=0.30,
             low_hi=0.55, spike_mult=3.0, spike_prob=0.02)
    if benchmark:
        b.update(benchmark)
    c.bench_iterations, c.bench_regime_length = b["iterations"], b["regime_length"]
    c.bench_high_lo, c.bench_high_hi = b["high_lo"], b["high_hi"]
    c.bench_low_lo, c.bench_low_hi = b["low_lo"], b["low_hi"]
    c.bench_spike_mult, c.bench_spike_prob = b["spike_mult"], b["spike_prob"]
    kind = PREDICTORS[predictor] if isinstance(predictor, str) else predictor
    c.predictor = PredictorConfig(kind, alpha, warmup_iterations, speed_floor,
                                  train if train is not None else NarxTrainConfig.default())
    if gpu_profiles is not None:
        a = (GpuProfile * workers)(*[GpuProfile(*g) for g in gpu_profiles]); keep.append(a)
        c.gpu_profiles = a
    c.base_comm_s = base_comm_s
    c.bw_worker = -1
    if bandwidth_drop is not None:
        c.bw_worker, c.bw_at_iteration, c.bw_factor = bandwidth_drop
    c.learning_rate = learning_rate
    c.dataset_seed, c.dataset_size, c.dataset_dim = dataset_seed, dataset_size, dataset_dim
    c.dataset_noise = dataset_noise
    c.convergence_loss, c.convergence_consecutive = convergence_loss, convergence_consecutive
    c.max_updates, c.seed = max_updates, seed
    c.staleness_threshold = staleness_threshold
    if traces is not None:
        off, t, cp, mm = [0], [], [], []
        for pts in traces:
            for (a, b, d) in pts:
                t.append(a); cp.append(b); mm.append(d)
            off.append(len(t))
        arrs = [(C.c_int * len(off))(*off)] + [(C.c_double * max(len(x), 1))(*x)
                                                for x in (t, cp, mm)]
        keep.extend(arrs)
        c.trace_offsets, c.trace_t, c.trace_cpu, c.trace_mem = arrs
    if narx_weights_path:
        b = str(narx_weights_path).encode()
        keep.append(b)
        c.narx_weights_path = b
    return c, keep
