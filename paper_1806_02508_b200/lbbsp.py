"""Python host layer that mirrors the reference C++ API of the LB-BSP hot path
(/root/reference/proj/core/include/lbbsp/*.hpp) on top of the B200 C-ABI.

Same names, argument meaning and error behaviour as the reference, so the
parity tests read like the reference's own doctest suites. Every numeric
result comes from an sm_100a kernel in liblbbsp_b200.so; this module only
marshals arguments and maps status codes to the reference exception types.
"""
import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import abi
from ._lib import check, lib
from .abi import (GpuProfile, NarxModel, NarxReport, NarxTrainConfig, PredictorConfig,
                  make_sim_config)
from .errors import InvalidArgument, LogicError, OutOfRange, RuntimeFailure  # noqa: F401

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


def _d(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(_dp)


# --------------------------------------------------------------------------
# batch_sizer.hpp
# --------------------------------------------------------------------------
@dataclass
class BatchAssignment:
    """BatchAssignment, batch_sizer.hpp:17-20"""
    sizes: List[int]
    total_budget: int


def cpu_allocate(speeds: Sequence[float], total_budget: int) -> BatchAssignment:
    """cpu_allocate (batch_sizer.cpp:54-99) -> K1 single-block kernel."""
    v, vp = _d(speeds)
    out = np.zeros(max(len(v), 1), np.int32)
    check(lib().lbbsp_cpu_allocate(vp, len(v), int(total_budget), out.ctypes.data_as(_ip)))
    return BatchAssignment([int(x) for x in out[: len(v)]], int(total_budget))


def gpu_allocate(profiles, comm_s, total_budget: int) -> BatchAssignment:
    """gpu_allocate (batch_sizer.cpp:101-199) -> K2 single-block kernel."""
    n = len(profiles)
    arr = (GpuProfile * max(n, 1))(*[p if isinstance(p, GpuProfile) else GpuProfile(*p)
                                     for p in profiles])
    c, cp = _d(comm_s)
    out = np.zeros(max(n, 1), np.int32)
    check(lib().lbbsp_gpu_allocate(arr, cp, n, int(total_budget), out.ctypes.data_as(_ip)))
    return BatchAssignment([int(x) for x in out[:n]], int(total_budget))


def clamp_speed_floor(speed: float, floor: float = 1e-3) -> float:
    """clamp_speed_floor (batch_sizer.cpp:12-14). On the device path this is
    fused into the solver kernel (lbbsp_solve_prop's speed_floor)."""
    return speed if speed > floor else floor


def cpu_makespan(speeds, a: BatchAssignment) -> float:
    """cpu_makespan (batch_sizer.cpp:288-293), a host-side test metric."""
    return max(x / v for x, v in zip(a.sizes, speeds))


def gpu_makespan(profiles, comm_s, a: BatchAssignment) -> float:
    """gpu_makespan (batch_sizer.cpp:295-301), a host-side test metric."""
    ps = [p if isinstance(p, GpuProfile) else GpuProfile(*p) for p in profiles]
    return max(p.sec_per_sample * max(x, p.saturation_point) + p.base_time_s + c
               for p, c, x in zip(ps, comm_s, a.sizes))


# --------------------------------------------------------------------------
# predictor.hpp
# --------------------------------------------------------------------------
class SpeedHistory:
    """SpeedHistory, predictor.hpp:15-26"""

    def __init__(self):
        self.speed: List[float] = []
        self.cpu_avail: List[float] = []
        self.mem_avail: List[float] = []

    def push(self, v, c, m):
        self.speed.append(float(v))
        self.cpu_avail.append(float(c))
        self.mem_avail.append(float(m))

    def size(self):
        return len(self.speed)

    __len__ = size


def ema(series, alpha: float) -> float:
    """ema (predictor.cpp:18-25) evaluated by the device kernel."""
    s, sp = _d(series)
    out = C.c_double()
    check(lib().lbbsp_ema(sp, len(s), float(alpha), C.byref(out)))
    return out.value


def predict_memoryless(history: SpeedHistory) -> float:
    """predict_memoryless (predictor.cpp:13-16)"""
    if history.size() == 0:
        raise InvalidArgument("predict_memoryless: empty history")
    return history.speed[-1]


def predict_ema(history: SpeedHistory, alpha: float) -> float:
    return ema(history.speed, alpha)


def predict_comm_ema(comm_s, alpha: float) -> float:
    return ema(comm_s, alpha)


class Narx(NarxModel):
    """NarxModel (predictor.hpp:49-67) plus its training_loss log."""
    kSpeedLags, kCpuWindow, kMemWindow, kInputs = 2, 3, 3, 8

    @staticmethod
    def parameter_count():
        return 11

    def __init__(self, *a, **kw):
        super().__init__(*a, **kw)
        self.training_loss: List[float] = []
        if not a and not kw:
            self.output_weight = 1.0
            self.speed_stddev = self.cpu_stddev = self.mem_stddev = 1.0

    def copy(self):
        m = Narx()
        C.memmove(C.byref(m), C.byref(self), C.sizeof(NarxModel))
        m.training_loss = list(self.training_loss)
        return m


def narx_init(seed: int) -> Narx:
    m = Narx()
    check(lib().lbbsp_narx_init(C.c_uint64(seed), C.cast(C.byref(m), C.POINTER(NarxModel))))
    return m


def narx_predict(model: NarxModel, recent_speeds, cpu_window, mem_window,
                 floor: float = 1e-3) -> float:
    """narx_predict (predictor.cpp:147-153) -> K4 kernel."""
    v, vp = _d(recent_speeds); c, cp = _d(cpu_window); m, mp = _d(mem_window)
    out = C.c_double()
    check(lib().lbbsp_narx_predict(C.cast(C.byref(model), C.POINTER(NarxModel)), vp, cp, mp,
                                   float(floor), C.byref(out)))
    return out.value


def glibc_tanh(xs) -> np.ndarray:
    """The device restatement of glibc tanh (exactmath.cuh) over an array."""
    x = np.ascontiguousarray(xs, dtype=np.float64)
    y = np.empty_like(x)
    check(lib().lbbsp_glibc_tanh(x.ctypes.data_as(C.POINTER(C.c_double)),
                                 y.ctypes.data_as(C.POINTER(C.c_double)), x.size))
    return y


@dataclass
class NarxTrainReport:
    ran: bool = False
    epochs: int = 0
    final_loss: float = 0.0


def narx_train_online(model: Narx, history: SpeedHistory,
                      cfg: Optional[NarxTrainConfig] = None) -> NarxTrainReport:
    """narx_train_online (predictor.cpp:155-196) -> K5 bit-exact fp64 kernel.
    Mutates `model` (weights, scalers) and appends to model.training_loss."""
    cfg = cfg if cfg is not None else NarxTrainConfig.default()
    v, vp = _d(history.speed); c, cp = _d(history.cpu_avail); m, mp = _d(history.mem_avail)
    rep = NarxReport()
    log = np.zeros(max(cfg.max_epochs, 1))
    check(lib().lbbsp_narx_train_online(C.cast(C.byref(model), C.POINTER(NarxModel)), vp, cp, mp,
                                        len(v), C.byref(cfg), C.byref(rep),
                                        log.ctypes.data_as(_dp)))
    if hasattr(model, "training_loss"):
        model.training_loss.extend(float(x) for x in log[: rep.epochs])
    return NarxTrainReport(bool(rep.ran), rep.epochs, rep.final_loss)


class SpeedPredictor:
    """SpeedPredictor (predictor.hpp:118-136 / predictor.cpp:257-297)."""

    def __init__(self, cfg: PredictorConfig, seed: int, initial: Optional[Narx] = None):
        self.cfg = PredictorConfig(cfg.kind, cfg.alpha, cfg.warmup_iterations, cfg.speed_floor,
                                   cfg.train)
        self.cfg.train.min_history = self.cfg.warmup_iterations  # predictor.cpp:264
        self.model_ = initial.copy() if initial is not None else narx_init(seed)

    def predict(self, history: SpeedHistory, cpu_now: float, mem_now: float) -> float:
        k = history.size()
        kind = self.cfg.kind
        if kind == abi.PRED_MEMORYLESS:
            return predict_memoryless(history)
        if kind in (abi.PRED_EMA, abi.PRED_PERFECT):
            return predict_ema(history, self.cfg.alpha)
        if k < self.cfg.warmup_iterations or k < 2:
            return predict_ema(history, self.cfg.alpha)
        return narx_predict(self.model_, [history.speed[-1], history.speed[-2]],
                            [cpu_now, history.cpu_avail[-1], history.cpu_avail[-2]],
                            [mem_now, history.mem_avail[-1], history.mem_avail[-2]],
                            self.cfg.speed_floor)

    def train(self, history: SpeedHistory) -> NarxTrainReport:
        if self.cfg.kind != abi.PRED_NARX:
            return NarxTrainReport()
        return narx_train_online(self.model_, history, self.cfg.train)

    def model(self):
        return self.model_


# --------------------------------------------------------------------------
# sgd.hpp / coordination.hpp  (reference logistic-regression workload)
# --------------------------------------------------------------------------
class Dataset:
    """Dataset (sgd.hpp:15-21) resident in device memory."""

    def __init__(self, handle, n, d):
        self._h = handle
        self.n = n
        self.dim = d

    def size(self):
        return self.n

    def __del__(self):
        try:
            if self._h:
                lib().lbbsp_lr_data_destroy(self._h)
        except Exception:
            pass


def generate_dataset(seed: int, n: int, d: int, noise_amplitude: float = 0.2) -> Dataset:
    h = C.c_void_p()
    check(lib().lbbsp_lr_data_create(C.c_uint64(seed), n, d, float(noise_amplitude), C.byref(h)))
    return Dataset(h, n, d)


def upload_dataset(features, labels) -> Dataset:
    f, fp = _d(features); l, lp = _d(labels)
    h = C.c_void_p()
    check(lib().lbbsp_lr_data_upload(fp, lp, f.shape[0], f.shape[1], C.byref(h)))
    return Dataset(h, f.shape[0], f.shape[1])


@dataclass
class ModelState:
    """ModelState, sgd.hpp:23-27"""
    params: List[float]
    learning_rate: float = 0.1
    clock: int = 0


@dataclass
class Gradient:
    """Gradient, sgd.hpp:29-32"""
    values: List[float]
    batch_size: int = 0


def batch_gradient(model: ModelState, data: Dataset, indices) -> Gradient:
    """batch_gradient (sgd.cpp:72-90) -> K7 kernel."""
    p, pp = _d(model.params)
    idx = np.ascontiguousarray(indices, dtype=np.int32)
    out = np.zeros(data.dim)
    check(lib().lbbsp_batch_gradient(data._h, pp, idx.ctypes.data_as(_ip), len(idx),
                                      out.ctypes.data_as(_dp)))
    return Gradient(out.tolist(), len(idx))


def loss(model: ModelState, data: Dataset) -> float:
    """loss (sgd.cpp:65-70) -> K10 kernel."""
    p, pp = _d(model.params)
    out = C.c_double()
    check(lib().lbbsp_loss(data._h, pp, C.byref(out)))
    return out.value


def _check_dims(grads):
    if len(grads) == 0:
        raise InvalidArgument("aggregate: empty gradient list")
    dim = len(grads[0].values)
    for g in grads:
        if len(g.values) != dim:
            raise InvalidArgument("aggregate: gradient dimension mismatch")
    return dim


def _aggregate(grads, weighted):
    dim = _check_dims(grads)
    g = np.array([gr.values for gr in grads], dtype=np.float64)
    sizes = np.array([gr.batch_size for gr in grads], dtype=np.int32)
    out = np.zeros(dim)
    check(lib().lbbsp_aggregate(g.ctypes.data_as(_dp), sizes.ctypes.data_as(_ip), len(grads), dim,
                                1 if weighted else 0, out.ctypes.data_as(_dp)))
    return Gradient(out.tolist(), int(sizes.sum()))


def aggregate_weighted(grads) -> Gradient:
    """aggregate_weighted (coordination.cpp:52-68) -> K8 kernel."""
    return _aggregate(grads, True)


def aggregate_naive(grads) -> Gradient:
    """aggregate_naive (coordination.cpp:39-50) -> K8 kernel."""
    return _aggregate(grads, False)


def apply_update(model: ModelState, g: Gradient) -> ModelState:
    """apply_update (sgd.cpp:92-99): params -= lr * g on device (K9)."""
    if len(g.values) != len(model.params):
        raise InvalidArgument("apply_update: gradient dimension mismatch")
    import torch
    p = torch.tensor(model.params, dtype=torch.float64, device="cuda")
    gr = torch.tensor([g.values], dtype=torch.float64, device="cuda")
    sz = torch.tensor([max(g.batch_size, 1)], dtype=torch.int32, device="cuda")
    st = torch.zeros(4, dtype=torch.int64, device="cuda")
    check(lib().lbbsp_aggregate_apply(gr.data_ptr(), sz.data_ptr(), 1, len(model.params), 0,
                                      float(model.learning_rate), p.data_ptr(), None, None,
                                      st.data_ptr(), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    return ModelState(p.cpu().tolist(), model.learning_rate, model.clock + 1)


@dataclass
class SchemeConfig:
    """SchemeConfig, coordination.hpp:15-19"""
    kind: int = abi.SCHEME_BSP
    staleness_threshold: int = 0
    total_budget: int = 0


@dataclass
class PendingUpdate:
    """PendingUpdate, coordination.hpp:21-25"""
    worker_id: int
    gradient: Gradient
    worker_clock: int = 0


def ps_step(scheme: SchemeConfig, worker_count: int, model: ModelState, ready) -> ModelState:
    """ps_step (coordination.cpp:75-114), BSP / LB-BSP branch. The
    one-update-per-worker validation is a host-side precondition; the
    aggregation and update run on device."""
    if len(ready) == 0:
        raise InvalidArgument("ps_step: no pending updates")
    if scheme.kind in (abi.SCHEME_ASP, abi.SCHEME_SSP):
        raise InvalidArgument("ps_step: only the synchronous bsp / lb-bsp schemes are on the "
                              "B200 hot path")
    seen = [0] * worker_count
    for u in ready:
        if u.worker_id < 0 or u.worker_id >= worker_count:
            raise InvalidArgument(f"ps_step: unknown worker id {u.worker_id}")
        if seen[u.worker_id]:
            raise InvalidArgument(f"ps_step: duplicate update from worker {u.worker_id}")
        seen[u.worker_id] = 1
    if len(ready) != worker_count:
        raise InvalidArgument(f"ps_step: missing worker update (got {len(ready)} of {worker_count})")
    grads = [u.gradient for u in ready]
    agg = aggregate_weighted(grads) if scheme.kind == abi.SCHEME_LBBSP else aggregate_naive(grads)
    return apply_update(model, agg)


# --------------------------------------------------------------------------
# cluster_sim.hpp: the fused iteration driver
# --------------------------------------------------------------------------
@dataclass
class SimResult:
    """SimResult (cluster_sim.hpp:182-188) as arrays: per-iteration scalars
    and [rows, n] per-worker stats."""
    k: np.ndarray
    loss: np.ndarray
    grad_norm: np.ndarray
    wall: np.ndarray
    batch: np.ndarray
    tp: np.ndarray
    tm: np.ndarray
    wait: np.ndarray
    v_pred: np.ndarray
    v_actual: np.ndarray
    params: np.ndarray
    converged: bool = False
    extra: dict = field(default_factory=dict)
    worker_id: Optional[np.ndarray] = None    # [rows, n] worker of each slot (ASP: slot 0)
    row_workers: Optional[np.ndarray] = None  # [rows] stats per record (ASP: 1)


class Simulation:
    """Simulation (cluster_sim.hpp:197-258) for the BSP / LB-BSP schemes,
    every round executed on device (lbbsp_sim_run) with no host round trip."""

    def __init__(self, cfg=None, **kw):
        if cfg is None:
            cfg, keep = make_sim_config(**kw)
        else:
            keep = None
        self._keep = keep
        self.cfg = cfg
        h = C.c_void_p()
        check(lib().lbbsp_sim_create(C.byref(cfg), C.byref(h)))
        self._h = h

    def __del__(self):
        try:
            if self._h:
                lib().lbbsp_sim_destroy(self._h)
        except Exception:
            pass

    def launches_per_iteration(self):
        x = C.c_int()
        check(lib().lbbsp_sim_launches_per_iteration(self._h, C.byref(x)))
        return x.value

    def run_rounds(self, iterations, stream=None):
        check(lib().lbbsp_sim_run(self._h, int(iterations), stream))

    def status(self):
        done, conv = C.c_int(), C.c_int()
        check(lib().lbbsp_sim_status(self._h, C.byref(done), C.byref(conv)))
        return bool(done.value), bool(conv.value)

    def records(self) -> SimResult:
        n, d = self.cfg.n_workers, self.cfg.dataset_dim
        cap = int(self.cfg.max_updates)
        sc = (abi.IterScalars * cap)()
        arr = {k: np.zeros(cap * n) for k in ("tp", "tm", "wait", "v_pred", "v_actual")}
        batch = np.zeros(cap * n, np.int32)
        params = np.zeros(cap * d)
        rows = C.c_int()
        check(lib().lbbsp_sim_records(self._h, cap, C.byref(rows), sc, batch.ctypes.data_as(_ip),
                                      *[arr[k].ctypes.data_as(_dp) for k in
                                        ("tp", "tm", "wait", "v_pred", "v_actual")],
                                      params.ctypes.data_as(_dp)))
        r = rows.value
        wid = np.zeros(cap * n, np.int32)
        nw = np.zeros(cap, np.int32)
        check(lib().lbbsp_sim_record_workers(self._h, cap, wid.ctypes.data_as(_ip),
                                             nw.ctypes.data_as(_ip)))
        done, conv = self.status()
        return SimResult(worker_id=wid[: r * n].reshape(r, n), row_workers=nw[:r].copy(),
                         k=np.array([sc[i].k for i in range(r)]),
                         loss=np.array([sc[i].loss for i in range(r)]),
                         grad_norm=np.array([sc[i].grad_norm for i in range(r)]),
                         wall=np.array([sc[i].wall_s for i in range(r)]),
                         batch=batch[: r * n].reshape(r, n),
                         **{k: v[: r * n].reshape(r, n) for k, v in arr.items()},
                         params=params[: r * d].reshape(r, d), converged=conv)

    def run(self) -> SimResult:
        """Simulation::run (cluster_sim.cpp:633-643): all rounds on device."""
        self.run_rounds(int(self.cfg.max_updates))
        return self.records()

    def summary(self):
        """(SimResult::total_time_s, max_ssp_skew) (cluster_sim.cpp:633-643)"""
        t, k = C.c_double(), C.c_int64()
        check(lib().lbbsp_sim_summary(self._h, C.byref(t), C.byref(k)))
        return t.value, k.value

    def metrics(self) -> abi.Metrics:
        """SimResult::metrics = compute_metrics(records, converged, warmup)
        (cluster_sim.cpp:638), computed on device from the resident records."""
        m = abi.Metrics()
        check(lib().lbbsp_sim_metrics(self._h, int(self.cfg.predictor.warmup_iterations),
                                      C.byref(m)))
        return m

    @classmethod
    def from_scenario(cls, scenario: "Scenario") -> "Simulation":
        """Simulation(build_sim_config(cfg)) (scenario.cpp:219-304)."""
        sim = cls(scenario.sim_config())
        sim._scenario = scenario  # the config's arrays live in the scenario
        return sim


# --------------------------------------------------------------------------
# Records, metrics and exporters (cluster_sim.cpp:217-245, scenario.cpp:60-358)
# --------------------------------------------------------------------------
def _records_view(r: SimResult):
    rows, n = r.batch.shape
    sc = (abi.IterScalars * max(rows, 1))(*[abi.IterScalars(int(r.k[i]), float(r.grad_norm[i]),
                                                            float(r.loss[i]), float(r.wall[i]))
                                            for i in range(rows)])
    keep = [sc]
    arrs = []
    for name in ("tp", "tm", "wait", "v_pred", "v_actual"):
        a = np.ascontiguousarray(getattr(r, name), dtype=np.float64).reshape(-1)
        keep.append(a)
        arrs.append(a.ctypes.data_as(_dp))
    b = np.ascontiguousarray(r.batch, dtype=np.int32).reshape(-1)
    keep.append(b)
    ids = [None, None]
    for q, a in enumerate((r.worker_id, r.row_workers)):
        if a is not None:
            a = np.ascontiguousarray(a, dtype=np.int32).reshape(-1)
            keep.append(a)
            ids[q] = a.ctypes.data_as(_ip)
    v = abi.RecordsView(rows, n, sc, b.ctypes.data_as(_ip), *arrs, *ids)
    return v, keep


def compute_metrics(records: SimResult, converged: bool, rmse_from_iteration: int,
                    rounded: bool = False) -> abi.Metrics:
    """compute_metrics (cluster_sim.cpp:217-245); rounded=True applies the
    exporter's 9-significant-digit rounding first (scenario.cpp:66-88)."""
    v, keep = _records_view(records)
    m = abi.Metrics()
    check(lib().lbbsp_compute_metrics(C.byref(v), int(bool(converged)), int(rmse_from_iteration),
                                      int(bool(rounded)), C.byref(m)))
    return m


def write_records_csv(records: SimResult, path) -> None:
    """write_records_csv (scenario.cpp:306-342)."""
    v, keep = _records_view(records)
    check(lib().lbbsp_write_records_csv(C.byref(v), str(path).encode()))


def write_metrics_json(metrics: abi.Metrics, convergence_loss: float, convergence_consecutive: int,
                       warmup_iterations: int, path) -> None:
    """write_metrics_json (scenario.cpp:344-358)."""
    check(lib().lbbsp_write_metrics_json(C.byref(metrics), float(convergence_loss),
                                         int(convergence_consecutive), int(warmup_iterations),
                                         str(path).encode()))


# --------------------------------------------------------------------------
# trace.hpp: recorded resource traces
# --------------------------------------------------------------------------
@dataclass
class ResourceTrace:
    """ResourceTrace (trace.hpp:18-24): points as (t_offset_s, cpu, mem)."""
    machine_id: str
    points: list

    def mean_cpu(self) -> float:
        s = 0.0
        for p in self.points:
            s += p[1]
        return s / len(self.points) if self.points else 0.0


class _Traces:
    def __init__(self, h):
        self._h = h

    def __del__(self):
        try:
            lib().lbbsp_trace_destroy(self._h)
        except Exception:
            pass

    @classmethod
    def parse(cls, path):
        h = C.c_void_p()
        check(lib().lbbsp_trace_parse(str(path).encode(), C.byref(h)))
        return cls(h)

    @classmethod
    def from_list(cls, traces: Sequence[ResourceTrace]):
        ids = (C.c_char_p * max(len(traces), 1))(*[t.machine_id.encode() for t in traces])
        off = [0]
        for t in traces:
            off.append(off[-1] + len(t.points))
        pts = [p for t in traces for p in t.points]
        cols = [np.array([p[j] for p in pts] or [0.0]) for j in range(3)]
        o = np.array(off, np.int32)
        h = C.c_void_p()
        check(lib().lbbsp_trace_create(len(traces), ids, o.ctypes.data_as(_ip),
                                       *[c.ctypes.data_as(_dp) for c in cols], C.byref(h)))
        return cls(h)

    def to_list(self):
        n = C.c_int()
        check(lib().lbbsp_trace_count(self._h, C.byref(n)))
        out = []
        for i in range(n.value):
            mid, cnt, mean = C.c_char_p(), C.c_int(), C.c_double()
            check(lib().lbbsp_trace_info(self._h, i, C.byref(mid), C.byref(cnt), C.byref(mean)))
            cols = [np.zeros(max(cnt.value, 1)) for _ in range(3)]
            check(lib().lbbsp_trace_points(self._h, i, *[c.ctypes.data_as(_dp) for c in cols]))
            out.append(ResourceTrace(mid.value.decode(),
                                     [(float(cols[0][q]), float(cols[1][q]), float(cols[2][q]))
                                      for q in range(cnt.value)]))
        return out


def parse_trace(path) -> List[ResourceTrace]:
    """parse_trace (trace.cpp:54-97)."""
    return _Traces.parse(path).to_list()


def write_trace(traces: Sequence[ResourceTrace], path) -> None:
    """write_trace (trace.cpp:99-107)."""
    t = _Traces.from_list(traces)
    check(lib().lbbsp_trace_write(t._h, str(path).encode()))


def map_traces(traces: Sequence[ResourceTrace], workers: int, seed: int) -> List[int]:
    """map_traces (trace.cpp:109-135)."""
    t = _Traces.from_list(traces)
    out = np.zeros(max(workers, 1), np.int32)
    check(lib().lbbsp_trace_map(t._h, int(workers), C.c_uint64(seed), out.ctypes.data_as(_ip)))
    return [int(x) for x in out[:workers]]


def trace_at(trace: ResourceTrace, time_s: float):
    """trace_at (trace.cpp:137-143) -> (cpu, mem)."""
    t = _Traces.from_list([trace])
    c, m = C.c_double(), C.c_double()
    check(lib().lbbsp_trace_at(t._h, 0, float(time_s), C.byref(c), C.byref(m)))
    return c.value, m.value


def load_narx_csv(path) -> Narx:
    """load_narx_csv (predictor.cpp:215-243)."""
    m = Narx()
    check(lib().lbbsp_narx_load_csv(str(path).encode(), C.byref(m)))
    return m


def save_narx_csv(model: NarxModel, path) -> None:
    """save_narx_csv (predictor.cpp:198-213)."""
    check(lib().lbbsp_narx_save_csv(C.byref(model), str(path).encode()))


# --------------------------------------------------------------------------
# scenario.hpp: JSON scenarios and the CLI entry points
# --------------------------------------------------------------------------
class Scenario:
    """ScenarioConfig loaded by load_scenario (scenario.cpp:92-181)."""

    def __init__(self, path):
        h = C.c_void_p()
        check(lib().lbbsp_scenario_load(str(path).encode(), C.byref(h)))
        self._h = h

    def __del__(self):
        try:
            lib().lbbsp_scenario_destroy(self._h)
        except Exception:
            pass

    @property
    def info(self) -> abi.ScenarioInfo:
        i = abi.ScenarioInfo()
        check(lib().lbbsp_scenario_get_info(self._h, C.byref(i)))
        return i

    def set_seed(self, seed: int) -> None:
        check(lib().lbbsp_scenario_set_seed(self._h, C.c_uint64(seed)))

    def sim_config(self) -> abi.SimConfig:
        """build_sim_config (scenario.cpp:219-294); owned by this object."""
        p = C.POINTER(abi.SimConfig)()
        check(lib().lbbsp_scenario_sim_cfg(self._h, C.byref(p)))
        return p.contents


def load_scenario(path) -> Scenario:
    return Scenario(path)


def make_benchmark_series(seed: int, iterations=1200, regime_length=50, high_band=(0.75, 1.0),
                          low_band=(0.30, 0.55), spike_mult=3.0, spike_prob=0.02):
    """make_benchmark_series (cluster_sim.cpp:41-64) -> (cpu, mem, mult) arrays."""
    c, m, x = np.zeros(iterations), np.zeros(iterations), np.zeros(iterations)
    check(lib().lbbsp_benchmark_series(C.c_uint64(seed), iterations, regime_length, *high_band,
                                       *low_band, spike_mult, spike_prob, c.ctypes.data_as(_dp),
                                       m.ctypes.data_as(_dp), x.ctypes.data_as(_dp)))
    return c, m, x


def predictor_series_rmse(kind, base: PredictorConfig, cpu, mem, mult, base_speed: float,
                          seed: int, measure_from: int) -> float:
    """predictor_series_rmse (cluster_sim.cpp:645-672), one device CTA."""
    c, cp = _d(cpu); m, mp = _d(mem); x, xp = _d(mult)
    kind = abi.PREDICTORS[kind] if isinstance(kind, str) else int(kind)
    out = C.c_double()
    check(lib().lbbsp_predictor_series_rmse(kind, C.byref(base), cp, mp, xp, len(c),
                                            float(base_speed), C.c_uint64(seed),
                                            int(measure_from), C.byref(out)))
    return out.value


def _seed_args(seed_override):
    return (0, 0) if seed_override is None else (1, int(seed_override))


def cmd_run(config, out_dir, seed_override: Optional[int] = None) -> int:
    """cmd_run (scenario.cpp:369-386); returns the CLI exit status."""
    h, s = _seed_args(seed_override)
    return lib().lbbsp_cmd_run(str(config).encode(), str(out_dir).encode(), h, C.c_uint64(s))
