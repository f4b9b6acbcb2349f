"""Host layer of the MLP gradient engine (lbbsp_mlp_* in include/lbbsp_c.h).

Builds the straggler traces (iteration-indexed availability per worker),
configures emulated / sharded workers and runs LB-BSP rounds entirely on the
device. Multi-GPU: one process per GPU; NCCL is initialised inside the
library from a unique id that rank 0 broadcasts through torch.distributed.
"""
import ctypes as C

import numpy as np

from . import abi
from ._lib import check, lib

MAX_LAYERS = 8
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


class MlpConfig(C.Structure):
    _fields_ = [
        ("n_layers", C.c_int), ("dims", C.c_int * (MAX_LAYERS + 1)),
        ("n_workers_total", C.c_int), ("n_workers_local", C.c_int), ("rank", C.c_int),
        ("world", C.c_int), ("global_batch", C.c_int), ("scheme", C.c_int),
        ("static_sizes", C.c_int), ("h_static_sizes", _ip),
        ("predictor", abi.PredictorConfig), ("learning_rate", C.c_double),
        ("seed", C.c_uint64), ("dataset_seed", C.c_uint64), ("dataset_size", C.c_int),
        ("loss_every", C.c_int), ("sm_budget", C.c_int),
        ("h_trace_c", _dp), ("h_trace_m", _dp), ("h_trace_mult", _dp), ("trace_len", C.c_int),
        ("h_worker_share", _dp), ("max_iterations", C.c_int), ("straggler_mode", C.c_int),
        ("solver", C.c_int), ("h_gpu_profiles", C.POINTER(abi.GpuProfile)),
        ("observe", C.c_int),
    ]


STRAGGLE = {"interfere": 0, "sm_cap": 1}
SOLVERS = {"proportional": 0, "gamma": 1}
OBSERVE = {"rate": 0, "capacity": 1}


_SIG = {
    "lbbsp_mlp_create": [C.POINTER(MlpConfig), C.POINTER(C.c_void_p)],
    "lbbsp_mlp_destroy": [C.c_void_p],
    "lbbsp_nccl_unique_id": [C.c_char_p],
    "lbbsp_mlp_init_comm": [C.c_void_p, C.c_char_p],
    "lbbsp_mlp_run": [C.c_void_p, C.c_int],
    "lbbsp_mlp_records": [C.c_void_p, C.c_int, _ip, _ip, _dp, _dp, _ip, _dp, _dp],
    "lbbsp_mlp_params": [C.c_void_p, C.POINTER(C.c_float), C.POINTER(C.c_longlong),
                         C.POINTER(C.c_longlong)],
    "lbbsp_mlp_set_params": [C.c_void_p, C.POINTER(C.c_float)],
    "lbbsp_mlp_dataset": [C.c_void_p, C.c_void_p, _ip],
    "lbbsp_mlp_launches_per_iteration": [C.c_void_p, _ip],
    "lbbsp_mlp_work": [C.c_void_p, _dp, _dp],
    "lbbsp_mlp_rows_per_cta": [C.c_void_p, _ip],
    "lbbsp_mlp_load_data_async": [C.c_void_p, C.c_void_p, C.c_void_p],
    "lbbsp_mlp_read_result_async": [C.c_void_p, C.c_void_p, C.c_void_p],
    "lbbsp_mlp_step_e2e": [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p],
    "lbbsp_mlp_phase_times": [C.c_void_p, _dp, _ip],
    "lbbsp_benchmark_series": [C.c_uint64, C.c_int, C.c_int] + [C.c_double] * 6 + [_dp] * 3,
}


def _L():
    L = lib()
    if not getattr(L, "_mlp_sigs", False):
        for k, v in _SIG.items():
            getattr(L, k).argtypes = v
            getattr(L, k).restype = C.c_int
        L.lbbsp_mlp_stream.argtypes = [C.c_void_p]
        L.lbbsp_mlp_stream.restype = C.c_void_p
        L.lbbsp_mlp_result_stream.argtypes = [C.c_void_p]
        L.lbbsp_mlp_result_stream.restype = C.c_void_p
        L._mlp_sigs = True
    return L


def mix_seed(*a):
    """rng.hpp:9-20 (host utility for trace seeding)."""
    M = (1 << 64) - 1

    def mix64(z):
        z = (z + 0x9e3779b97f4a7c15) & M
        z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & M
        z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & M
        return z ^ (z >> 31)

    def ms2(x, y):
        return mix64((x ^ mix64(y)) & M)

    if len(a) == 2:
        return ms2(a[0] & M, a[1] & M)
    return ms2(ms2(a[0] & M, a[1] & M), a[2] & M)


# ---------------------------------------------------------------------------
# straggler traces: arrays [n_workers, iterations] of (cpu, mem, mult)
# ---------------------------------------------------------------------------
def benchmark_trace(n_workers, iterations, seed=3, **bench):
    """Per-worker make_benchmark_series(mix_seed(seed, 0xbe7c, i)) -- the
    Dynamics 'benchmark' kind (cluster_sim.cpp:41-75) -- as a recorded trace,
    iteration-indexed. c drives the worker's SM availability."""
    b = dict(regime_length=50, high_lo=0.75, high_hi=1.0, low_lo=0.30, low_hi=0.55,
             spike_mult=3.0, spike_prob=0.02)
    b.update(bench)
    c = np.zeros((n_workers, iterations)); m = np.zeros_like(c); x = np.zeros_like(c)
    L = _L()
    for i in range(n_workers):
        check(L.lbbsp_benchmark_series(mix_seed(seed, 0xbe7c, i), iterations, b["regime_length"],
                                       b["high_lo"], b["high_hi"], b["low_lo"], b["low_hi"],
                                       b["spike_mult"], b["spike_prob"],
                                       c[i].ctypes.data_as(_dp), m[i].ctypes.data_as(_dp),
                                       x[i].ctypes.data_as(_dp)))
    return c, m, x


def recorded_trace(path, n_workers, iterations, seed=1, seconds_per_iteration=60.0):
    """A recorded resource-trace CSV (parse_trace + map_traces, trace.cpp:54-135)
    as the engine's iteration-indexed straggler trace: worker i follows the
    machine map_traces assigns it, sampled with trace_at (trace.cpp:137-143)
    at t = k * seconds_per_iteration. The SM cap
    follows cpu_avail * MemPenalty(mem_avail) (cluster_sim.cpp:22-29); no
    transient spikes."""
    from . import lbbsp as LB
    traces = LB.parse_trace(path)
    assign = LB.map_traces(traces, n_workers, seed)
    c = np.zeros((n_workers, iterations)); m = np.zeros_like(c)
    for i, t in enumerate(assign):
        tr = traces[t]
        for k in range(iterations):
            c[i, k], m[i, k] = LB.trace_at(tr, k * seconds_per_iteration)
    return c, m, np.ones_like(c)


def constant_trace(n_workers, iterations, availability=None):
    a = np.ones(n_workers) if availability is None else np.asarray(availability, dtype=np.float64)
    c = np.repeat(a[:, None], iterations, axis=1)
    return c, np.ones_like(c), np.ones_like(c)


def calibrate_gamma(dims, batch, n_workers_local=8, rounds=6, warm=2, **kw):
    """Unloaded Gamma profile of every local worker, the paper's offline GPU
    profiling (PAPER.md GPU cluster: time flat below x_s, then linear) done on
    this engine: each worker runs at availability 1 on its own CTA partition
    with three batch sizes around its nominal share x = batch / n (x/2, x,
    3x/2; static sizes summing to `batch`), and t = m0 x + b0 is fitted to the
    median worker time of each by least squares. Returns
    [(m0, b0, x_s=1, x_o)] per local worker, x_o = the rows one tile wave of
    the worker's CTA partition covers (caps x rows_per_cta, at most `batch`):
    past it the time steps up by a whole wave, which the linear profile does
    not describe, so gpu_allocate must not go there (the reference's
    oom_point, batch_sizer.hpp:12-18). One worker per GPU (n_workers_local ==
    1): three single-worker engines with global batch x/2, x, 3x/2, x_o =
    batch."""
    n = n_workers_local
    x = batch // n
    if n == 1:
        configs = [[max(1, x // 2)], [x], [x + x // 2]]
    else:
        lo, hi = x // 2, x + x // 2
        alt = [hi if i % 2 == 0 else lo for i in range(n)]
        alt2 = [lo if i % 2 == 0 else hi for i in range(n)]
        if n % 2:
            alt[-1] = alt2[-1] = x
        configs = [[x] * n, alt, alt2]
    pts = [[] for _ in range(n)]
    wave = [batch] * n
    iters = warm + rounds + 2
    for sizes in configs:
        eng = MlpEngine(dims=dims, global_batch=int(sum(sizes)), n_workers_local=n, predictor="ema",
                        max_iterations=iters, trace=constant_trace(n, iters),
                        static_sizes=sizes if n > 1 else None, **kw)
        eng.run(warm + rounds)
        rec = eng.records()
        t = rec["t_worker"][warm:]
        rpc = eng.rows_per_cta()
        for i in range(n):
            pts[i].append((sizes[i], float(np.median(t[:, i]))))
            if n > 1:
                wave[i] = min(wave[i], int(rec["caps"][warm:, i].min()) * rpc)
        del eng
    prof = []
    for i in range(n):
        xs = np.array([p[0] for p in pts[i]], dtype=np.float64)
        ts = np.array([p[1] for p in pts[i]], dtype=np.float64)
        m0, b0 = np.polyfit(xs, ts, 1)
        m0 = max(float(m0), 1e-12)
        b0 = max(float(b0), 0.0)
        prof.append((m0, b0, 1, min(batch, wave[i])))
    return prof


class MlpEngine:
    def __init__(self, dims, global_batch, n_workers_local=8, world=1, rank=0,
                 scheme="lb-bsp", predictor="narx", warmup_iterations=50, alpha=0.2,
                 learning_rate=0.05, seed=1, dataset_seed=7, dataset_size=1000, loss_every=1,
                 sm_budget=0, trace=None, worker_share=None, max_iterations=1000,
                 static_sizes=None, train=None, straggler="interfere", solver="proportional",
                 gamma_profiles=None, observe="rate"):
        n_total = n_workers_local * world
        if trace is None:
            trace = constant_trace(n_total, max_iterations)
        c = MlpConfig()
        c.n_layers = len(dims) - 1
        for i, d in enumerate(dims):
            c.dims[i] = d
        c.n_workers_total, c.n_workers_local = n_total, n_workers_local
        c.rank, c.world = rank, world
        c.global_batch = global_batch
        c.scheme = abi.SCHEMES[scheme] if isinstance(scheme, str) else scheme
        self._keep = []
        if static_sizes is not None:
            a = np.ascontiguousarray(static_sizes, dtype=np.int32)
            self._keep.append(a)
            c.static_sizes = 1
            c.h_static_sizes = a.ctypes.data_as(_ip)
        kind = abi.PREDICTORS[predictor] if isinstance(predictor, str) else predictor
        c.predictor = abi.PredictorConfig(kind, alpha, warmup_iterations, 1e-3,
                                          train if train is not None else abi.NarxTrainConfig.default())
        c.learning_rate = learning_rate
        c.seed, c.dataset_seed, c.dataset_size = seed, dataset_seed, dataset_size
        c.loss_every, c.sm_budget = loss_every, sm_budget
        tc, tm, tx = [np.ascontiguousarray(t, dtype=np.float64) for t in trace]
        assert tc.shape[0] == n_total, "trace must have one row per worker"
        self._keep += [tc, tm, tx]
        c.h_trace_c, c.h_trace_m, c.h_trace_mult = (t.ctypes.data_as(_dp) for t in (tc, tm, tx))
        c.trace_len = tc.shape[1]
        if worker_share is not None:
            s = np.ascontiguousarray(worker_share, dtype=np.float64)
            self._keep.append(s)
            c.h_worker_share = s.ctypes.data_as(_dp)
        c.max_iterations = max_iterations
        c.straggler_mode = STRAGGLE[straggler] if isinstance(straggler, str) else straggler
        c.solver = SOLVERS[solver] if isinstance(solver, str) else solver
        c.observe = OBSERVE[observe] if isinstance(observe, str) else observe
        if gamma_profiles is not None:
            arr = (abi.GpuProfile * len(gamma_profiles))(
                *[abi.GpuProfile(float(m), float(b), int(xs), int(xo)) for m, b, xs, xo in gamma_profiles])
            self._keep.append(arr)
            c.h_gpu_profiles = C.cast(arr, C.POINTER(abi.GpuProfile))
        self.cfg = c
        self.dims = list(dims)
        self.n_total = n_total
        self.trace = (tc, tm, tx)
        h = C.c_void_p()
        check(_L().lbbsp_mlp_create(C.byref(c), C.byref(h)))
        self._h = h

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                _L().lbbsp_mlp_destroy(self._h)
        except Exception:
            pass

    # -- multi-GPU ------------------------------------------------------------
    @staticmethod
    def nccl_unique_id():
        buf = C.create_string_buffer(128)
        check(_L().lbbsp_nccl_unique_id(buf))
        return buf.raw

    def init_comm(self, uid: bytes):
        check(_L().lbbsp_mlp_init_comm(self._h, C.c_char_p(uid)))

    def peer_handle(self) -> bytes:
        buf = C.create_string_buffer(64)
        check(_L().lbbsp_mlp_peer_handle(self._h, buf))
        return buf.raw

    def init_peers(self, handles):
        """handles: the per-rank 64-byte IPC handles in rank order."""
        blob = b"".join(handles)
        check(_L().lbbsp_mlp_init_peers(self._h, C.c_char_p(blob)))

    # -- run --------------------------------------------------------------------
    def run(self, iterations):
        check(_L().lbbsp_mlp_run(self._h, int(iterations)))

    @property
    def stream(self):
        return _L().lbbsp_mlp_stream(self._h)

    @property
    def result_stream(self):
        """stream of the e2e result reads (read_result_async / step_e2e)"""
        return _L().lbbsp_mlp_result_stream(self._h)

    def launches_per_iteration(self):
        x = C.c_int()
        check(_L().lbbsp_mlp_launches_per_iteration(self._h, C.byref(x)))
        return x.value

    def work(self):
        f, b = C.c_double(), C.c_double()
        check(_L().lbbsp_mlp_work(self._h, C.byref(f), C.byref(b)))
        return f.value, b.value

    def rows_per_cta(self):
        x = C.c_int()
        check(_L().lbbsp_mlp_rows_per_cta(self._h, C.byref(x)))
        return x.value

    def load_data_async(self, x_ptr, y_ptr):
        check(_L().lbbsp_mlp_load_data_async(self._h, x_ptr, y_ptr))

    def read_result_async(self, sizes_ptr, loss_ptr):
        check(_L().lbbsp_mlp_read_result_async(self._h, sizes_ptr, loss_ptr))

    def step_e2e(self, x_ptr, y_ptr, sizes_ptr, loss_ptr):
        """one end-to-end round: stage host inputs, run, write sizes + loss to host"""
        check(_L().lbbsp_mlp_step_e2e(self._h, x_ptr, y_ptr, sizes_ptr, loss_ptr))

    def phase_times(self):
        """device duration (s) of each worker phase of the last round"""
        buf = np.zeros(64)
        n = C.c_int()
        check(_L().lbbsp_mlp_phase_times(self._h, buf.ctypes.data_as(_dp), C.byref(n)))
        return buf[: n.value] * 1e-9

    def worker_phase_times(self):
        """[n_phases, n_local] device seconds of each worker in each phase (last round)"""
        buf = np.zeros(64 * self.cfg.n_workers_local)
        n = C.c_int()
        f = _L().lbbsp_mlp_worker_phase_times
        f.argtypes = [C.c_void_p, _dp, C.POINTER(C.c_int)]
        check(f(self._h, buf.ctypes.data_as(_dp), C.byref(n)))
        return buf[: n.value * self.cfg.n_workers_local].reshape(n.value, -1) * 1e-9

    def records(self):
        cap = self.cfg.max_iterations
        n = self.n_total
        sizes = np.zeros(cap * n, np.int32); caps = np.zeros(cap * n, np.int32)
        vp = np.zeros(cap * n); vo = np.zeros(cap * n); tw = np.zeros(cap * n); loss = np.zeros(cap)
        rows = C.c_int()
        check(_L().lbbsp_mlp_records(self._h, cap, C.byref(rows), sizes.ctypes.data_as(_ip),
                                     vp.ctypes.data_as(_dp), vo.ctypes.data_as(_dp),
                                     caps.ctypes.data_as(_ip), tw.ctypes.data_as(_dp),
                                     loss.ctypes.data_as(_dp)))
        r = rows.value
        shp = lambda a: a[: r * n].reshape(r, n)
        return dict(sizes=shp(sizes), v_pred=shp(vp), v_obs=shp(vo), caps=shp(caps),
                    t_worker=shp(tw), loss=loss[:r].copy(), rows=r)

    def params(self):
        n = C.c_longlong()
        check(_L().lbbsp_mlp_params(self._h, None, None, C.byref(n)))
        p = np.zeros(n.value, np.float32)
        offs = np.zeros(2 * (len(self.dims) - 1), np.int64)
        check(_L().lbbsp_mlp_params(self._h, p.ctypes.data_as(C.POINTER(C.c_float)),
                                    offs.ctypes.data_as(C.POINTER(C.c_longlong)), C.byref(n)))
        out = []
        for l in range(len(self.dims) - 1):
            dout, din = self.dims[l + 1], self.dims[l]
            w = p[offs[2 * l]: offs[2 * l] + dout * din].reshape(dout, din).copy()
            b = p[offs[2 * l + 1]: offs[2 * l + 1] + dout].copy()
            out.append((w, b))
        return out

    def dataset(self):
        N, d0 = self.cfg.dataset_size, self.dims[0]
        x = np.zeros(N * d0, np.uint16)
        y = np.zeros(N, np.int32)
        check(_L().lbbsp_mlp_dataset(self._h, x.ctypes.data_as(C.c_void_p), y.ctypes.data_as(_ip)))
        xf = (x.astype(np.uint32) << 16).view(np.float32).reshape(N, d0)
        return xf, y


def connect(eng, world, rank, nccl=True, peers=True, group=None):
    """Multi-GPU control plane of one rank, over an initialised
    torch.distributed process group: rank 0's NCCL unique id is broadcast and
    every rank joins the communicator (the speed all-gather and the fallback
    all-reduce), then the 64-byte CUDA-IPC handles of every rank's peer
    buffers are all-gathered in rank order and mapped (the NVLink peer-memory
    exchange of speeds and gradients, the copy-engine gradient buckets). The
    same order on every rank; returns the gathered handles.
    Reference: the coordinator's all-gather of v_actual before the replicated
    solver (cluster_sim.cpp:371-402)."""
    import torch.distributed as dist
    if world <= 1:
        return []
    if nccl:
        uid = [eng.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0, group=group)
        eng.init_comm(uid[0])
    hs = []
    if peers:
        hs = [None] * world
        dist.all_gather_object(hs, eng.peer_handle(), group=group)
        if any(h is None or len(h) != len(hs[rank]) for h in hs):
            raise RuntimeError("connect: a rank sent no peer handle")
        eng.init_peers(hs)
    return hs
