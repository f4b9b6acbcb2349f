"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes bindings for the two CPU checkers:
  * ``restatement()`` -- oracle/liblbbsp_oracle.so, the plain-C restatement
    (oracle/lbbsp_oracle.c) of the reference hot path;
  * ``reference()``   -- oracle/_ref/liblbbsp_ref.so, the UNMODIFIED reference
    core compiled from /root/reference/proj/core/src by oracle/Makefile.
Both expose the same Python interface. Only tests/, bench.py's cpu_baseline /
--impl reference legs and __graft_entry__.smoke() may import this module.
"""
import ctypes as C
import os

import numpy as np

from paper_1806_02508_b200 import abi
from paper_1806_02508_b200.errors import raise_for

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATEMENT_SO = os.path.join(HERE, "liblbbsp_oracle.so")
REFERENCE_SO = os.path.join(HERE, "_ref", "liblbbsp_ref.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


def _d(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(_dp)


def _i(a):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, a.ctypes.data_as(_ip)


class CpuChecker:
    def __init__(self, path, prefix):
        self.path = path
        self.prefix = prefix
        self.lib = C.CDLL(path)
        L = self.lib
        f = lambda name: getattr(L, prefix + name)
        self._err = f("last_error"); self._err.restype = C.c_char_p
        self._mix3 = f("mix_seed3"); self._mix3.restype = C.c_uint64
        self._mix3.argtypes = [C.c_uint64] * 3
        self._mix2 = f("mix_seed2"); self._mix2.restype = C.c_uint64
        self._mix2.argtypes = [C.c_uint64] * 2
        for name in ("cpu_allocate", "gpu_allocate", "ema", "narx_train", "generate_dataset",
                     "batch_gradient", "loss", "aggregate", "benchmark_series", "sim_run",
                     "replay_cpu"):
            getattr(L, prefix + name).restype = C.c_int
        self._narx_predict = f("narx_predict"); self._narx_predict.restype = C.c_double
        self._rng_u64 = f("rng_u64")
        self._rng_ui = f("rng_uniform_int")

    # -- helpers ------------------------------------------------------------
    def _check(self, code):
        if code != 0:
            raise_for(code, self._err().decode())

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def mix_seed(self, *a):
        a = [int(x) & (2 ** 64 - 1) for x in a]
        return self._mix3(*a) if len(a) == 3 else self._mix2(*a)

    def rng_u64(self, seed, count):
        out = np.zeros(count, np.uint64)
        self._rng_u64(C.c_uint64(seed), C.c_int(count), out.ctypes.data_as(C.POINTER(C.c_uint64)))
        return out

    def rng_uniform_int(self, seed, count, lo, hi):
        out = np.zeros(count, np.int32)
        self._rng_ui(C.c_uint64(seed), C.c_int(count), C.c_int(lo), C.c_int(hi),
                     out.ctypes.data_as(_ip))
        return out

    def sample_stream(self, seed, k, budget, dataset_size):
        """cluster_sim.cpp:302-307 via the public Rng/mix_seed API"""
        return self.rng_uniform_int(self.mix_seed(seed, 0x57e3a9, k), budget, 0, dataset_size - 1)

    # -- solver ---------------------------------------------------------------
    def cpu_allocate(self, speeds, budget):
        v, vp = _d(speeds)
        out = np.zeros(len(v), np.int32)
        self._check(self._fn("cpu_allocate")(vp, C.c_int(len(v)), C.c_int(budget),
                                             out.ctypes.data_as(_ip)))
        return out

    def gpu_allocate(self, profiles, comm, budget):
        n = len(profiles)
        arr = (abi.GpuProfile * max(n, 1))(*[abi.GpuProfile(*p) for p in profiles])
        cm, cp = _d(comm)
        out = np.zeros(max(n, 1), np.int32)
        self._check(self._fn("gpu_allocate")(arr, cp, C.c_int(n), C.c_int(budget),
                                             out.ctypes.data_as(_ip)))
        return out[:n]

    # -- predictor --------------------------------------------------------------
    def ema(self, series, alpha):
        s, sp = _d(series)
        out = C.c_double()
        self._check(self._fn("ema")(sp, C.c_int(len(s)), C.c_double(alpha), C.byref(out)))
        return out.value

    def narx_init(self, seed):
        m = abi.NarxModel()
        self._fn("narx_init")(C.c_uint64(seed), C.byref(m))
        return m

    def narx_predict(self, model, speeds, cpu, mem, floor=1e-3):
        v, vp = _d(speeds); c, cp = _d(cpu); m, mp = _d(mem)
        return self._narx_predict(C.byref(model), vp, cp, mp, C.c_double(floor))

    def narx_train(self, model, speed, cpu, mem, cfg):
        """mutates model in place; returns (report, loss_log)"""
        v, vp = _d(speed); c, cp = _d(cpu); m, mp = _d(mem)
        rep = abi.NarxReport()
        log = np.zeros(max(cfg.max_epochs, 1), np.float64)
        self._check(self._fn("narx_train")(
            C.byref(model), vp, cp, mp, C.c_int(len(v)), C.byref(cfg), C.byref(rep),
            log.ctypes.data_as(_dp), C.c_int(len(log))))
        return rep, log[:rep.epochs].copy()

    # -- workload ---------------------------------------------------------------
    def generate_dataset(self, seed, n, d, noise=0.2):
        feat = np.zeros((n, d)); lab = np.zeros(n)
        self._check(self._fn("generate_dataset")(
            C.c_uint64(seed), C.c_int(n), C.c_int(d), C.c_double(noise),
            feat.ctypes.data_as(_dp), lab.ctypes.data_as(_dp)))
        return feat, lab

    def batch_gradient(self, feat, lab, params, idx):
        f, fp = _d(feat); l, lp = _d(lab); p, pp = _d(params); ix, ip = _i(idx)
        out = np.zeros(f.shape[1])
        self._check(self._fn("batch_gradient")(
            fp, lp, C.c_int(f.shape[0]), C.c_int(f.shape[1]), pp, ip, C.c_int(len(ix)),
            out.ctypes.data_as(_dp)))
        return out

    def loss(self, feat, lab, params):
        f, fp = _d(feat); l, lp = _d(lab); p, pp = _d(params)
        out = C.c_double()
        self._check(self._fn("loss")(fp, lp, C.c_int(f.shape[0]), C.c_int(f.shape[1]), pp,
                                     C.byref(out)))
        return out.value

    def aggregate(self, grads, sizes, weighted=True):
        g, gp = _d(grads); s, sp = _i(sizes)
        out = np.zeros(g.shape[1])
        self._check(self._fn("aggregate")(
            gp, sp, C.c_int(g.shape[0]), C.c_int(g.shape[1]), C.c_int(1 if weighted else 0),
            out.ctypes.data_as(_dp)))
        return out

    def benchmark_series(self, seed, iterations=1200):
        c = np.zeros(iterations); m = np.zeros(iterations); x = np.zeros(iterations)
        self._check(self._fn("benchmark_series")(
            C.c_uint64(seed), C.c_int(iterations), c.ctypes.data_as(_dp), m.ctypes.data_as(_dp),
            x.ctypes.data_as(_dp)))
        return c, m, x

    # -- iteration driver ---------------------------------------------------------
    def sim_run(self, cfg):
        n, d = cfg.n_workers, cfg.dataset_dim
        rows_cap = int(max(cfg.max_updates, 1))
        sc = (abi.IterScalars * rows_cap)()
        keys = ("tp", "tm", "wait", "v_pred", "v_actual")
        arr = {k: np.zeros(rows_cap * n) for k in keys}
        batch = np.zeros(rows_cap * n, np.int32)
        wid = np.zeros(rows_cap * n, np.int32)
        nw = np.zeros(rows_cap, np.int32)
        params = np.zeros(rows_cap * d)
        rows = C.c_int(); conv = C.c_int()
        self._check(self._fn("sim_run")(
            C.byref(cfg), C.c_int(rows_cap), C.byref(rows), sc, batch.ctypes.data_as(_ip),
            *[arr[k].ctypes.data_as(_dp) for k in keys],
            params.ctypes.data_as(_dp), C.byref(conv), wid.ctypes.data_as(_ip),
            nw.ctypes.data_as(_ip)))
        r = rows.value
        out = {k: v[: r * n].reshape(r, n) for k, v in arr.items()}
        out["batch"] = batch[: r * n].reshape(r, n)
        out["worker_id"] = wid[: r * n].reshape(r, n)
        out["row_workers"] = nw[:r].copy()
        out["params"] = params[: r * d].reshape(r, d)
        out["k"] = np.array([sc[i].k for i in range(r)])
        out["grad_norm"] = np.array([sc[i].grad_norm for i in range(r)])
        out["loss"] = np.array([sc[i].loss for i in range(r)])
        out["wall"] = np.array([sc[i].wall_s for i in range(r)])
        out["converged"] = bool(conv.value)
        return out

    def replay_cpu(self, pcfg, seeds, budget, v_obs, c_obs, m_obs):
        v, vp = _d(v_obs); c, cp = _d(c_obs); m, mp = _d(m_obs)
        iters, n = v.shape
        sd = (C.c_uint64 * n)(*[int(s) for s in seeds])
        sizes = np.zeros((iters, n), np.int32)
        vpred = np.zeros((iters, n))
        self._check(self._fn("replay_cpu")(
            C.byref(pcfg), sd, C.c_int(n), C.c_int(budget), C.c_int(iters), vp, cp, mp,
            sizes.ctypes.data_as(_ip), vpred.ctypes.data_as(_dp)))
        return sizes, vpred


    # -- scenario / CLI (reference build only: scenario.cpp, trace.cpp) -----------
    def cmd_run(self, config, out_dir, seed=None):
        f = self._fn("cmd_run")
        f.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_uint64]
        return f(str(config).encode(), str(out_dir).encode(), int(seed is not None),
                 int(seed or 0))

    def cmd_compare(self, configs, out_dir, seed=None):
        f = self._fn("cmd_compare")
        f.argtypes = [C.POINTER(C.c_char_p), C.c_int, C.c_char_p, C.c_int, C.c_uint64]
        arr = (C.c_char_p * len(configs))(*[str(c).encode() for c in configs])
        return f(arr, len(configs), str(out_dir).encode(), int(seed is not None), int(seed or 0))

    def cmd_predict_bench(self, config, out_dir, seed=None):
        f = self._fn("cmd_predict_bench")
        f.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_uint64]
        return f(str(config).encode(), str(out_dir).encode(), int(seed is not None),
                 int(seed or 0))

    def scenario_error(self, config):
        """load_scenario's exception text, or None when the file loads."""
        f = self._fn("scenario_check")
        f.argtypes = [C.c_char_p]
        return None if f(str(config).encode()) == 0 else self._err().decode()

    def trace_map(self, path, workers, seed):
        f = self._fn("trace_map")
        f.argtypes = [C.c_char_p, C.c_int, C.c_uint64, _ip, _ip]
        out = np.zeros(workers, np.int32)
        nt = C.c_int()
        self._check(f(str(path).encode(), workers, seed, out.ctypes.data_as(_ip), C.byref(nt)))
        return out.tolist()

    def trace_at(self, path, i, t):
        f = self._fn("trace_at")
        f.argtypes = [C.c_char_p, C.c_int, C.c_double, _dp, _dp]
        c, m = C.c_double(), C.c_double()
        self._check(f(str(path).encode(), i, t, C.byref(c), C.byref(m)))
        return c.value, m.value

    def series_rmse(self, kind, base, cpu, mem, mult, base_speed, seed, measure_from):
        f = self._fn("series_rmse")
        c, cp = _d(cpu); m, mp = _d(mem); x, xp = _d(mult)
        out = C.c_double()
        self._check(f(C.c_int(kind), C.byref(base), cp, mp, xp, C.c_int(len(c)),
                      C.c_double(base_speed), C.c_uint64(seed), C.c_int(measure_from),
                      C.byref(out)))
        return out.value


class RestatementChecker(CpuChecker):
    def __init__(self):
        super().__init__(RESTATEMENT_SO, "orc_")
        L = self.lib
        L.orc_tanh_glibc_fma.restype = C.c_double
        L.orc_tanh_glibc_fma.argtypes = [C.c_double]
        L.orc_expm1_glibc_fma.restype = C.c_double
        L.orc_expm1_glibc_fma.argtypes = [C.c_double]

    def sample_stream(self, seed, k, budget, dataset_size):
        out = np.zeros(budget, np.int32)
        self.lib.orc_sample_stream(C.c_uint64(seed), C.c_int64(k), C.c_int(budget),
                                   C.c_int(dataset_size), out.ctypes.data_as(_ip))
        return out

    def tanh_port(self, x):
        return self.lib.orc_tanh_glibc_fma(float(x))

    # -- generalised NARX (delay d, hidden h), the C4 sweep shape -------------
    def narxg_param_count(self, d, h):
        return self.lib.orc_narxg_param_count(C.c_int(d), C.c_int(h))

    def narxg_init(self, seed, d, h):
        p = np.zeros(self.narxg_param_count(d, h))
        self.lib.orc_narxg_init(C.c_uint64(seed), C.c_int(d), C.c_int(h), p.ctypes.data_as(_dp))
        return p

    def narxg_train(self, params, d, h, speed, cpu, mem, cfg, fixed_epochs=0):
        """mutates params in place; returns (report, loss_log)"""
        v, vp = _d(speed); c, cp = _d(cpu); m, mp = _d(mem)
        rep = abi.NarxReport()
        cap = max(cfg.max_epochs, fixed_epochs, 1)
        log = np.zeros(cap)
        assert params.dtype == np.float64 and params.flags.c_contiguous
        self._check(self.lib.orc_narxg_train(params.ctypes.data_as(_dp), C.c_int(d), C.c_int(h), vp,
                                             cp, mp, C.c_int(len(v)), C.byref(cfg),
                                             C.c_int(fixed_epochs), C.byref(rep),
                                             log.ctypes.data_as(_dp), C.c_int(cap)))
        return rep, log[:rep.epochs].copy()

    def narxg_predict(self, params, d, h, vlags, cwin, mwin, floor=1e-3):
        v, vp = _d(vlags); c, cp = _d(cwin); m, mp = _d(mwin)
        self.lib.orc_narxg_predict.restype = C.c_double
        return self.lib.orc_narxg_predict(params.ctypes.data_as(_dp), C.c_int(d), C.c_int(h), vp, cp,
                                          mp, C.c_double(floor))


_cache = {}


def restatement():
    if "orc" not in _cache:
        _cache["orc"] = RestatementChecker()
    return _cache["orc"]


def reference_available():
    return os.path.exists(REFERENCE_SO)


def reference():
    if "ref" not in _cache:
        _cache["ref"] = CpuChecker(REFERENCE_SO, "ref_")
    return _cache["ref"]


def build():
    """Compile the checkers (make -C oracle). Building the checker is not using it."""
    import subprocess
    subprocess.run(["make", "-s", "-C", HERE], check=True)
