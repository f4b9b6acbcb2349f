"""Probe (GPU): C2 round and worker-window times with the fused worker kernel
vs the three separate launches, no stragglers (a = 1 everywhere)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
from paper_1806_02508_b200.mlp import MlpEngine, constant_trace

for fuse in ("pair",):
    os.environ.pop("LBBSP_NO_FUSE", None)
    os.environ.pop("LBBSP_FUSE_SINGLE", None)
    if fuse == "single":
        os.environ["LBBSP_FUSE_SINGLE"] = "1"
    elif not fuse:
        os.environ["LBBSP_NO_FUSE"] = "1"
    for static in ([512] * 8, None):
        eng = MlpEngine(dims=[784, 256, 10], global_batch=4096, n_workers_local=8, predictor="ema",
                        max_iterations=80, trace=constant_trace(8, 80), static_sizes=static)
        st = torch.cuda.ExternalStream(eng.stream)
        eng.run(20)
        torch.cuda.synchronize()
        ms = []
        for _ in range(40):
            s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
            s.record(st); eng.run(1); e.record(st); e.synchronize()
            ms.append(s.elapsed_time(e))
        rec = eng.records()
        tw = rec["t_worker"][20:60]
        ph = eng.phase_times()
        print(f"fuse={fuse} static={static is not None}: round median {np.median(ms)*1e3:.1f} us, "
              f"worker t median {np.median(tw)*1e6:.1f} us (min {tw.min()*1e6:.1f} max {tw.max()*1e6:.1f}), "
              f"phases(us) {[round(x*1e6,1) for x in ph]}, launches {eng.launches_per_iteration()}", flush=True)
        del eng

# per-CTA stage timeline of one fused launch (LBBSP_FZ_DEBUG)
import ctypes as C
from paper_1806_02508_b200.mlp import _L
os.environ.pop("LBBSP_NO_FUSE", None)
os.environ.pop("LBBSP_FUSE_SINGLE", None)
os.environ["LBBSP_FZ_DEBUG"] = "1"
eng = MlpEngine(dims=[784, 256, 10], global_batch=4096, n_workers_local=8, predictor="ema",
                max_iterations=40, trace=constant_trace(8, 40), static_sizes=[512] * 8)
eng.run(30)
buf = np.zeros(148 * 16, np.uint64)
n = C.c_int()
f = _L().lbbsp_mlp_fused_debug
f.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_int)]
f(eng._h, buf.ctypes.data_as(C.c_void_p), C.byref(n))
t = buf.reshape(148, 16).astype(np.int64)
base = t[t[:, 0] > 0, 0].min()
for c in range(0, 40):
    r = t[c]
    print(c, [(int(x - base) if x > 0 else -1) for x in r[:14]])
