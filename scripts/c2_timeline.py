"""Device timeline of one steady-state C2 round (debug helper)."""
import os, sys, ctypes as C
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
from paper_1806_02508_b200.mlp import MlpEngine, benchmark_trace, constant_trace
from paper_1806_02508_b200._lib import lib
n, B = 8, 4096
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for pred in ("ema", "narx"):
    eng = MlpEngine(dims=[784, 256, 10], global_batch=B, n_workers_local=n, predictor=pred,
                    warmup_iterations=50, max_iterations=300, trace=benchmark_trace(n, 300, seed=3))
    st = torch.cuda.ExternalStream(eng.stream)
    eng.run(100)
    for rep in range(3):
        flush.zero_(); torch.cuda.synchronize()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            s.record(st)
        eng.run(1)
        with torch.cuda.stream(st):
            e.record(st)
        e.synchronize()
        buf = np.zeros(16 + 2 * 28 * n, np.uint64); nph = C.c_int()
        lib().lbbsp_mlp_debug_timeline(C.c_void_p(eng._h.value if hasattr(eng._h, "value") else eng._h),
                                       buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), C.byref(nph))
        t0 = int(buf[0])
        st_ = {k: (int(buf[i]) - t0) / 1e3 for i, k in enumerate(["plan_in", "plan_out", "gather_in", "obs_in", "obs_out", "reduce_in", "losshead_in", "losshead_out"])}
        tim = buf[16:16 + 2 * nph.value * n].astype(np.int64).reshape(nph.value, n, 2)
        ph = [((tim[p, :, 0].min() - t0) / 1e3, (tim[p, :, 1].max() - t0) / 1e3) for p in range(nph.value)]
        print(f"{pred} round {s.elapsed_time(e)*1e3:.1f} us  stamps(us from plan entry) {st_}  phases {[(round(a,1), round(b,1)) for a,b in ph]}")
    del eng
