"""Device timeline of one steady-state C3-shape round on 1 GPU, one worker (debug helper)."""
import os, sys, ctypes as C
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
from paper_1806_02508_b200.mlp import MlpEngine, constant_trace
from paper_1806_02508_b200._lib import lib
dims = [4096] * 5
eng = MlpEngine(dims=dims, global_batch=2048, n_workers_local=1, predictor="narx",
                warmup_iterations=50, max_iterations=200, trace=constant_trace(1, 200), learning_rate=0.01)
st = torch.cuda.ExternalStream(eng.stream)
eng.run(80)
for rep in range(3):
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        s.record(st)
    eng.run(1)
    with torch.cuda.stream(st):
        e.record(st)
    e.synchronize()
    buf = np.zeros(16 + 2 * 28, np.uint64); nph = C.c_int()
    lib().lbbsp_mlp_debug_timeline(C.c_void_p(eng._h.value if hasattr(eng._h, "value") else eng._h),
                                   buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), C.byref(nph))
    t0 = int(buf[0])
    names = ["plan_in", "plan_out", "gather_in", "obs_in", "obs_out", "reduce_in", "losshead_in", "losshead_out"]
    stt = {k: round((int(buf[i]) - t0) / 1e3, 1) for i, k in enumerate(names) if buf[i] not in (0, 2**64 - 1)}
    tim = buf[16:16 + 2 * nph.value].astype(np.int64).reshape(nph.value, 2)
    ph = [(round((a - t0) / 1e3, 1), round((b - t0) / 1e3, 1)) for a, b in tim]
    print(f"round {s.elapsed_time(e)*1e3:.1f} us stamps {stt}\n  phases {ph}")
