"""Probe (GPU): where a C2 round's event-timed duration goes outside its
kernels. Bench-style loop (L2 flush queued before each round, no host sync
between rounds); stamp kernels on the engine stream right before and after
the round's graph; the plan's entry stamp and the last kernel stamps come
from lbbsp_mlp_debug_timeline. Reports per round: event time, stamp0 ->
plan entry (graph head), plan entry -> last stamped kernel end, last stamped
end -> stamp1 (graph tail). PRED=ema|narx, TRACE=const|bench."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
from paper_1806_02508_b200._lib import lib
from paper_1806_02508_b200.mlp import MlpEngine, benchmark_trace, constant_trace

n, B = 8, 4096
pred = os.environ.get("PRED", "narx")
tr = benchmark_trace(n, 400, seed=3) if os.environ.get("TRACE") == "bench" else constant_trace(n, 400)
eng = MlpEngine(dims=[784, 256, 10], global_batch=B, n_workers_local=n, predictor=pred,
                warmup_iterations=50, max_iterations=400, trace=tr)
L = lib()
h = C.c_void_p(eng._h.value if hasattr(eng._h, "value") else eng._h)
L.lbbsp_mlp_debug_stamp.argtypes = [C.c_void_p, C.c_int]
L.lbbsp_mlp_debug_stamps.argtypes = [C.c_void_p, C.POINTER(C.c_ulonglong)]
st = torch.cuda.ExternalStream(eng.stream)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
eng.run(110)
torch.cuda.synchronize()
rows = []
for rep in range(int(os.environ.get("REPS", "12"))):
    with torch.cuda.stream(st):
        flush.zero_()
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record(st)
    assert L.lbbsp_mlp_debug_stamp(h, 0) == 0
    eng.run(1)
    assert L.lbbsp_mlp_debug_stamp(h, 1) == 0
    with torch.cuda.stream(st):
        e.record(st)
    e.synchronize()
    ds = np.zeros(8, np.uint64)
    L.lbbsp_mlp_debug_stamps(h, ds.ctypes.data_as(C.POINTER(C.c_ulonglong)))
    buf = np.zeros(16 + 2 * 28 * n, np.uint64)
    nph = C.c_int()
    L.lbbsp_mlp_debug_timeline(h, buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), C.byref(nph))
    t0 = int(buf[0])  # plan entry
    stamps = [int(x) for x in buf[:16] if int(x) > 0 and abs(int(x) - t0) < 10**9]
    tim = buf[16:16 + 2 * nph.value * n].astype(np.int64).reshape(nph.value, n, 2)
    ends = stamps + [int(tim[:, :, 1].max())]
    last = max(ends)
    rows.append((s.elapsed_time(e) * 1e3, (t0 - int(ds[0])) / 1e3, (last - t0) / 1e3, (int(ds[1]) - last) / 1e3,
                 (int(ds[1]) - int(ds[0])) / 1e3))
    print(f"{pred} event {rows[-1][0]:6.1f} us | stamp0->plan {rows[-1][1]:5.1f} | plan->last kernel "
          f"{rows[-1][2]:5.1f} | last->stamp1 {rows[-1][3]:5.1f} | stamp0->stamp1 {rows[-1][4]:6.1f}", flush=True)
r = np.array(rows)
print("median", " ".join(f"{x:.1f}" for x in np.median(r, axis=0)))
