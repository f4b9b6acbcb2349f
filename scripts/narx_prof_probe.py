"""Probe (GPU, profiling build): where the NARX training time of a C2 round
goes. Needs the library built with -DLBBSP_NARX_PROF (LBBSP_LIB_OVERRIDE).
Bench-style rounds (benchmark trace, NARX warm-up 50, L2 flushed before each
round); per round and per training CTA: history copy, scaler folds, training
set build, first evaluation, the epochs (evaluations / epochs), L."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
from paper_1806_02508_b200._lib import lib
from paper_1806_02508_b200.mlp import MlpEngine, benchmark_trace, constant_trace

n, B = 8, 4096
tr = constant_trace(n, 400) if os.environ.get("TRACE") == "const" else benchmark_trace(n, 400, seed=3)
eng = MlpEngine(dims=[784, 256, 10], global_batch=B, n_workers_local=n, predictor="narx",
                warmup_iterations=50, max_iterations=400, trace=tr,
                loss_every=int(os.environ.get("LOSS_EVERY", "1")))
L_ = lib()
L_.lbbsp_debug_narx_prof.argtypes = [C.POINTER(C.c_ulonglong)]
st = torch.cuda.ExternalStream(eng.stream)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
eng.run(int(os.environ.get("START", "100")))
torch.cuda.synchronize()
tot = []
for rep in range(int(os.environ.get("REPS", "20"))):
    if not os.environ.get("NOFLUSH"):
        with torch.cuda.stream(st):
            flush.zero_()
    eng.run(1)
    torch.cuda.synchronize()
    p = np.zeros((64, 16), np.uint64)
    L_.lbbsp_debug_narx_prof(p.ctypes.data_as(C.POINTER(C.c_ulonglong)))
    row = []
    for b in range(4):
        t = p[b].astype(np.int64)
        d = [(t[i + 1] - t[i]) / 1e3 for i in range(5)]
        row.append(d + [int(t[6]), int(t[7]), int(t[8])])
        tot.append(d + [int(t[6]), int(t[7]), int(t[8]), t[9] * 1.0, t[10] * 1.0, t[11] * 1.0, 0.0, (t[14] - t[2]) / 1e3, t[15], t[12]])
    print("round", " | ".join(f"copy {r[0]:.1f} scal {r[1]:.1f} build {r[2]:.1f} eval0 {r[3]:.1f} "
                              f"epochs {r[4]:.1f} ({r[5]} ev, {r[6]} ep, L {r[7]})" for r in row), flush=True)
a = np.array(tot)
print("median per training: copy %.2f scalers %.2f build %.2f eval0 %.2f epochs %.2f us, evals %.1f, epochs %.1f"
      % tuple(np.median(a[:, :7], axis=0)))
print("mean per evaluation (epochs phase): %.2f us" % (a[:, 4].sum() / max(1, (a[:, 5] - 1).sum())))
print("per evaluation (SM cycles): terms+barrier %.0f, fold+barrier %.0f (E-fold lane alone %.0f)"
      % (a[:, 8].sum() / a[:, 5].sum(), a[:, 9].sum() / a[:, 5].sum(), a[:, 10].sum() / a[:, 5].sum()))
print("training-set loop alone: %.2f us" % np.median(a[:, 12]))
