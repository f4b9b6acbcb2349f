"""Times the bit-exact NARX trainer (K5) on a C2-like history (debug helper)."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
from paper_1806_02508_b200 import abi, lbbsp
rng = np.random.default_rng(0)
for L in (60, 110, 250):
    c = np.clip(rng.choice([0.9, 0.4], L) + rng.normal(0, 0.02, L), 0.05, 1)
    v = 4000 * c * rng.uniform(0.8, 1.2, L)
    h = lbbsp.SpeedHistory()
    for i in range(L):
        h.push(v[i], c[i], 1.0)
    for epochs in (10, 110):
        cfg = abi.NarxTrainConfig.default(min_history=50, max_epochs=epochs, early_stop_delta=-1.0)
        best = 1e9
        for rep in range(5):
            m = lbbsp.narx_init(7)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = lbbsp.narx_train_online(m, h, cfg)
            best = min(best, time.perf_counter() - t0)
        print(f"L={L} epochs={r.epochs} wall {best*1e6:.1f} us")
