"""Debug: run the C4 tcgen05 trainer on the test shapes and print per-model epochs (negative = watchdog code)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import numpy as np, torch
from paper_1806_02508_b200 import abi
from paper_1806_02508_b200.narx_sweep import NarxSweep
from test_gpu_narx_sweep import histories
for d, h, L, E in [(10, 64, 300, 25), (10, 64, 1000, 3), (2, 1, 200, 5), (4, 16, 400, 5)]:
    v, c, m = histories(6, L)
    sw = NarxSweep(list(range(1, 7)), delay=d, hidden=h)
    cfg = abi.NarxTrainConfig.default(min_history=d + 1)
    ep, loss = sw.train(v, c, m, cfg, fixed_epochs=E)
    torch.cuda.synchronize()
    print(d, h, L, E, ep.cpu().numpy().tolist(), [round(float(x), 5) for x in loss.cpu().numpy()], flush=True)
