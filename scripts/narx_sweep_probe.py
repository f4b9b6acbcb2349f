"""C4 throughput (histories resident in HBM, one train launch timed with CUDA events): W in {8..1024} histories of L=1000, delay 10, hidden 64,
fixed 20 epochs; model-epochs/s and achieved fp32 FLOP/s."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import numpy as np, torch
from paper_1806_02508_b200 import abi
from paper_1806_02508_b200.narx_sweep import NarxSweep
from test_gpu_narx_sweep import histories
L, d, h, E = 1000, 10, 64, 20
vv, cc, mm = histories(1024, L)
for W in (8, 64, 148, 296, 1024):
    sw = NarxSweep(list(range(1, W + 1)), delay=d, hidden=h)
    cfg = abi.NarxTrainConfig.default(min_history=d + 1)
    dv, dc, dm = (torch.from_numpy(np.ascontiguousarray(x[:W])).cuda() for x in (vv, cc, mm))
    sw.train(dv, dc, dm, cfg, fixed_epochs=2); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); ep, loss = sw.train(dv, dc, dm, cfg, fixed_epochs=E); e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    I = 3 * d + 2; cnt = L - d
    flop = W * E * cnt * (2 * I * h * 2 + 10 * h)  # fwd + dW1 fold per eval, 1 eval/epoch (no halvings)
    print(f"W={W:5d}: {ms:9.2f} ms for {E} epochs  {W*E/ms*1e3:10.0f} model-epochs/s  ~{flop/ms/1e9:7.2f} TFLOP/s  epochs[0]={int(ep[0])}")
