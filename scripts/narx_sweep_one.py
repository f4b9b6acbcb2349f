"""One C4 sweep launch (W models, L=1000, delay 10, hidden 64, 20 epochs) for ncu."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import torch
from paper_1806_02508_b200 import abi
from paper_1806_02508_b200.narx_sweep import NarxSweep
from test_gpu_narx_sweep import histories
W = int(sys.argv[1]) if len(sys.argv) > 1 else 148
vv, cc, mm = histories(W, 1000)
sw = NarxSweep(list(range(1, W + 1)), delay=10, hidden=64)
cfg = abi.NarxTrainConfig.default(min_history=11)
sw.train(vv, cc, mm, cfg, fixed_epochs=20)
torch.cuda.synchronize()
print("ok")
