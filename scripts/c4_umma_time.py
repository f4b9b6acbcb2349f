import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import torch
from paper_1806_02508_b200 import abi
from paper_1806_02508_b200.narx_sweep import NarxSweep
from test_gpu_narx_sweep import histories
v, c, m = histories(148, 1000)
sw = NarxSweep(list(range(1, 149)), delay=10, hidden=64)
cfg = abi.NarxTrainConfig.default(min_history=11)
cfg.max_epochs = 12345
ep, loss = sw.train(v, c, m, cfg, fixed_epochs=5)
torch.cuda.synchronize()
print("done", ep[:3].tolist())
