"""Rank process for tests/test_capi_cpu.py::test_two_rank_gloo_control_exchange.

Each rank owns n_local workers, measures (here: draws) their speeds, all-gathers
them, and sizes the global batch with the solver every rank runs on identical
inputs (the restatement oracle stands in for the device solver on CPU)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

rank, world = int(sys.argv[1]), int(sys.argv[2])
dist.init_process_group("gloo", rank=rank, world_size=world)
sys.path.insert(0, os.environ["PYTHONPATH"])
from oracle import oracle as O  # noqa: E402

orc = O.restatement()
n_local, B = 4, 4096
rng = np.random.default_rng(100 + rank)
sizes_hist = []
for k in range(5):
    local = torch.tensor(rng.uniform(1.0, 10.0, n_local), dtype=torch.float64)
    allv = [torch.zeros(n_local, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(allv, local)
    speeds = torch.cat(allv).numpy()
    sizes = orc.cpu_allocate(speeds, B)
    mine = sizes[rank * n_local:(rank + 1) * n_local]
    tot = torch.tensor([int(mine.sum())])
    dist.all_reduce(tot)
    assert int(tot.item()) == B
    sizes_hist.append(",".join(map(str, sizes)))
dist.destroy_process_group()
print("|".join(sizes_hist))
