"""Rank process for tests/test_capi_cpu.py::test_gloo_connect_handshake: the
product's control-plane handshake (paper_1806_02508_b200.mlp.connect) over a
gloo group, with an engine stand-in that records what the handshake hands it
(the real init_comm / init_peers need a GPU)."""
import json
import os
import sys

import torch.distributed as dist

rank, world = int(sys.argv[1]), int(sys.argv[2])
sys.path.insert(0, os.environ["PYTHONPATH"])
dist.init_process_group("gloo", rank=rank, world_size=world)
from paper_1806_02508_b200.mlp import connect  # noqa: E402


class Recorder:
    def __init__(self, r):
        self.r, self.uid, self.handles, self.calls = r, None, None, []

    def nccl_unique_id(self):
        self.calls.append("uid")
        return b"uid-of-rank-%d" % self.r + bytes(114)

    def init_comm(self, uid):
        self.calls.append("comm")
        self.uid = uid

    def peer_handle(self):
        self.calls.append("handle")
        return bytes([self.r]) * 64

    def init_peers(self, hs):
        self.calls.append("peers")
        self.handles = hs


eng = Recorder(rank)
hs = connect(eng, world, rank)
dist.destroy_process_group()
print(json.dumps({"uid": eng.uid.rstrip(b"\0").decode(), "handles": [h[0] for h in eng.handles],
                  "lens": [len(h) for h in eng.handles], "calls": eng.calls, "ret": len(hs)}))
