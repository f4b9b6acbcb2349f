"""Multi-GPU exchange checks, run through torchrun on 2 GPUs of
this box; skipped when fewer than 2 GPUs are visible (the round-end GPU tier
runs on one). The checks themselves are tests/mp_peer_check.py (several
workers per GPU: NVLink peer-memory speed all-gather + gradient all-reduce vs
NCCL) and tests/mp_bucket_check.py (one worker per GPU: copy-engine bucket
exchange, one-shot and two-shot, vs NCCL bf16 buckets)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _gpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("script,port", [("mp_peer_check.py", 29811), ("mp_bucket_check.py", 29812)])
def test_exchange_matches_nccl_on_2_gpus(script, port):
    if _gpus() < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(HERE, script)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
