"""Multi-rank checks of the sharded path.

test_dynamic_lbbsp_two_ranks_*: 2 ranks with DYNAMIC LB-BSP sizes
(tests/mp_lbbsp_dynamic.py), on 2 GPUs when the box has them and always as two
processes sharing cuda:0 (same CUDA-IPC peer-exchange code), so the 1-GPU
tier covers it. Checks: every rank holds the same sizes, equal to the
reference (oracle/_ref) replaying the all-gathered measured speeds
(cluster_sim.cpp:355-402, 458-464); every rank holds bitwise-equal weights;
the weights match the single-process restatement iterated with those sizes
(oracle/mlp_oracle.lbbsp_round_bf16) within the trajectory bar of
tests/test_gpu_parity_rounds.py.

test_exchange_matches_nccl_on_2_gpus: the peer / copy-engine exchanges
against NCCL (tests/mp_peer_check.py, tests/mp_bucket_check.py)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import mlp_oracle as MO
from paper_1806_02508_b200 import abi

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _gpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _torchrun(script, port, args, timeout=600):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(HERE, script)] + args
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]


def _unflat(flat, dims):
    out, o = [], 0
    for l in range(len(dims) - 1):
        dout, din = dims[l + 1], dims[l]
        w = flat[o:o + dout * din].reshape(dout, din)
        o += dout * din
        b = flat[o:o + dout]
        o += dout
        out.append((w, b))
    return out


def _check_dynamic(orc, out_dir):
    r = [dict(np.load(os.path.join(out_dir, f"rank{i}.npz"))) for i in range(2)]
    R = int(r[0]["rounds"])
    n = int(r[0]["n_local"]) * int(r[0]["world"])
    B = int(r[0]["B"])
    dims = r[0]["dims"].tolist()
    # every rank computed the same sizes from the all-gathered speeds
    assert np.array_equal(r[0]["sizes"], r[1]["sizes"])
    assert np.array_equal(r[0]["v_obs"], r[1]["v_obs"])
    sizes = r[0]["sizes"]
    assert (sizes.sum(axis=1) == B).all()
    assert len({tuple(s) for s in sizes[3:].tolist()}) > 1, "sizes never changed (not dynamic)"
    # ... and the reference replay of those speeds gives them bit for bit
    from oracle import oracle as O
    chk = O.reference() if O.reference_available() else O.restatement()
    kind = abi.PRED_NARX if int(r[0]["n_local"]) > 1 else abi.PRED_EMA
    pcfg = abi.PredictorConfig.default(kind, warmup_iterations=8)
    seeds = [chk.mix_seed(1, 0x9ced1c70, i) for i in range(n)]
    rs, rvp = chk.replay_cpu(pcfg, seeds, B, r[0]["v_obs"][:R],
                             r[0]["trace_c"][:, :R].T, r[0]["trace_m"][:, :R].T)
    assert rs.tolist() == sizes.tolist()
    assert np.array_equal(rvp, r[0]["v_pred"])
    # bitwise-equal weights on every rank
    assert np.array_equal(r[0]["params"], r[1]["params"])
    # the weights vs the single-process restatement over the same sizes
    bucket = int(r[0]["n_local"]) == 1
    p0 = _unflat(r[0]["p0"], dims)
    porc = [(w.astype(np.float32), b.astype(np.float32)) for w, b in p0]
    x, y = r[0]["x"], r[0]["y"]
    lr = float(r[0]["lr"])
    for k in range(R):
        stream = orc.sample_stream(1, k, B, 1000)
        nxt, _ = MO.lbbsp_round_bf16(porc, x, y, stream, sizes[k].tolist(), lr, bucket_bf16=bucket)
        porc = [(w.astype(np.float32), b.astype(np.float32)) for w, b in nxt]
    dev = _unflat(r[0]["params"], dims)
    for l, ((W0, b0), (W1, b1), (Wo, bo)) in enumerate(zip(p0, dev, porc)):
        ew = np.linalg.norm(W1.astype(np.float64) - Wo) / np.linalg.norm(Wo.astype(np.float64) - W0)
        eb = np.linalg.norm(b1.astype(np.float64) - bo) / max(np.linalg.norm(bo.astype(np.float64) - b0), 1e-30)
        assert ew <= 1e-2 and eb <= 1e-2, (l, ew, eb)


@pytest.mark.parametrize("mode,port", [("c2", 29821), ("c3", 29822)])
def test_dynamic_lbbsp_two_ranks_one_gpu(orc, tmp_path, mode, port):
    _torchrun("mp_lbbsp_dynamic.py", port, ["--mode", mode, "--same-device", "--out", str(tmp_path)])
    _check_dynamic(orc, str(tmp_path))


@pytest.mark.parametrize("mode,port", [("c2", 29823), ("c3", 29824)])
def test_dynamic_lbbsp_two_ranks_two_gpus(orc, tmp_path, mode, port):
    if _gpus() < 2:
        pytest.skip("needs 2 GPUs")
    _torchrun("mp_lbbsp_dynamic.py", port, ["--mode", mode, "--out", str(tmp_path)])
    _check_dynamic(orc, str(tmp_path))


@pytest.mark.parametrize("script,port", [("mp_peer_check.py", 29811), ("mp_bucket_check.py", 29812)])
def test_exchange_matches_nccl_on_2_gpus(script, port):
    if _gpus() < 2:
        pytest.skip("needs 2 GPUs")
    _torchrun(script, port, [])
