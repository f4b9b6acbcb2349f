"""C4: generalised NARX (delay 10, hidden 64) batched trainer/predictor vs the
fp64 generalised oracle (oracle/lbbsp_oracle.c:orc_narxg_*, itself pinned to
the reference at (2, 1) by tests/test_oracle.py).

Tolerance (fp32 vs fp64 full-batch GD): with the same number of epochs the
final training loss agrees within 2e-2 relative and the next-step predictions
within 1e-2 relative (of the speed scale)."""
import numpy as np
import pytest

from paper_1806_02508_b200 import abi

pytestmark = pytest.mark.gpu


def histories(W, L, seed=3):
    from oracle import oracle as O
    orc = O.restatement()
    v = np.zeros((W, L)); c = np.zeros((W, L)); m = np.zeros((W, L))
    for i in range(W):
        ci, mi, xi = orc.benchmark_series(orc.mix_seed(seed, 0xbe7c, i), L)
        c[i], m[i], v[i] = ci, mi, 10.0 * ci * xi
    return v, c, m


@pytest.mark.parametrize("d,h,L,epochs", [(10, 64, 300, 25), (2, 1, 200, 40), (4, 16, 400, 30)])
def test_sweep_matches_fp64_generalised_oracle(orc, d, h, L, epochs):
    from paper_1806_02508_b200.narx_sweep import NarxSweep
    W = 6
    seeds = [orc.mix_seed(1, 0x9ced1c70, i) for i in range(W)]
    v, c, m = histories(W, L)
    sw = NarxSweep(seeds, delay=d, hidden=h)
    cfg = abi.NarxTrainConfig.default(min_history=d + 1)
    ep, loss = sw.train(v, c, m, cfg, fixed_epochs=epochs)
    import torch
    torch.cuda.synchronize()
    ep, loss = ep.cpu().numpy(), loss.cpu().numpy()
    pred = sw.predict(v, c, m, c[:, -1], m[:, -1]).cpu().numpy()
    for i, s in enumerate(seeds):
        p = orc.narxg_init(s, d, h)
        rep, log = orc.narxg_train(p, d, h, v[i], c[i], m[i], cfg, fixed_epochs=epochs)
        assert abs(loss[i] - rep.final_loss) <= 2e-2 * max(rep.final_loss, 1e-3), (i, loss[i], rep.final_loss)
        ref = orc.narxg_predict(p, d, h, v[i, ::-1][:d], np.r_[c[i, -1], c[i, ::-1][:d]],
                                np.r_[m[i, -1], m[i, ::-1][:d]])
        assert abs(pred[i] - ref) <= 1e-2 * max(abs(ref), 1.0), (i, pred[i], ref)
