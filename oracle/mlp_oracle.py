"""ORACLE / TEST INFRASTRUCTURE ONLY.

fp64 numpy restatement of one LB-BSP round of the MLP workload. The reference
has no MLP, so this restates the reference's round semantics with
the model swapped:
  * sample stream        cluster_sim.cpp:302-307 (indices supplied by caller)
  * contiguous chunking  cluster_sim.cpp:422-431 (worker i = stream[off_i : off_i + b_i])
  * per-worker mean grad sgd.cpp:72-90
  * Eq. 7 weighting      coordination.cpp:52-68 (b_i / B), Eq. 6 for BSP (:39-50)
  * update               sgd.cpp:92-99 (w -= lr g)
  * full-dataset loss    sgd.cpp:65-70 / cluster_sim.cpp:445 (mean softmax-CE)
with logistic loss -> softmax cross-entropy and the linear model -> ReLU MLP.
"""
import numpy as np


def forward(params, X):
    acts = [X]
    h = X
    for l, (W, b) in enumerate(params):
        z = h @ W.T + b
        h = np.maximum(z, 0.0) if l < len(params) - 1 else z
        acts.append(h)
    return acts


def softmax_ce(logits, y):
    m = logits.max(axis=1, keepdims=True)
    e = np.exp(logits - m)
    s = e.sum(axis=1, keepdims=True)
    p = e / s
    loss = (np.log(s[:, 0]) + m[:, 0] - logits[np.arange(len(y)), y])
    return p, loss


def worker_mean_grad(params, X, y):
    """batch_gradient (sgd.cpp:72-90) for the MLP: mean over the segment."""
    acts = forward(params, X)
    p, _ = softmax_ce(acts[-1], y)
    d = p.copy()
    d[np.arange(len(y)), y] -= 1.0
    d /= len(y)
    grads = [None] * len(params)
    for l in range(len(params) - 1, -1, -1):
        W, b = params[l]
        grads[l] = (d.T @ acts[l], d.sum(axis=0))
        if l > 0:
            d = (d @ W) * (acts[l] > 0)
    return grads


def lbbsp_round(params, data_x, data_y, stream, sizes, lr, weighted=True):
    """One round: per-worker mean gradients over contiguous chunks, Eq. 7 (or
    Eq. 6) aggregation, SGD apply. Returns (new_params, per-worker grads)."""
    params = [(W.astype(np.float64), b.astype(np.float64)) for W, b in params]
    off = 0
    parts = []
    for b_i in sizes:
        idx = stream[off: off + b_i]
        parts.append((b_i, worker_mean_grad(params, data_x[idx].astype(np.float64), data_y[idx])))
        off += b_i
    B = float(sum(sizes))
    n = len(sizes)
    agg = []
    for l in range(len(params)):
        gW = sum((b_i / B if weighted else 1.0 / n) * g[l][0] for b_i, g in parts)
        gb = sum((b_i / B if weighted else 1.0 / n) * g[l][1] for b_i, g in parts)
        agg.append((gW, gb))
    new = [(W - lr * gW, b - lr * gb) for (W, b), (gW, gb) in zip(params, agg)]
    return new, agg


def full_loss(params, data_x, data_y):
    acts = forward([(W.astype(np.float64), b.astype(np.float64)) for W, b in params],
                   data_x.astype(np.float64))
    _, loss = softmax_ce(acts[-1], data_y)
    return float(loss.mean())


# ---------------------------------------------------------------------------
# bf16-aware restatement: same round, with the device's rounding points
# (bf16 GEMM operands and activations, fp32 accumulation), so the kernels'
# arithmetic can be checked tightly. Row scales fold the Eq. 7 weights
# (b_i/B * 1/b_i = 1/B) or Eq. 6 (1/(n b_i)) into dlogits, as on device.
# ---------------------------------------------------------------------------
def bf16(x):
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def lbbsp_round_bf16(params, data_x, data_y, stream, sizes, lr, weighted=True, small_head=None,
                     acc32=False, bucket_bf16=False):
    """params: fp32 master weights. Returns new params (fp64) and the
    aggregated gradient, emulating the device rounding points.

    acc32: accumulate every matrix product in fp32 (BLAS sgemm order) instead
    of fp64. The operands are bf16 values either way, so both variants are
    legitimate restatements of the device arithmetic; their disagreement is
    the noise floor of any bf16 implementation (activation roundings that
    flip with the accumulation order), which sizes the parity bars.

    bucket_bf16: one worker per GPU exchanges bf16 gradient buckets -- each
    worker's (1/B-scaled) partial dW/db is rounded to bf16 and the partials
    are summed in worker (rank) order in fp32 (csrc/mlp.cu, peer buckets)."""
    L = len(params)
    dt = np.float32 if acc32 else np.float64

    def mm(a, b):
        return (np.asarray(a, dtype=dt) @ np.asarray(b, dtype=dt)).astype(np.float64)
    if small_head is None:
        small_head = params[-1][0].shape[0] <= 16
    P = [(W.astype(np.float64), b.astype(np.float64)) for W, b in params]
    Wq = [bf16(W) for W, _ in P]
    B = int(sum(sizes))
    idx = np.asarray(stream[:B])
    X = data_x[idx].astype(np.float64)
    y = data_y[idx]
    n = len(sizes)
    if weighted:
        scale = np.full(B, 1.0 / B)
    else:
        scale = np.concatenate([np.full(b, 1.0 / (n * b)) for b in sizes])
    acts = [X]
    h = X
    for l in range(L - 1):
        h = bf16(np.maximum(mm(h, Wq[l].T) + P[l][1], 0.0))
        acts.append(h)
    # the small head runs on warp MMAs: bf16 W and bf16 dlogits operands,
    # fp32 accumulation; its bias gradient sums the unrounded dlogits
    logits = mm(h, Wq[-1].T) + P[-1][1]
    if not small_head:
        logits = bf16(logits)
    p, _ = softmax_ce(logits, y)
    d = p.copy()
    d[np.arange(B), y] -= 1.0
    d *= scale[:, None]
    grads = [None] * L
    for l in range(L - 1, -1, -1):
        if small_head and l == L - 1:
            grads[l] = (mm(bf16(d).T, acts[l]), d.sum(axis=0))
            d = bf16(mm(bf16(d), Wq[l]) * (acts[l] > 0))
            continue
        if l == L - 1:
            d = bf16(d)
        if bucket_bf16:
            gW = np.zeros((d.shape[1], acts[l].shape[1]), np.float32)
            gb = np.zeros(d.shape[1], np.float32)
            off = 0
            for b_i in sizes:
                seg = slice(off, off + b_i)
                gW += bf16(mm(d[seg].T, acts[l][seg])).astype(np.float32)
                gb += bf16(d[seg].sum(axis=0)).astype(np.float32)
                off += b_i
            grads[l] = (gW.astype(np.float64), gb.astype(np.float64))
        else:
            grads[l] = (mm(d.T, acts[l]), d.sum(axis=0))
        if l > 0:
            d = bf16(mm(d, Wq[l]) * (acts[l] > 0))
    new = [(W - lr * gW, b - lr * gb) for (W, b), (gW, gb) in zip(P, grads)]
    return new, grads
