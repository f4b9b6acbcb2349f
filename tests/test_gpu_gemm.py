"""tcgen05/TMA GEMM of the gradient engine vs a plain PyTorch fp32 reference of
the same op (bf16 inputs, fp32 accumulation). Tolerance: 1e-3 relative to the
output scale for fp32 epilogues, bf16 rounding (2^-8) for bf16 epilogues."""
import ctypes as C

import pytest

pytestmark = pytest.mark.gpu


def _lib():
    from paper_1806_02508_b200._lib import lib
    L = lib()
    L.lbbsp_gemm_bf16.argtypes = [C.c_void_p] * 3 + [C.c_int] * 6 + [C.c_void_p] * 2 + \
        [C.c_int] * 2 + [C.c_void_p] * 4 + [C.c_int, C.c_void_p, C.c_int, C.c_void_p]
    L.lbbsp_gemm_bf16.restype = C.c_int
    return L


def run_gemm(A, B, M, N, K, a_mn, b_mn, epi, bias=None, aux=None, mode=0, groups=None,
             out=None, bn=0):
    import torch
    from paper_1806_02508_b200._lib import check
    L = _lib()
    if out is None:
        if epi == 0:
            shape = (len(groups[0]), M, N) if (mode == 1 and groups) else (M, N)
            out = torch.full(shape, float("nan"), dtype=torch.float32, device="cuda")
        else:
            out = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device="cuda")
    g = [0, None, None, None, None]
    keep = []
    if groups:
        r0, r1, c0, cn = [torch.tensor(x, dtype=torch.int32, device="cuda") for x in groups]
        keep += [r0, r1, c0, cn]
        g = [len(groups[0]), r0.data_ptr(), r1.data_ptr(), c0.data_ptr(), cn.data_ptr()]
    check(L.lbbsp_gemm_bf16(A.data_ptr(), B.data_ptr(), out.data_ptr(), M, N, K, int(a_mn),
                            int(b_mn), epi, bias.data_ptr() if bias is not None else None,
                            aux.data_ptr() if aux is not None else None, mode, *g, 0, None, bn,
                            torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    return out


def mk(shape, seed):
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.rand(shape, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 256, 784), (300, 200, 130),
                                   (2048, 4096, 512), (1000, 784, 256)])
@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, True), (True, False)])
def test_gemm_f32_all_majors(M, N, K, a_mn, b_mn):
    import torch
    if a_mn and M % 8:
        pytest.skip("MN-major A needs 16-byte rows")
    if b_mn and N % 8:
        pytest.skip("MN-major B needs 16-byte rows")
    if (not a_mn or not b_mn) and K % 8:
        pytest.skip("K-major operand needs 16-byte rows")
    A = mk((K, M) if a_mn else (M, K), 1)
    B = mk((K, N) if b_mn else (N, K), 2)
    Af = (A.float().t() if a_mn else A.float())
    Bf = (B.float() if b_mn else B.float().t())
    ref = Af @ Bf
    for bn in (64, 128, 256):
        out = run_gemm(A, B, M, N, K, a_mn, b_mn, 0, bn=bn)
        err = (out - ref).abs().max().item()
        assert err <= 1e-3 * max(1.0, ref.abs().max().item()), (bn, err)


def test_gemm_bias_relu_and_drelu_epilogues():
    import torch
    M, N, K = 512, 256, 784
    X = mk((M, K), 3); W = mk((N, K), 4)
    bias = torch.linspace(-0.5, 0.5, N, device="cuda")
    ref = torch.relu(X.float() @ W.float().t() + bias)
    out = run_gemm(X, W, M, N, K, False, False, 1, bias=bias)
    assert (out.float() - ref).abs().max().item() <= 2 ** -7 * max(1.0, ref.abs().max().item())
    # dX = dY W through ReLU(H): A = dY [M][N2] K-major, B = W [N2][N] as [K][N] MN-major
    N2 = 256
    dY = mk((M, N2), 5); W2 = mk((N2, N), 6)
    H = out
    ref2 = (dY.float() @ W2.float()) * (H.float() > 0)
    out2 = run_gemm(dY, W2, M, N, N2, False, True, 3, aux=H)
    assert (out2.float() - ref2).abs().max().item() <= 2 ** -7 * max(1.0, ref2.abs().max().item())


def test_gemm_ragged_worker_groups():
    """Per-worker CTA partitions with ragged segments: rows mode (forward) and
    k-split mode (dW partial per worker), odd segment lengths."""
    import torch
    sizes = [137, 611, 64, 1, 300, 777, 2000, 206]
    offs = [0]
    for s in sizes:
        offs.append(offs[-1] + s)
    Btot = offs[-1]
    r0, r1 = offs[:-1], offs[1:]
    caps = [18, 18, 18, 18, 18, 18, 20, 20]
    c0 = [sum(caps[:i]) for i in range(len(caps))]
    D_in, D_out = 784, 256
    X = mk((Btot, D_in), 7); W = mk((D_out, D_in), 8)
    bias = torch.zeros(D_out, device="cuda")
    ref = torch.relu(X.float() @ W.float().t())
    out = run_gemm(X, W, Btot, D_out, D_in, False, False, 1, bias=bias, mode=0,
                   groups=(r0, r1, c0, caps))
    assert (out.float() - ref).abs().max().item() <= 2 ** -7 * max(1.0, ref.abs().max().item())
    # dW_g = dY[seg g]^T X[seg g] : A = dY [B][D_out] (MN-major), B = X [B][D_in] (MN-major)
    dY = mk((Btot, D_out), 9)
    parts = run_gemm(dY, X, D_out, D_in, Btot, True, True, 0, mode=1, groups=(r0, r1, c0, caps))
    for gi, (a, b) in enumerate(zip(r0, r1)):
        refg = dY[a:b].float().t() @ X[a:b].float()
        err = (parts[gi] - refg).abs().max().item()
        assert err <= 1e-3 * max(1.0, refg.abs().max().item()), (gi, err)


@pytest.mark.parametrize("M,N,K", [(256, 256, 64), (512, 512, 1024), (1000, 784, 320), (2048, 4096, 512)])
@pytest.mark.parametrize("a_mn,b_mn,epi", [(False, False, 0), (False, True, 0), (True, True, 0),
                                           (False, False, 1), (False, True, 3)])
def test_gemm_cta_pair(M, N, K, a_mn, b_mn, epi):
    """CTA-pair (tcgen05.mma.cta_group::2, 256-row tiles) variant."""
    import torch
    A = mk((K, M) if a_mn else (M, K), 11)
    B = mk((K, N) if b_mn else (N, K), 12)
    Af = (A.float().t() if a_mn else A.float())
    Bf = (B.float() if b_mn else B.float().t())
    ref = Af @ Bf
    bias = aux = None
    if epi == 1:
        bias = torch.linspace(-0.5, 0.5, N, device="cuda")
        ref = torch.relu(ref + bias)
    if epi == 3:
        aux = mk((M, N), 13)
        ref = ref * (aux.float() > 0)
    out = run_gemm(A, B, M, N, K, a_mn, b_mn, epi, bias=bias, aux=aux, bn=-256)
    tol = 1e-3 if epi == 0 else 2 ** -7
    err = (out.float() - ref).abs().max().item()
    assert err <= tol * max(1.0, ref.abs().max().item()), err
