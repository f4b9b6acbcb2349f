"""Times the tcgen05 GEMM on the C3 shapes (b=2048 rows per GPU, 4096x4096
layers): back-to-back launches on one stream bracketed by CUDA events (no
host sync inside the timed loop); prints TFLOP/s per variant vs cuBLAS."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
from test_gpu_gemm import _lib, mk
from paper_1806_02508_b200._lib import check

M, N, K = 2048, 4096, 4096
X = mk((M, K), 1); W = mk((N, K), 2); dY = mk((M, N), 3)
bias = torch.zeros(N, device="cuda")
outb = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
outf = torch.empty((N, K), dtype=torch.float32, device="cuda")
L = _lib()


def launch(A, B, out, m, n, k, a_mn, b_mn, epi, bn, aux=None):
    st = torch.cuda.current_stream().cuda_stream
    check(L.lbbsp_gemm_bf16(A.data_ptr(), B.data_ptr(), out.data_ptr(), m, n, k, int(a_mn), int(b_mn),
                            epi, bias.data_ptr() if epi in (1, 2) else None,
                            aux.data_ptr() if aux is not None else None, 0, 0, None, None, None,
                            None, 0, None, bn, st))


cases = {
    "fwd  X.W^T (K-maj,K-maj) bias+relu": lambda bn: launch(X, W, outb, M, N, K, False, False, 1, bn),
    "dX   dY.W  (K-maj,MN-maj) drelu   ": lambda bn: launch(dY, W, outb, M, K, N, False, True, 3, bn, aux=X),
    "dW   dY^T.X (MN,MN) f32           ": lambda bn: launch(dY, X, outf, N, K, M, True, True, 0, bn),
}
flop = 2.0 * M * N * K


def timeit(fn, it=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / it


for name, fn in cases.items():
    for bn in (128, 256, -256):
        ms = timeit(lambda: fn(bn))
        print(f"{name} bn={bn}: {ms*1e3:8.1f} us  {flop/ms/1e9:8.1f} TFLOP/s")
ms = timeit(lambda: torch.matmul(X, W.t()))
print(f"cuBLAS bf16 X.W^T: {ms*1e3:8.1f} us  {flop/ms/1e9:8.1f} TFLOP/s")
