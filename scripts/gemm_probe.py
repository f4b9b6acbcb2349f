"""Times the tcgen05 GEMM on the C3 shapes (b=2048 rows per GPU, 4096x4096
layers) with CUDA events; prints TFLOP/s per variant."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
from test_gpu_gemm import run_gemm, mk

M, N, K = 2048, 4096, 4096
X = mk((M, K), 1); W = mk((N, K), 2); dY = mk((M, N), 3)
bias = torch.zeros(N, device="cuda")
outb = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
outf = torch.empty((N, K), dtype=torch.float32, device="cuda")
cases = {
  "fwd  X.W^T (K-maj,K-maj) bias+relu": lambda bn: run_gemm(X, W, M, N, K, False, False, 1, bias=bias, out=outb, bn=bn),
  "dX   dY.W  (K-maj,MN-maj) drelu   ": lambda bn: run_gemm(dY, W, M, K, N, False, True, 3, aux=X, out=outb, bn=bn),
  "dW   dY^T.X (MN,MN) f32           ": lambda bn: run_gemm(dY, X, N, K, M, True, True, 0, out=outf, bn=bn),
}
flop = 2.0 * M * N * K
for name, fn in cases.items():
    for bn in (128, 256, -256):
        for _ in range(3): fn(bn)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); s.record()
        it = 20
        for _ in range(it): fn(bn)
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / it
        print(f"{name} bn={bn}: {ms*1e3:8.1f} us  {flop/ms/1e9:8.1f} TFLOP/s")
a = X.float(); b = W.float()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3): torch.matmul(X, W.t())
torch.cuda.synchronize(); s.record()
for _ in range(20): torch.matmul(X, W.t())
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 20
print(f"cuBLAS bf16 X.W^T: {ms*1e3:8.1f} us  {flop/ms/1e9:8.1f} TFLOP/s")
