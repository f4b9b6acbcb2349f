"""Runs one GEMM variant a few times (for ncu --set full)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
from test_gpu_gemm import run_gemm, mk
M, N, K = 2048, 4096, 4096
bn = int(sys.argv[1]) if len(sys.argv) > 1 else -256
X = mk((M, K), 1); W = mk((N, K), 2)
bias = torch.zeros(N, device="cuda")
outb = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
for _ in range(4):
    run_gemm(X, W, M, N, K, False, False, 1, bias=bias, out=outb, bn=bn)
torch.cuda.synchronize()
print("ok")
