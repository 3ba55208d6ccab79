"""One of our GEMMs and cuBLAS's on the same shape (for a side-by-side ncu
capture): python tools/gemm_ncu_pair.py M N K"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_10802_b200 import kernels as K  # noqa: E402

m, n, k = (int(x) for x in sys.argv[1:4])
a = torch.randn(m, k, device="cuda").bfloat16()
b = torch.randn(n, k, device="cuda").bfloat16()
d = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    K.gemm(a, b, d)
    torch.matmul(a, b.t(), out=d)
torch.cuda.synchronize()
K.gemm(a, b, d)
torch.matmul(a, b.t(), out=d)
torch.cuda.synchronize()
