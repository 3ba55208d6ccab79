import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2110_10802_b200 import kernels as K
from tools.gemm_vs_cublas import timeit
x = torch.randn(4096, 3072, device="cuda").bfloat16()
out = torch.empty(3072, device="cuda")
us = timeit(lambda: K.colsum(x, out))
print(f"colsum 4096x3072 bf16: {us:.2f} us {4096*3072*2/us/1e3:.0f} GB/s; err {(out - x.float().sum(0)).abs().max().item():.3e}")
