"""Standalone timing of the EfficientNet-B0 (C5, N=96, 224²) project / expand
1x1-conv weight-gradient GEMMs: dW[Cout, Cin] = Σ_pixels dY[p, Cout] · X[p, Cin]
(A = dYᵀ and B = Xᵀ read MN-major, f32 out), CUDA-graph replay."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_10802_b200 import kernels as K  # noqa: E402
from tools.gemm_vs_cublas import timeit  # noqa: E402

N = 96
# (name, pixels per image, Cin, Cout) of the project convs (expanded -> out)
SHAPES = [("b0.project", 112 * 112, 32, 16), ("b1.project", 56 * 56, 96, 24), ("b2.project", 56 * 56, 144, 24),
          ("b4.project", 28 * 28, 240, 40), ("b9.project", 14 * 14, 672, 112), ("b12.project", 7 * 7, 1152, 192),
          ("b15.project", 7 * 7, 1152, 320), ("b1.expand", 112 * 112, 16, 96), ("b12.expand", 7 * 7, 192, 1152)]
for name, hw, cin, cout in SHAPES:
    P = N * hw
    dy = torch.randn(P, cout, device="cuda").bfloat16()
    x = torch.randn(P, cin, device="cuda").bfloat16()
    d = torch.empty(cout, cin, device="cuda", dtype=torch.float32)
    us = timeit(lambda: K.gemm(dy.t(), x.t(), d))
    byts = P * (cin + cout) * 2
    print(f"{name:12s} M={cout:5d} N={cin:5d} K={P:8d} {us:8.2f} us {2 * P * cin * cout / us / 1e6:7.1f} TF/s "
          f"{byts / us / 1e3:7.1f} GB/s")
