"""EfficientNet-B0 1x1-conv GEMMs (M = pixels, tiny N or K) under each tile
choice vs cuBLAS: the memory-bound skinny shapes of the early blocks."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_10802_b200 import kernels as K  # noqa: E402
from tools.gemm_vs_cublas import timeit  # noqa: E402

M1, M2 = 96 * 112 * 112, 96 * 56 * 56
for name, m, n, k in [("b0.project", M1, 16, 32), ("b1.expand", M1, 96, 16), ("b1.exp_dgrad", M1, 16, 96),
                      ("b1.project", M2, 24, 96), ("b2.expand", M2, 144, 24), ("b2.project", M2, 24, 144)]:
    a = torch.randn(m, k, device="cuda").bfloat16()
    b = torch.randn(n, k, device="cuda").bfloat16()
    d = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    byts = (m * k + m * n + n * k) * 2
    res = []
    for f in ["", "1,64", "1,128", "2,128", "1,256"]:
        if f:
            os.environ["DFX_GEMM_FORCE"] = f
        else:
            os.environ.pop("DFX_GEMM_FORCE", None)
        us = timeit(lambda: K.gemm(a, b, d), reps=10)
        res.append(f"{f or 'plan'}={us:.1f}")
    os.environ.pop("DFX_GEMM_FORCE", None)
    cub = timeit(lambda: torch.matmul(a, b.t(), out=d), reps=10)
    print(f"{name:13s} {m}x{n}x{k} {byts / 1e6:6.1f} MB | " + " ".join(res) + f" | cuBLAS {cub:.1f} us"
          f" | ideal {byts / 6.5e6:.1f} us")
