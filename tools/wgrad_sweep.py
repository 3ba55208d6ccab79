"""out_wgrad (768 x 768 x 4096, MN-major operands, f32 out) under each tile
choice (DFX_GEMM_FORCE, read per call) vs the planner's split-K plan."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_10802_b200 import kernels as K  # noqa: E402
from tools.gemm_vs_cublas import timeit  # noqa: E402

T, H = 4096, 768
for name, n in [("out_wgrad", 768), ("qkv_wgrad", 2304), ("ffn1_wgrad", 3072)]:
    A = torch.randn(T, n, device="cuda").bfloat16()   # dY [T, n] -> A = dY^T (MN-major)
    B = torch.randn(T, H, device="cuda").bfloat16()   # X  [T, H] -> B = X^T (MN-major)
    d = torch.empty(n, H, device="cuda", dtype=torch.float32)
    for f in ["", "1,64", "1,128", "1,192", "1,256", "2,128", "2,256"]:
        if f:
            os.environ["DFX_GEMM_FORCE"] = f
        else:
            os.environ.pop("DFX_GEMM_FORCE", None)
        us = timeit(lambda: K.gemm(A.t(), B.t(), d))
        print(f"{name:10s} force={f or 'plan':6s} {us:7.2f} us {2 * n * H * T / us / 1e6:7.1f} TF/s")
    os.environ.pop("DFX_GEMM_FORCE", None)
