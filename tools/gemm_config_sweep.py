"""BERT C2 GEMM shapes under forced tile configs (DFX_GEMM_FORCE=cg,bn[,splits]):
max error vs a float reference and graph-replay time per call."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_10802_b200 import kernels as K  # noqa: E402
from tools.gemm_vs_cublas import timeit  # noqa: E402

T, H, F = 4096, 768, 3072
SHAPES = [("qkv", T, 3 * H, H, False, False, torch.bfloat16), ("out", T, H, H, False, False, torch.bfloat16),
          ("ffn1", T, F, H, False, False, torch.bfloat16), ("ffn2", T, H, F, False, False, torch.bfloat16),
          ("ffn2_dgrad", T, F, H, False, True, torch.bfloat16), ("ffn1_dgrad", T, H, F, False, True, torch.bfloat16),
          ("ffn2_wgrad", H, F, T, True, True, torch.float32), ("qkv_wgrad", 3 * H, H, T, True, True, torch.float32),
          ("ffn1_wgrad", F, H, T, True, True, torch.float32), ("out_wgrad", H, H, T, True, True, torch.float32)]
CONFIGS = sys.argv[1:] or ["", "2,256", "2,192", "2,128", "1,256", "1,192", "1,128"]

for name, m, n, k, a_t, b_t, out in SHAPES:
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(k, m, device="cuda", generator=g).bfloat16() if a_t else torch.randn(m, k, device="cuda", generator=g).bfloat16()
    B = torch.randn(k, n, device="cuda", generator=g).bfloat16() if b_t else torch.randn(n, k, device="cuda", generator=g).bfloat16()
    a = A.t() if a_t else A
    b = B.t() if b_t else B
    ref = a.float() @ b.float().t()
    d = torch.empty(m, n, device="cuda", dtype=out)
    line = []
    for f in CONFIGS:
        os.environ["DFX_GEMM_FORCE"] = f
        d.zero_()
        K.gemm(a, b, d)
        torch.cuda.synchronize()
        err = ((d.float() - ref).abs().max() / ref.abs().max()).item()
        us = timeit(lambda: K.gemm(a, b, d))
        line.append(f"[{f or 'auto'}] {us:6.2f}us {2 * m * n * k / us / 1e6:6.0f}TF e={err:.1e}")
    print(f"{name:11s} " + " | ".join(line), flush=True)
os.environ.pop("DFX_GEMM_FORCE", None)
