"""Cost of the fused epilogues on the BERT FFN shapes: plain GEMM vs
bias+GELU (+ pre-activation stash) vs GELU-backward (aux read), isolated."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_10802_b200 import _lib  # noqa: E402
from paper_2110_10802_b200 import kernels as K  # noqa: E402
from tools.gemm_vs_cublas import timeit  # noqa: E402

T, H, F = 4096, 768, 3072
a = torch.randn(T, H, device="cuda").bfloat16()
w1 = torch.randn(F, H, device="cuda").bfloat16()
bias = torch.randn(F, device="cuda")
g = torch.empty(T, F, device="cuda", dtype=torch.bfloat16)
pre = torch.empty_like(g)
fl = 2.0 * T * F * H
for name, fn in [("plain", lambda: K.gemm(a, w1, g)),
                 ("bias", lambda: K.gemm(a, w1, g, _lib.EPI_BIAS, bias=bias)),
                 ("bias+gelu", lambda: K.gemm(a, w1, g, _lib.EPI_BIAS_GELU, bias=bias)),
                 ("bias+gelu+stash", lambda: K.gemm(a, w1, g, _lib.EPI_BIAS_GELU, bias=bias, aux_out=pre)),
                 ("gelu_bwd(aux)", lambda: K.gemm(a, w1, g, _lib.EPI_GELU_BWD, aux=pre))]:
    us = timeit(fn)
    print(f"{name:18s} {us:7.2f} us {fl / us / 1e6:7.1f} TF/s")
