"""Throughput sweep of the tcgen05 GEMM over shapes/layouts (CUDA events,
20 back-to-back launches after warm-up).  Prints TFLOP/s per case and the
plan the dispatcher picked; used to tune the tile planner."""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_10802_b200 import kernels as K  # noqa: E402
from paper_2110_10802_b200._lib import EPI_BIAS, EPI_BIAS_GELU, EPI_NONE  # noqa: E402


def run(m, n, k, la="k", lb="k", out=torch.bfloat16, epi=EPI_NONE, reps=20):
    a = torch.randn(m, k, device="cuda").bfloat16() if la == "k" else torch.randn(k, m, device="cuda").bfloat16().t()
    b = torch.randn(n, k, device="cuda").bfloat16() if lb == "k" else torch.randn(k, n, device="cuda").bfloat16().t()
    d = torch.empty(m, n, device="cuda", dtype=out)
    bias = torch.zeros(n, device="cuda")
    pre = torch.empty_like(d)
    kw = {}
    if epi == EPI_BIAS:
        kw = dict(bias=bias)
    elif epi == EPI_BIAS_GELU:
        kw = dict(bias=bias, aux_out=pre)
    for _ in range(3):
        K.gemm(a, b, d, epi, **kw)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        K.gemm(a, b, d, epi, **kw)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return 2 * m * n * k / ms / 1e9, ms * 1e3


cases = [
    ("qkv fwd", 4096, 2304, 768, "k", "k", torch.bfloat16, EPI_BIAS),
    ("ffn1 fwd", 4096, 3072, 768, "k", "k", torch.bfloat16, EPI_BIAS_GELU),
    ("ffn1 fwd noepi", 4096, 3072, 768, "k", "k", torch.bfloat16, EPI_NONE),
    ("ffn2 fwd", 4096, 768, 3072, "k", "k", torch.bfloat16, EPI_NONE),
    ("K=6144", 4096, 3072, 6144, "k", "k", torch.bfloat16, EPI_NONE),
    ("8192^3", 8192, 8192, 8192, "k", "k", torch.bfloat16, EPI_NONE),
    ("wgrad ffn", 3072, 768, 4096, "m", "n", torch.float32, EPI_NONE),
    ("dgrad ffn2", 4096, 3072, 768, "k", "n", torch.bfloat16, EPI_NONE),
]
for name, m, n, k, la, lb, out, epi in cases:
    tf, us = run(m, n, k, la, lb, out, epi)
    print(f"{name:16s} {m}x{n}x{k} {la}{lb} -> {tf:7.1f} TFLOP/s  {us:8.1f} us")
