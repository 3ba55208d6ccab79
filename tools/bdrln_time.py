"""CUDA-graph timing of the BDRLN forward / backward kernels at the C2 shape
(T = 4096 rows x 768, bf16, dropout keep flags) with achieved HBM GB/s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_10802_b200 import kernels as K  # noqa: E402
from tools.gemm_vs_cublas import timeit  # noqa: E402

T, H = int(os.environ.get("BDRLN_T", "4096")), 768
g = torch.Generator(device="cuda").manual_seed(0)
bf = torch.bfloat16
h = torch.randn(T, H, device="cuda", generator=g).to(bf)
res = torch.randn(T, H, device="cuda", generator=g).to(bf)
bias = torch.randn(H, device="cuda", generator=g)
gamma = torch.randn(H, device="cuda", generator=g)
beta = torch.randn(H, device="cuda", generator=g)
keep = (torch.rand(T, H, device="cuda", generator=g) > 0.1).to(torch.uint8)
y = torch.empty_like(h)
s = torch.empty_like(h)
dy = torch.randn(T, H, device="cuda", generator=g).to(bf)
ds = torch.empty_like(h)
dh = torch.empty_like(h)
ws = torch.empty(8 << 20, device="cuda", dtype=torch.uint8)
fwd = lambda: K.bdrln_fwd(h, bias, keep, 1 / 0.9, res, gamma, beta, 1e-12, y=y, s=s)  # noqa: E731
bwd = lambda: K.bdrln_bwd(dy, s, gamma, keep, 1 / 0.9, 1e-12, ds=ds, dh=dh, ws=ws)  # noqa: E731
if os.environ.get("BDRLN_ONLY"):
    fwd(); bwd(); torch.cuda.synchronize(); sys.exit(0)  # noqa: E702
for name, fn, nbytes in [("fwd", fwd, T * H * (2 + 2 + 2 + 2 + 1)), ("bwd", bwd, T * H * (2 + 2 + 2 + 2 + 1))]:
    us = timeit(fn)
    print(f"bdrln {name}: {us:6.2f} us  {nbytes / us / 1e3:7.1f} GB/s (algorithmic {nbytes / 1e6:.1f} MB)")
