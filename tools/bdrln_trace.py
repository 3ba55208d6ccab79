"""Per-CTA timeline of the one-wave BDRLN backward (debug hook
dfx_debug_bdrln_trace): 0 start (after pdl wait), 1 mean, 2 rstd, 3 m1/m2,
4 output pass done, 5 after the first CTA barrier, 6 dbias/dgamma column sums,
7 exit — mean µs from each CTA's start, and the kernel span."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_10802_b200 import _lib  # noqa: E402
from paper_2110_10802_b200 import kernels as K  # noqa: E402

T, H = int(os.environ.get("BDRLN_T", "4096")), 768
lib = _lib.load()
fn = lib.dfx_debug_bdrln_trace
fn.argtypes = [ctypes.c_void_p]
bf = torch.bfloat16
dy = torch.randn(T, H, device="cuda").to(bf)
s = torch.randn(T, H, device="cuda").to(bf)
gamma = torch.randn(H, device="cuda")
keep = K.pack_keep_bits((torch.rand(T, H, device="cuda") > 0.1).to(torch.uint8))
ds, dh = torch.empty_like(dy), torch.empty_like(dy)
ws = torch.empty(8 << 20, device="cuda", dtype=torch.uint8)
run = lambda: K.bdrln_bwd(dy, s, gamma, keep, 1 / 0.9, 1e-12, ds=ds, dh=dh, ws=ws)  # noqa: E731
for _ in range(3):
    run()
tr = torch.zeros(400 * 8, dtype=torch.int64, device="cuda")
fn(tr.data_ptr())
run()
torch.cuda.synchronize()
fn(None)
t = tr.view(400, 8).cpu().double()
t = t[t[:, 0] > 0]
rel = (t - t[:, :1]) / 1e3
print("CTAs", t.shape[0], "mean phase ends (us from CTA start):", [round(rel[:, i].mean().item(), 2) for i in range(8)])
print("kernel span (first start -> last exit) us:", round((t[:, 7].max() - t[:, 0].min()).item() / 1e3, 2),
      "start spread us:", round((t[:, 0].max() - t[:, 0].min()).item() / 1e3, 2))
