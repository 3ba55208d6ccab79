"""Per-CTA timeline of one tensor-core GEMM (debug build hook
dfx_debug_gemm_trace): kernel entry, setup done, first stage landed, MMA
tile completions, epilogue start/end per tile, exit — all in ns relative to
the earliest entry.  Usage: python tools/gemm_trace.py M N K [cg,bn]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 4:
    os.environ["DFX_GEMM_FORCE"] = sys.argv[4]
import torch  # noqa: E402

from paper_2110_10802_b200 import _lib  # noqa: E402
from paper_2110_10802_b200 import kernels as K  # noqa: E402

m, n, k = (int(v) for v in sys.argv[1:4])
lib = _lib.load()
fn = lib.dfx_debug_gemm_trace
fn.argtypes = [ctypes.c_void_p]
a = torch.randn(m, k, device="cuda").bfloat16()
b = torch.randn(n, k, device="cuda").bfloat16()
d = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
epi = os.environ.get("GT_EPI", "none")  # none | gelu (bias + GELU + pre-activation stash, the FFN1 forward)
bias = torch.randn(n, device="cuda") * 0.1
pre = torch.empty_like(d)


def run():
    if epi == "gelu":
        K.gemm(a, b, d, _lib.EPI_BIAS_GELU, bias=bias, aux_out=pre)
    else:
        K.gemm(a, b, d, beta=float(os.environ.get("GT_BETA", "1.0")))


for _ in range(3):
    run()
tr = torch.zeros(148 * 32, dtype=torch.int64, device="cuda")
fn(tr.data_ptr())
run()
torch.cuda.synchronize()
fn(None)
t = tr.view(148, 32).cpu()
t0 = t[:, 0][t[:, 0] > 0].min().item()
rel = lambda v: (v - t0) / 1e3 if v > 0 else float("nan")  # noqa: E731
print("cta  entry  setup  first  | mma_done...  | epi_start... | epi_end... | exit   (us)")
for c in list(range(0, 148, 16)) + [147]:
    r = t[c].tolist()
    if r[0] == 0:
        continue
    mma = [f"{rel(v):6.2f}" for v in r[3:11] if v > 0]
    es = [f"{rel(v):6.2f}" for v in r[11:19] if v > 0]
    ee = [f"{rel(v):6.2f}" for v in r[19:27] if v > 0]
    print(f"{c:3d} {rel(r[0]):6.2f} {rel(r[1]):6.2f} {rel(r[2]):6.2f} | {' '.join(mma)} | {' '.join(es)} | "
          f"{' '.join(ee)} | {rel(r[27]):6.2f} | t0 epi: ld {rel(r[28]):6.2f} units {rel(r[29]):6.2f} {rel(r[30]):6.2f} {rel(r[31]):6.2f}")
