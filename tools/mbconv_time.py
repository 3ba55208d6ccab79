"""C3 MBConv block (N=96, 112x112, C=96, bf16, stride 1) fwd+bwd timed as a
CUDA graph (device time per step, L2 flushed between replays) with a
per-kernel ncu-free breakdown via event pairs around each library call."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_10802_b200 import kernels as K  # noqa: E402
from paper_2110_10802_b200.mbconv import MBConvBlock, MBConvConfig  # noqa: E402

N, HW, C = int(os.environ.get("MB_N", 96)), 112, 96
blk = MBConvBlock(MBConvConfig(channels=C, dtype=torch.bfloat16), device="cuda", seed=1)
x = torch.randn(N, HW, HW, C, device="cuda").bfloat16()
dy = torch.randn(N, HW, HW, C, device="cuda").bfloat16()


def step():
    blk.forward(x)
    blk.backward(dy)


s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3):
        step()
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for _ in range(10):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
ms = ts[len(ts) // 2]
elems = N * HW * HW * C
print(f"MBConv C3 fwd+bwd: {ms * 1e3:.1f} us/step ({N / ms * 1e3:.0f} img/s); "
      f"6 compulsory passes-equivalent {6 * elems * 2 / 1e6:.0f} MB fwd+bwd min traffic")
timer = K.KernelTimer()
with timer:
    step()
torch.cuda.synchronize()
for r in timer.summary():
    us = r["ms"] * 1e3 / r["calls"]
    print(f"  {r['label']:28s} {us:8.1f} us  {r['work'] / r['calls'] / (us * 1e-6) / 1e9:7.0f} GB/s (algorithmic)")
