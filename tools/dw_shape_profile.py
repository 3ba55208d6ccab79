"""One MBConv block at a chosen EfficientNet-B0 shape (default b12: 96 x 7x7 x
1152, k5, stride 1), bf16 fwd+bwd a few times — for ncu captures of the
depthwise ring kernels at small maps.  Usage: python tools/dw_shape_profile.py [H C k s]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_10802_b200.mbconv import MBConvBlock, MBConvConfig  # noqa: E402

H, C, k, s = (int(a) for a in sys.argv[1:5]) if len(sys.argv) >= 5 else (7, 1152, 5, 1)
N = int(os.environ.get("DW_N", 96))
blk = MBConvBlock(MBConvConfig(channels=C, se=max(1, C // 24), stride=s, pads=(k // 2,) * 4, ksize=k, eps=1e-3,
                               momentum=0.9, dtype=torch.bfloat16), seed=1)
x = torch.randn(N, H, H, C, device="cuda").bfloat16()
y = blk.forward(x)
dy = torch.randn_like(y)
for _ in range(3):
    blk.forward(x)
    blk.backward(dy)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    blk.forward(x)
    blk.backward(dy)
b.record()
torch.cuda.synchronize()
print(f"H={H} C={C} k={k} s={s}: {a.elapsed_time(b) / 10 * 1e3:.1f} us fwd+bwd (eager)")
