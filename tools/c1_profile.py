"""Per-call-site times of the C1 step (BERT-base fp32, B=2, S=128)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_10802_b200 import kernels as K  # noqa: E402
from paper_2110_10802_b200.bert import BertEncoderLayer, BertLayerConfig  # noqa: E402

B, S = 2, 128
layer = BertEncoderLayer(BertLayerConfig(dtype=torch.float32), seed=3)
dev = layer.device_inputs(B, S)
dev["x"].normal_()
dev["dout"].normal_()
dev["add_mask"].zero_()
for k in ("keep_attn", "keep1", "keep2"):
    dev[k].copy_((torch.rand(dev[k].shape, device="cuda") > 0.1).to(dev[k].dtype))
timer = K.KernelTimer()
cs, inst = layer.capture_step(B, S, 1e-4, timer)
for _ in range(3):
    inst.replay()
torch.cuda.synchronize()
timer.totals = {}
for _ in range(5):
    inst.replay()
    timer.collect()
rows = timer.summary()
tot = sum(r["ms"] for r in rows) / 5
print(f"instrumented {tot * 1e3:.1f} us")
for r in rows:
    ms = r["ms"] / 5
    print(f"{r['label']:34s} {ms * 1e3:8.1f} us  {r['kind']}")
