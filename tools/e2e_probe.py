"""Where the BERT C2 end-to-end step time goes: back-to-back graph replays
alone vs the pipelined host-buffer step (H2D inputs + replay + D2H dx), with
and without each copy direction.  Prints ms per step for each variant."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_10802_b200 import kernels as K  # noqa: E402
from paper_2110_10802_b200.bert import BertEncoderLayer, BertLayerConfig  # noqa: E402

B, S, H, NH = 8, 512, 768, 12
T = B * S
layer = BertEncoderLayer(BertLayerConfig(dtype=torch.bfloat16), device="cuda", seed=1)
g = torch.Generator().manual_seed(0)
u8 = lambda *s: (torch.rand(*s, generator=g) >= 0.1).to(torch.uint8)  # noqa: E731
host = {k: v.pin_memory() for k, v in dict(
    x=torch.randn(T, H, generator=g).bfloat16(), dout=torch.randn(T, H, generator=g).bfloat16(),
    add_mask=torch.zeros(B, S), keep_attn=K.pack_keep_bits(u8(B, NH, S, S)),
    keep1=K.pack_keep_bits(u8(T, H)), keep2=K.pack_keep_bits(u8(T, H))).items()}
dx = torch.empty(T, H, dtype=torch.bfloat16).pin_memory()
lr = 1e-4
dev = layer.device_inputs(B, S)
for k, v in host.items():
    dev[k].copy_(v)
cs = layer.capture_step(B, S, lr)


def timed(fn, n=100):
    for _ in range(5):
        fn()
    layer.finish_host()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    layer.finish_host()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


print("replay only        ms", round(timed(cs.replay), 4))
print("async h2d+d2h      ms", round(timed(lambda: layer.train_step_host_async(host, lr=lr, dx_host=dx)), 4))
print("async h2d only     ms", round(timed(lambda: layer.train_step_host_async(host, lr=lr, dx_host=None)), 4))
h2d = torch.cuda.Stream()
print("h2d copies alone   ms", round(timed(lambda: [dev[k].copy_(v, non_blocking=True) for k, v in host.items()]), 4))
