"""Locate a gradient mismatch in the EfficientNet-B0 step: per-block input
gradients of our path vs torch fp32 autograd (retain_grad), f32 small config."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

from paper_2110_10802_b200 import efficientnet as E  # noqa: E402

torch.backends.cudnn.allow_tf32 = False
torch.backends.cuda.matmul.allow_tf32 = False
net = E.EfficientNetB0(E.EffNetConfig(image=32, classes=16, width=0.25, dtype=torch.float32), seed=3)
g = torch.Generator(device="cpu").manual_seed(0)
x = torch.randn(4, 32, 32, 3, generator=g).cuda()
labels = torch.randint(0, 16, (4,), generator=g, dtype=torch.int32).cuda()
rec = {}
orig = E._Block.backward


def bwd(self, do):
    rec[self.p + "do"] = do.clone()
    dx = orig(self, do)
    rec[self.p + "dx"] = dx.clone()
    rec[self.p + "da"] = self.mb._bufs[tuple(self.a.shape)]["dx"].clone()
    return dx


E._Block.backward = bwd
net.forward(x, labels)
net.backward()
torch.cuda.synchronize()

c = net.cfg
P = {k: v.detach().clone().requires_grad_(True) for k, v in net.master.views.items()}
xx = x.float().permute(0, 3, 1, 2)


def bn(t, gg, b):
    return F.batch_norm(t, None, None, gg, b, training=True, eps=c.eps)


w0 = P["stem.w"][:, :27].reshape(c.stem, 3, 3, 3).permute(0, 3, 1, 2)
h = F.silu(bn(F.conv2d(xx, w0, stride=2, padding=1), P["stem.g"], P["stem.b"]))
T = {}
for i, (e, k, s, ci, cx, co, se) in enumerate(c.blocks()):
    p, inp = f"b{i}.", h
    inp.retain_grad()
    T[p + "dx"] = inp
    if e != 1:
        h = F.silu(bn(F.conv2d(h, P[p + "we"][:, :, None, None]), P[p + "g1"], P[p + "b1"]))
    h.retain_grad()
    T[p + "da"] = h
    z = F.conv2d(h, P[p + "wdw"].permute(2, 0, 1)[:, None], stride=s, padding=k // 2, groups=cx)
    a = F.silu(bn(z, P[p + "g"], P[p + "b"]))
    r = F.silu(a.mean((2, 3)) @ P[p + "wr"].t() + P[p + "br"])
    gate = torch.sigmoid(r @ P[p + "wse"].t() + P[p + "bse"])
    o = bn(F.conv2d(a * gate[:, :, None, None], P[p + "wp"][:, :, None, None]), P[p + "g3"], P[p + "b3"])
    h = o + inp if (s == 1 and ci == co) else o
    h.retain_grad()
    T[p + "do"] = h
h2 = F.silu(bn(F.conv2d(h, P["head.w"][:, :, None, None]), P["head.g"], P["head.b"]))
logits = h2.mean((2, 3)) @ P["fc.w"].t() + P["fc.b"]
F.cross_entropy(logits, labels.long()).backward()
for i in reversed(range(len(c.blocks()))):
    for nm in ("do", "da", "dx"):
        key = f"b{i}.{nm}"
        mine = rec[key].permute(0, 3, 1, 2)
        ref = T[key].grad
        err = ((mine - ref).abs().max() / ref.abs().max()).item()
        print(f"{key:8s} rel-to-max err {err:.2e}  max|ref| {ref.abs().max().item():.2e}")
for k in ("head.w", "fc.w", "b15.wp", "b15.wdw", "b15.g", "b15.wr", "b15.we"):
    if k in P:
        ref = P[k].grad
        print(k, ((net.grad[k] - ref).abs().max() / ref.abs().max()).item())
