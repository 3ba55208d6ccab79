"""EfficientNet-B0 training step (config C5) against a torch fp32 autograd
composition of the same operators with the same parameters (SURVEY §8d C5:
"the full net against torch fp32 at small batch").  The per-block math is
pinned to the dfir oracle by test_gpu_mbconv.py / test_gpu_norms.py."""

import pytest
import torch
import torch.nn.functional as F

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _net(**kw):
    from paper_2110_10802_b200.efficientnet import EfficientNetB0, EffNetConfig

    return EfficientNetB0(EffNetConfig(**kw), device="cuda", seed=3)


def torch_reference(net, x_nhwc, labels, dtype=torch.float64):
    """On the host CPU (no TF32 / fast-math paths): float64 = the exact
    reference; float32 = the noise floor of an fp32 evaluation order."""
    c = net.cfg
    P = {k: v.detach().to(dtype).cpu().requires_grad_(True) for k, v in net.master.views.items()}
    x = x_nhwc.to(dtype).cpu().permute(0, 3, 1, 2)
    labels = labels.cpu()

    def bn(t, g, b):
        return F.batch_norm(t, None, None, g, b, training=True, eps=c.eps)

    w0 = P["stem.w"][:, :27].reshape(c.stem, 3, 3, 3).permute(0, 3, 1, 2)
    h = F.silu(bn(F.conv2d(x, w0, stride=2, padding=1), P["stem.g"], P["stem.b"]))
    for i, (e, k, s, ci, cx, co, se) in enumerate(c.blocks()):
        p, inp = f"b{i}.", h
        if e != 1:
            h = F.silu(bn(F.conv2d(h, P[p + "we"][:, :, None, None]), P[p + "g1"], P[p + "b1"]))
        z = F.conv2d(h, P[p + "wdw"].permute(2, 0, 1)[:, None], stride=s, padding=k // 2, groups=cx)
        a = F.silu(bn(z, P[p + "g"], P[p + "b"]))
        r = F.silu(a.mean((2, 3)) @ P[p + "wr"].t() + P[p + "br"])
        gate = torch.sigmoid(r @ P[p + "wse"].t() + P[p + "bse"])
        o = bn(F.conv2d(a * gate[:, :, None, None], P[p + "wp"][:, :, None, None]), P[p + "g3"], P[p + "b3"])
        h = o + inp if (s == 1 and ci == co) else o
    h = F.silu(bn(F.conv2d(h, P["head.w"][:, :, None, None]), P["head.g"], P["head.b"]))
    logits = h.mean((2, 3)) @ P["fc.w"].t() + P["fc.b"]
    loss = F.cross_entropy(logits, labels.long())
    loss.backward()
    return loss.item(), {k: v.grad for k, v in P.items()}


def _errs(net, ref_grads, metric):
    """The reference's comparator (interp.compare_outputs, interp.py:1332-1352)."""
    return {k: metric(net.grad[k].double().cpu().numpy(), g.double().numpy()) for k, g in ref_grads.items()}


def test_f32_small_matches_torch():
    """Width 0.25, 128x128 images, batch 4, f32 path: every parameter gradient
    against float64, at the reference's 1e-4 bar or within 10x of what an
    fp32 evaluation in another summation order (torch CPU fp32) achieves — the
    BatchNorms over few elements in the late stages amplify rounding."""
    net = _net(image=128, classes=16, width=0.25, dtype=torch.float32)
    g = torch.Generator(device="cpu").manual_seed(0)
    x = torch.randn(4, 128, 128, 3, generator=g).cuda()
    labels = torch.randint(0, 16, (4,), generator=g, dtype=torch.int32).cuda()
    loss = net.forward(x, labels)
    net.backward()
    torch.cuda.synchronize()
    want, grads = torch_reference(net, x, labels)
    _, grads32 = torch_reference(net, x, labels, torch.float32)
    errs = _errs(net, grads, O.compare)
    floor = {k: O.compare(grads32[k].double().numpy(), grads[k].numpy()) for k in grads}
    assert abs(loss.item() - want) <= 1e-4 * max(1.0, abs(want)), (loss.item(), want)
    bad = {k: (v, floor[k]) for k, v in errs.items() if v > max(1e-4, 10 * floor[k])}
    assert not bad, sorted(bad.items(), key=lambda kv: -kv[1][0])[:12]


def test_bf16_full_width_matches_torch():
    """Full B0 width (every real channel count, k3/k5, stride 1/2), 160x160
    images, batch 4, bf16 storage vs float64 on the same parameters."""
    net = _net(image=160, classes=1000, dtype=torch.bfloat16)
    g = torch.Generator(device="cpu").manual_seed(1)
    x = torch.randn(4, 160, 160, 3, generator=g).bfloat16().cuda()
    labels = torch.randint(0, 1000, (4,), generator=g, dtype=torch.int32).cuda()
    loss = net.forward(x, labels)
    net.backward()
    torch.cuda.synchronize()
    want, grads = torch_reference(net, x, labels)
    assert abs(loss.item() - want) <= 2e-2 * max(1.0, abs(want))
    errs = _errs(net, grads, O.compare_scaled)
    # the bf16 bar (2e-2) on the layers whose gradient passes through few bf16
    # stores; deeper into the backward the rounding of 16 blocks of bf16
    # activations / gradients accumulates (each block alone meets 2e-2:
    # test_gpu_mbconv.py, test_gpu_norms.py), so the early layers get 0.1
    late = ("fc.", "head.", "b15.", "b14.", "b13.")
    bad = {k: v for k, v in errs.items() if v > (2e-2 if k.startswith(late) else 0.1)}
    assert not bad, sorted(bad.items(), key=lambda kv: -kv[1])[:12]


def test_graph_step_equals_eager():
    """The CUDA-graph step (bench path) computes the same update as eager calls."""
    net = _net(image=64, classes=128, width=0.5, dtype=torch.bfloat16)
    dev = net.device_inputs(4)
    g = torch.Generator(device="cpu").manual_seed(2)
    dev["x"].copy_(torch.randn(4, 64, 64, 3, generator=g).bfloat16())
    dev["labels"].copy_(torch.randint(0, 128, (4,), generator=g, dtype=torch.int32))
    net.forward(dev["x"], dev["labels"])
    net.backward()
    torch.cuda.synchronize()
    eager = net.grad.flat.clone()
    cs = net.capture_step(4, lr=None)
    net.grad.flat.zero_()
    cs.replay()
    torch.cuda.synchronize()
    assert torch.equal(net.grad.flat, eager)


class _RoundBF16(torch.autograd.Function):
    """The bf16 storage model inside a float64 autograd chain: the value is
    rounded where the GPU stores it to HBM, and so is the gradient the GPU
    stores for it in the backward."""

    @staticmethod
    def forward(ctx, t):
        return t.to(torch.bfloat16).to(t.dtype)

    @staticmethod
    def backward(ctx, g):
        return g.to(torch.bfloat16).to(g.dtype)


def _block_reference(net, i, x, do, pr_gpu):
    """One EfficientNet-B0 block (expand 1x1 + BN + swish -> dw + BN + swish ->
    SE -> project 1x1 + BN (+ residual)) in float64 on the host, from the
    GPU's own bf16 block input ``x`` and output gradient ``do``; GEMM weights
    are the bf16 shadow the tensor cores read; every activation the GPU
    stores goes through the bf16 storage model."""
    c = net.cfg
    e, k, s, ci, cx, co, se = c.blocks()[i]
    p = f"b{i}."
    R = _RoundBF16.apply
    f64 = torch.float64
    P = {}
    for name in ("we", "wp"):
        if p + name in net.master.views:
            P[name] = net.wlow[p + name].detach().to(f64).cpu().requires_grad_(True)
    for name in ("g1", "b1", "wdw", "g", "b", "wr", "br", "wse", "bse", "g3", "b3"):
        if p + name in net.master.views:
            P[name] = net.master[p + name].detach().to(f64).cpu().requires_grad_(True)
    xt = x.detach().to(f64).cpu().permute(0, 3, 1, 2).contiguous().requires_grad_(True)

    def bn(t, g, b):
        return F.batch_norm(t, None, None, g, b, training=True, eps=c.eps)

    h = xt
    if e != 1:
        h = R(F.conv2d(h, P["we"][:, :, None, None]))
        h = R(F.silu(bn(h, P["g1"], P["b1"])))
    z = R(F.conv2d(h, P["wdw"].permute(2, 0, 1)[:, None], stride=s, padding=k // 2, groups=cx))
    a = F.silu(bn(z, P["g"], P["b"]))
    r = F.silu(a.mean((2, 3)) @ P["wr"].t() + P["br"])
    gate = torch.sigmoid(r @ P["wse"].t() + P["bse"])
    y = R(a * gate[:, :, None, None])
    pr = R(F.conv2d(y, P["wp"][:, :, None, None]))
    res = s == 1 and ci == co
    o = R(R(bn(pr, P["g3"], P["b3"])) + xt) if res else R(bn(pr, P["g3"], P["b3"]))
    o.backward(do.detach().to(f64).cpu().permute(0, 3, 1, 2))
    # the block output from the GPU's own stored projection (BN3 normalises
    # with statistics of the stored bf16 values, so a 1-ulp flip of pr between
    # an fp32 and an f64 accumulation is amplified by rstd; pinning BN3 on the
    # GPU's pr checks that op at the bf16 bar and pr itself separately)
    with torch.no_grad():
        pg = pr_gpu.detach().to(f64).cpu().permute(0, 3, 1, 2)
        og = R(bn(pg, P["g3"], P["b3"]))
        if res:
            og = R(og + xt)
    return og, pr.detach(), xt.grad, {name: t.grad for name, t in P.items()}


def test_bf16_c5_blocks_pinned_to_f64():
    """VERDICT r01 #1 (C5 at the bf16 bar): every one of the 16 blocks of the
    full-width bf16 EfficientNet-B0 step, fed with the GPU's own block input
    and output gradient, against float64 with the bf16 storage model — block
    output, input gradient and every block parameter gradient at 2e-2."""
    from paper_2110_10802_b200 import efficientnet as E

    net = _net(image=128, classes=1000, dtype=torch.bfloat16)
    rec = {}
    fwd, bwd = E._Block.forward, E._Block.backward
    from paper_2110_10802_b200.norms import BatchNormAct

    bn_fwd = BatchNormAct.forward
    owner = {id(b.bn3): b for b in net.blocks}

    def bnf(self, x, y=None):
        if id(self) in owner:
            rec.setdefault(owner[id(self)], {})["pr"] = x.clone()
        return bn_fwd(self, x, y)

    def f(self, x):
        o = fwd(self, x)
        rec.setdefault(self, {})["x"], rec[self]["o"] = x.clone(), o.clone()
        return o

    def b(self, do):
        dx = bwd(self, do)
        rec[self]["do"], rec[self]["dx"] = do.clone(), dx.clone()
        return dx

    E._Block.forward, E._Block.backward = f, b
    BatchNormAct.forward = bnf
    try:
        g = torch.Generator(device="cpu").manual_seed(4)
        x = torch.randn(4, 128, 128, 3, generator=g).bfloat16().cuda()
        labels = torch.randint(0, 1000, (4,), generator=g, dtype=torch.int32).cuda()
        net.concurrent = False
        net.forward(x, labels)
        net.backward()
        torch.cuda.synchronize()
    finally:
        E._Block.forward, E._Block.backward = fwd, bwd
        BatchNormAct.forward = bn_fwd
    report, bad = {}, {}
    for i, blk in enumerate(net.blocks):
        r = rec[blk]
        o_w, pr_w, dx_w, g_w = _block_reference(net, i, r["x"], r["do"], r["pr"])
        got = {"o": r["o"].double().cpu().permute(0, 3, 1, 2), "pr": r["pr"].double().cpu().permute(0, 3, 1, 2),
               "dx": r["dx"].double().cpu().permute(0, 3, 1, 2)}
        want = {"o": o_w, "pr": pr_w, "dx": dx_w}
        for name, gw in g_w.items():
            got[name] = net.grad[f"b{i}." + name].double().cpu()
            want[name] = gw
        for k_ in got:
            ew = O.compare(got[k_].numpy(), want[k_].numpy())
            sc = O.compare_scaled(got[k_].numpy(), want[k_].numpy())
            report[f"b{i}.{k_}"] = (round(ew, 5), round(sc, 5))
            if ew > 2e-2:
                bad[f"b{i}.{k_}"] = (ew, sc)
    print("C5 blocks vs f64 (element-wise, scaled):", report)
    assert not bad, sorted(bad.items(), key=lambda kv: -kv[1][0])[:12]
