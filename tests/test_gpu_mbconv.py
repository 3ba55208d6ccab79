"""GPU parity of the MBConv block (dw3x3 + BN(train) + swish + SE), forward
and backward, against the reference's golden vectors and the oracle."""

import ctypes

import numpy as np
import pytest
import torch

from oracle import oracle as O
from golden_util import golden

pytestmark = pytest.mark.gpu

GRADS = ("x", "wdw", "g", "b", "wr", "br", "we", "be")


def _block(C, SE, stride, pads, dtype, eps=1e-3, momentum=0.99, prm=None):
    from paper_2110_10802_b200.mbconv import MBConvBlock, MBConvConfig

    blk = MBConvBlock(MBConvConfig(channels=C, se=SE, stride=stride, pads=tuple(pads), eps=eps,
                                   momentum=momentum, dtype=dtype), seed=5)
    if prm is not None:
        blk.load_params(prm)
    return blk


def _nhwc(a, dtype):
    return torch.as_tensor(np.ascontiguousarray(np.asarray(a).transpose(0, 2, 3, 1)),
                           dtype=torch.float32).to(dtype).cuda().contiguous()


def _nchw(t):
    return t.float().cpu().numpy().astype(np.float64).transpose(0, 3, 1, 2)


def _run(blk, x, dy, dtype):
    y = blk.forward(_nhwc(x, dtype))
    dx = blk.backward(_nhwc(dy, dtype))
    torch.cuda.synchronize()
    return _nchw(y), _nchw(dx)


def _check(errs, tol):
    bad = {k: v for k, v in errs.items() if v > tol}
    assert not bad, f"over {tol}: {bad} (all {errs})"


@pytest.mark.parametrize("name", ["mbconv_s1_f32", "mbconv_s1_f64", "mbconv_s2_f64"])
def test_golden(name):
    """The reference's own forward/backward (tests/golden), run in f32."""
    g = golden(name)
    C, SE, stride = int(g["C"]), int(g["SE"]), int(g["stride"])
    prm = {k: g[k] for k in O.MBCONV_WEIGHTS}
    blk = _block(C, SE, stride, (1, 1, 1, 1), torch.float32, float(g["eps"]), float(g["momentum"]), prm)
    y, dx = _run(blk, g["x"], g["dy"], torch.float32)
    errs = {"y": O.compare(y, g["y"]), "dx": O.compare(dx, g["d_x"]),
            "rm": O.compare(blk.running_mean.cpu().numpy(), g["new_rm"]),
            "rv": O.compare(blk.running_var.cpu().numpy(), g["new_rv"])}
    gr = blk.grads_numpy()
    for k in GRADS[1:]:
        errs[k] = O.compare(gr[k], g["d_" + k])
    _check(errs, 1e-4)


def _rand_case(rng, N, C, H, W, SE):
    prm = {"wdw": 0.3 * rng.standard_normal((C, 1, 3, 3)), "g": 1 + 0.1 * rng.standard_normal(C),
           "b": 0.1 * rng.standard_normal(C), "rm": 0.1 * rng.standard_normal(C),
           "rv": 1 + 0.1 * rng.random(C), "wr": 0.3 * rng.standard_normal((SE, C)),
           "br": 0.1 * rng.standard_normal(SE), "we": 0.3 * rng.standard_normal((C, SE)),
           "be": 0.1 * rng.standard_normal(C)}
    x = rng.standard_normal((N, C, H, W))
    return prm, x


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("stride,pads,hw", [(1, (1, 1, 1, 1), 28), (2, (1, 1, 1, 1), 28),
                                            (1, (1, 0, 0, 1), 17), (2, (0, 0, 1, 1), 19),
                                            (1, (1, 1, 1, 1), 9)])
def test_vs_oracle(dtype, stride, pads, hw):
    rng = np.random.default_rng(hw * 10 + stride)
    N, C, SE = 3, 96 if hw > 9 else 16, 4
    prm, x = _rand_case(rng, N, C, hw, hw, SE)
    if dtype == torch.bfloat16:
        x = O.round_bf16(x).astype(np.float64)
    rnd = (lambda a: O.round_bf16(a).astype(np.float64)) if dtype == torch.bfloat16 else None
    y_w, rm_w, rv_w, cache = O.mbconv_fwd(prm, x, stride, 1e-3, 0.99, rnd=rnd, pads=pads)
    dy = rng.standard_normal(y_w.shape)
    if dtype == torch.bfloat16:
        dy = O.round_bf16(dy).astype(np.float64)
    gw = O.mbconv_bwd(prm, cache, dy)
    blk = _block(C, SE, stride, pads, dtype, prm=prm)
    y, dx = _run(blk, x, dy, dtype)
    errs = {"y": O.compare(y, y_w), "dx": O.compare(dx, gw["x"]),
            "rm": O.compare(blk.running_mean.cpu().numpy(), rm_w),
            "rv": O.compare(blk.running_var.cpu().numpy(), rv_w)}
    gr = blk.grads_numpy()
    for k in GRADS[1:]:
        errs[k] = O.compare(gr[k], gw[k])
    _check(errs, 1e-4 if dtype == torch.float32 else 2e-2)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("stride,hw,C", [(1, 14, 48), (2, 15, 40), (1, 7, 1152 // 8)])
def test_5x5_vs_oracle(dtype, stride, hw, C):
    """5x5 depthwise (EfficientNet-B0 stages 3, 5, 6) through the TMA ring path."""
    rng = np.random.default_rng(hw * 7 + stride + C)
    N, SE, k, pads = 3, 8, 5, (2, 2, 2, 2)
    prm, x = _rand_case(rng, N, C, hw, hw, SE)
    prm["wdw"] = 0.2 * rng.standard_normal((C, 1, k, k))
    if dtype == torch.bfloat16:
        x = O.round_bf16(x).astype(np.float64)
    rnd = (lambda a: O.round_bf16(a).astype(np.float64)) if dtype == torch.bfloat16 else None
    y_w, rm_w, rv_w, cache = O.mbconv_fwd(prm, x, stride, 1e-3, 0.99, rnd=rnd, pads=pads)
    dy = rng.standard_normal(y_w.shape)
    if dtype == torch.bfloat16:
        dy = O.round_bf16(dy).astype(np.float64)
    gw = O.mbconv_bwd(prm, cache, dy)
    from paper_2110_10802_b200.mbconv import MBConvBlock, MBConvConfig

    blk = MBConvBlock(MBConvConfig(channels=C, se=SE, stride=stride, pads=pads, ksize=k, dtype=dtype), seed=5)
    blk.load_params(prm)
    y, dx = _run(blk, x, dy, dtype)
    errs = {"y": O.compare(y, y_w), "dx": O.compare(dx, gw["x"]),
            "rm": O.compare(blk.running_mean.cpu().numpy(), rm_w)}
    gr = blk.grads_numpy()
    for kk in GRADS[1:]:
        errs[kk] = O.compare(gr[kk], gw[kk])
    _check(errs, 1e-4 if dtype == torch.float32 else 2e-2)


def test_syncbn_merge_equals_global_batch():
    """SyncBN statistics: merging the per-rank (count, mean, M2) sets of two
    half batches equals BatchNorm over the concatenated batch."""
    from paper_2110_10802_b200 import _lib

    rng = np.random.default_rng(0)
    N, C, H = 8, 32, 20
    blk = _block(C, 4, 1, (1, 1, 1, 1), torch.float32)
    x = _nhwc(rng.standard_normal((N, C, H, H)), torch.float32)
    lib = _lib.load()
    pads = (ctypes.c_int * 4)(1, 1, 1, 1)
    st = torch.cuda.current_stream().cuda_stream

    def stats(xx):
        z = torch.empty_like(xx)
        loc = torch.empty(3, C, device="cuda")
        ws = torch.empty(lib.dfx_mbconv_workspace(xx.shape[0], H, H, C, 1, 3, pads, 4), dtype=torch.uint8,
                         device="cuda")
        _lib.check(lib.dfx_mbconv_fwd_stats(0, xx.shape[0], H, H, C, 1, 3, pads, xx.data_ptr(),
                                            blk.master["wdw"].data_ptr(), z.data_ptr(), loc.data_ptr(),
                                            ws.data_ptr(), ws.numel(), st))
        return loc

    full = stats(x)
    sets = torch.stack([stats(x[: N // 2].contiguous()), stats(x[N // 2:].contiguous())])
    out = {}
    for nm, s_, n in (("one", full, 1), ("two", sets, 2)):
        mean, var, rstd = (torch.empty(C, device="cuda") for _ in range(3))
        _lib.check(lib.dfx_bn_finalize(C, n, s_.data_ptr(), 1e-3, 0.9, mean.data_ptr(), var.data_ptr(),
                                       rstd.data_ptr(), None, None, st))
        out[nm] = (mean.cpu().numpy(), var.cpu().numpy())
    torch.cuda.synchronize()
    np.testing.assert_allclose(out["one"][0], out["two"][0], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(out["one"][1], out["two"][1], rtol=1e-5, atol=1e-6)


def test_c3_full_size_against_torch_fp32():
    """Config C3 (N=96, 112x112, C=96, f32) against a torch fp32 composition of
    the same operators on the GPU (conv2d groups=C, batch_norm, SE MLP)."""
    import torch.nn.functional as F

    N, C, H, SE = 96, 96, 112, 4
    g = torch.Generator(device="cpu").manual_seed(7)
    blk = _block(C, SE, 1, (1, 1, 1, 1), torch.float32)
    x = torch.randn(N, H, H, C, generator=g).cuda()
    y = blk.forward(x)
    dy = torch.randn(N, H, H, C, generator=g).cuda()
    dx = blk.backward(dy)
    torch.cuda.synchronize()
    P = blk.master
    xt = x.permute(0, 3, 1, 2).contiguous().requires_grad_(True)
    w = P["wdw"].permute(2, 0, 1).reshape(C, 1, 3, 3).clone().requires_grad_(True)
    gm, bt = P["g"].clone().requires_grad_(True), P["b"].clone().requires_grad_(True)
    z = F.conv2d(xt, w, padding=1, groups=C)
    u = F.batch_norm(z, None, None, gm, bt, training=True, eps=1e-3)
    a = u * torch.sigmoid(u)
    p = a.mean((2, 3))
    r = p @ P["wr"].t() + P["br"]
    s = torch.sigmoid((r * torch.sigmoid(r)) @ P["we"].t() + P["be"])
    yt = a * s[:, :, None, None]
    yt.backward(dy.permute(0, 3, 1, 2))

    def rel(a_, b_):
        return ((a_ - b_).abs() / b_.abs().clamp_min(1)).max().item()

    assert rel(y.permute(0, 3, 1, 2), yt.detach()) < 1e-3
    assert rel(dx.permute(0, 3, 1, 2), xt.grad) < 1e-3
    assert rel(blk.grad["wdw"].permute(2, 0, 1).reshape(C, 1, 3, 3), w.grad) < 1e-2
    assert rel(blk.grad["g"], gm.grad) < 1e-2
    assert rel(blk.grad["b"], bt.grad) < 1e-2


def test_c3_bf16_vs_oracle():
    """the benchmarked C3 block in its benchmarked dtype (bf16,
    112x112, C=96, SE=4, stride 1) at N=16 images against the float64 oracle
    on the same bf16-rounded inputs, with the bf16 storage model applied where
    the GPU stores z and y (oracle.mbconv_fwd docstring): y, dx, the running
    statistics and every parameter gradient at the bf16 bar 2e-2 (the
    interp.compare_outputs metric, interp.py:1332-1352)."""
    rng = np.random.default_rng(96)
    N, C, HW, SE = 16, 96, 112, 4
    prm, x = _rand_case(rng, N, C, HW, HW, SE)
    x = O.round_bf16(x).astype(np.float64)
    rnd = lambda a: O.round_bf16(a).astype(np.float64)  # noqa: E731
    y_w, rm_w, rv_w, cache = O.mbconv_fwd(prm, x, 1, 1e-3, 0.99, rnd=rnd)
    dy = O.round_bf16(rng.standard_normal(y_w.shape)).astype(np.float64)
    gw = O.mbconv_bwd(prm, cache, dy)
    del cache
    blk = _block(C, SE, 1, (1, 1, 1, 1), torch.bfloat16, prm=prm)
    y, dx = _run(blk, x, dy, torch.bfloat16)
    errs = {"y": O.compare(y, y_w), "dx": O.compare(dx, gw["x"]),
            "rm": O.compare(blk.running_mean.cpu().numpy(), rm_w),
            "rv": O.compare(blk.running_var.cpu().numpy(), rv_w)}
    gr = blk.grads_numpy()
    for k in GRADS[1:]:
        errs[k] = O.compare(gr[k], gw[k])
    print("C3 bf16 N=16 vs oracle:", {k: f"{v:.2e}" for k, v in errs.items()})
    _check(errs, 2e-2)
