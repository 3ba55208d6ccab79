"""GPU parity of the fused attention kernels (csrc/attn.cu) against the oracle.

Forward: ctx = (softmax(QKᵀ/divisor + mask) ∘ dropout) V, the chain of
reference operators Einsum / Div / Add / Softmax / Mul / Einsum
(frontend.py:294, 175-188, 408-501); backward: their VJPs
(autodiff.py:1363-1415, 1465-1484).  The oracle runs in float64 on the same
bf16-rounded Q/K/V and the same explicit keep masks; tolerance 2e-2 (bf16) with
the interp.compare_outputs metric."""

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu

P_DROP = 0.1


def K():
    from paper_2110_10802_b200 import kernels

    return kernels


def _case(B, NH, S, seed, dropout=True, masked=True):
    rng = np.random.default_rng(seed)
    H = NH * 64
    qkv = O.round_bf16(rng.standard_normal((B * S, 3 * H))).astype(np.float64)
    am = np.where(rng.random((B, S)) < 0.1, -10000.0, 0.0) if masked else np.zeros((B, S))
    keep = rng.random((B, NH, S, S)) >= P_DROP if dropout else np.ones((B, NH, S, S), bool)
    dctx = O.round_bf16(rng.standard_normal((B * S, H))).astype(np.float64)
    return qkv, am, keep, dctx


def _heads(x, B, S, NH, which):
    H = NH * 64
    return x[:, which * H:(which + 1) * H].reshape(B, S, NH, 64)


def _oracle(qkv, am, keep, dctx, B, S, NH, p_drop=P_DROP):
    q, k, v = (_heads(qkv, B, S, NH, i) for i in range(3))
    scores = np.einsum("bsnd,btnd->bnst", q, k)
    dm = O.mask_values(keep, p_drop, np.float64)
    p, pd = O.scaled_masked_softmax_fwd(scores, 8.0, am.reshape(B, 1, 1, S), dm)
    ctx = np.einsum("bnst,btnd->bsnd", pd, v).reshape(B * S, NH * 64)
    do = dctx.reshape(B, S, NH, 64)
    dpd = np.einsum("bsnd,btnd->bnst", do, v)
    dv = np.einsum("bnst,bsnd->btnd", pd, do)
    ds = O.scaled_masked_softmax_bwd(dpd, p, dm, 8.0)
    dq = np.einsum("bnst,btnd->bsnd", ds, k)
    dk = np.einsum("bnst,bsnd->btnd", ds, q)
    lse2 = np.log2(np.exp(scores / 8.0 + am.reshape(B, 1, 1, S)).sum(-1))
    dqkv = np.concatenate([t.reshape(B * S, NH * 64) for t in (dq, dk, dv)], 1)
    return ctx, lse2, dqkv


def _run(qkv, am, keep, dctx, B, S, NH, dropout=True):
    k = K()
    H = NH * 64
    t_qkv = torch.as_tensor(qkv, dtype=torch.float32).bfloat16().cuda()
    t_am = torch.as_tensor(am, dtype=torch.float32).cuda()
    t_keep = torch.as_tensor(keep.astype(np.uint8)).cuda() if dropout else None
    ctx = torch.empty(B * S, H, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(B, NH, S, dtype=torch.float32, device="cuda")
    kr = torch.empty(B, NH, S, S // 32, dtype=torch.int32, device="cuda") if dropout else None
    kc = torch.empty_like(kr) if dropout else None
    ks = 1.0 / (1.0 - P_DROP) if dropout else 1.0
    k.attn_fwd(t_qkv, B, S, NH, t_am, t_keep, ks, 0.125, ctx, lse, kr, kc)
    t_do = torch.as_tensor(dctx, dtype=torch.float32).bfloat16().cuda()
    dqkv = torch.zeros(B * S, 3 * H, dtype=torch.bfloat16, device="cuda")
    k.attn_bwd(t_qkv, ctx, t_do, B, S, NH, t_am, lse, kr, kc, ks, 0.125, dqkv)
    torch.cuda.synchronize()
    f = lambda t: t.float().cpu().numpy().astype(np.float64)  # noqa: E731
    return f(ctx), f(lse), f(dqkv), kr, kc


# the persistent forward / key-strip kernels run min(strips, SMs) CTAs: the
# last four shapes give every CTA two or three strips (1, 2, 3 and 4 chunks per
# strip), so the cross-strip buffer parities and barrier phases are exercised
@pytest.mark.parametrize("B,NH,S", [(2, 2, 128), (1, 3, 256), (2, 2, 384), (2, 12, 512), (8, 12, 512),
                                    (24, 12, 128), (6, 16, 256), (4, 16, 384)])
def test_attention_vs_oracle(B, NH, S):
    qkv, am, keep, dctx = _case(B, NH, S, seed=S + NH)
    ctx, lse, dqkv, _, _ = _run(qkv, am, keep, dctx, B, S, NH)
    w_ctx, w_lse, w_dqkv = _oracle(qkv, am, keep, dctx, B, S, NH)
    assert O.compare(ctx, w_ctx) <= 2e-2, O.compare(ctx, w_ctx)
    assert np.abs(lse - w_lse).max() <= 1e-2 * max(1.0, np.abs(w_lse).max()), np.abs(lse - w_lse).max()
    H = NH * 64
    for i, nm in enumerate("qkv"):
        got, want = dqkv[:, i * H:(i + 1) * H], w_dqkv[:, i * H:(i + 1) * H]
        err = O.compare_scaled(got, want)
        assert err <= 2e-2, f"d{nm}: {err:.3e}"


@pytest.mark.parametrize("B,NH,S", [(2, 2, 128), (2, 12, 512), (1, 3, 384), (4, 16, 384)])
def test_qkv_bias_grad_from_strip_partials(B, NH, S):
    """dfx_attn_bwd_bias_grad (per-strip fp32 column sums left by the backward)
    against the oracle's column sums of dQ | dK | dV, and against a column sum
    of the bf16 dqkv the same call wrote."""
    from paper_2110_10802_b200 import kernels as KK
    qkv, am, keep, dctx = _case(B, NH, S, seed=3 * S + NH)
    H = NH * 64
    t_qkv = torch.as_tensor(qkv, dtype=torch.float32).bfloat16().cuda()
    t_am = torch.as_tensor(am, dtype=torch.float32).cuda()
    t_keep = torch.as_tensor(keep.astype(np.uint8)).cuda()
    ctx = torch.empty(B * S, H, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(B, NH, S, dtype=torch.float32, device="cuda")
    kr = torch.empty(B, NH, S, S // 32, dtype=torch.int32, device="cuda")
    kc = torch.empty_like(kr)
    ks = 1.0 / (1.0 - P_DROP)
    KK.attn_fwd(t_qkv, B, S, NH, t_am, t_keep, ks, 0.125, ctx, lse, kr, kc)
    t_do = torch.as_tensor(dctx, dtype=torch.float32).bfloat16().cuda()
    dqkv = torch.zeros(B * S, 3 * H, dtype=torch.bfloat16, device="cuda")
    ws = KK.attn_bwd_workspace(B, S, NH)
    KK.attn_bwd(t_qkv, ctx, t_do, B, S, NH, t_am, lse, kr, kc, ks, 0.125, dqkv, ws=ws)
    db = torch.full((3 * H,), 7.0, device="cuda")
    KK.attn_bwd_bias_grad(B, S, NH, ws, db)
    db2 = torch.ones(3 * H, device="cuda")
    KK.attn_bwd_bias_grad(B, S, NH, ws, db2, accumulate=True)
    torch.cuda.synchronize()
    got = db.cpu().numpy().astype(np.float64)
    _, _, w_dqkv = _oracle(qkv, am, keep, dctx, B, S, NH)
    want = w_dqkv.sum(0)
    assert O.compare_scaled(got, want) <= 2e-2, O.compare_scaled(got, want)
    from_bf16 = dqkv.float().sum(0).cpu().numpy()
    assert np.abs(got - from_bf16).max() <= 1e-2 * max(1.0, np.abs(from_bf16).max())
    assert np.allclose(db2.cpu().numpy(), got + 1.0, rtol=1e-6, atol=1e-5)


def test_attention_no_dropout_no_mask():
    B, NH, S = 1, 2, 256
    qkv, am, keep, dctx = _case(B, NH, S, seed=7, dropout=False, masked=False)
    ctx, _, dqkv, _, _ = _run(qkv, am, keep, dctx, B, S, NH, dropout=False)
    w_ctx, _, w_dqkv = _oracle(qkv, am, keep, dctx, B, S, NH, p_drop=0.0)
    assert O.compare(ctx, w_ctx) <= 2e-2
    assert O.compare_scaled(dqkv, w_dqkv) <= 2e-2


def test_attention_online_rescale():
    """Key chunks whose scores exceed the first chunk's max by far more than
    2^8 (a large additive mask on the first 128 keys of some sequences, and
    one sequence where only some rows see it): the forward's lazily rescaled
    reference max must move, warp-uniformly, for exactly those rows."""
    B, NH, S = 2, 3, 512
    qkv, am, keep, dctx = _case(B, NH, S, seed=21)
    am[0, :128] = -30.0  # every row of sequence 0: chunk 0 is ~2^43 below the rest
    qkv = qkv.copy()
    H = NH * 64
    # sequence 1: large keys in chunk 2 for head 0, so rows with large q see a jump there
    qkv[S + 256:S + 384, H:H + 64] *= 6.0
    qkv = O.round_bf16(qkv).astype(np.float64)
    ctx, lse, dqkv, _, _ = _run(qkv, am, keep, dctx, B, S, NH)
    w_ctx, w_lse, w_dqkv = _oracle(qkv, am, keep, dctx, B, S, NH)
    assert O.compare(ctx, w_ctx) <= 2e-2, O.compare(ctx, w_ctx)
    assert np.abs(lse - w_lse).max() <= 1e-2 * max(1.0, np.abs(w_lse).max())
    assert O.compare_scaled(dqkv, w_dqkv) <= 2e-2


def test_attention_online_rescale_every_strip():
    """The rescale in every strip of a 384-strip grid (each persistent CTA walks
    two or three strips, so the rescale meets every buffer parity): the first
    128 keys of every sequence sit ~2^43 below the rest."""
    B, NH, S = 8, 12, 512
    qkv, am, keep, dctx = _case(B, NH, S, seed=23)
    am[:, :128] = -30.0
    ctx, lse, dqkv, _, _ = _run(qkv, am, keep, dctx, B, S, NH)
    w_ctx, w_lse, w_dqkv = _oracle(qkv, am, keep, dctx, B, S, NH)
    assert O.compare(ctx, w_ctx) <= 2e-2, O.compare(ctx, w_ctx)
    assert np.abs(lse - w_lse).max() <= 1e-2 * max(1.0, np.abs(w_lse).max())
    assert O.compare_scaled(dqkv, w_dqkv) <= 2e-2


def test_packed_keep_bits():
    B, NH, S = 1, 2, 256
    qkv, am, keep, dctx = _case(B, NH, S, seed=11)
    _, _, _, kr, kc = _run(qkv, am, keep, dctx, B, S, NH)
    w = (1 << np.arange(32, dtype=np.uint64))
    rowbits = (keep.reshape(B, NH, S, S // 32, 32).astype(np.uint64) * w).sum(-1)
    colbits = (np.swapaxes(keep, 2, 3).reshape(B, NH, S, S // 32, 32).astype(np.uint64) * w).sum(-1)
    assert np.array_equal(kr.cpu().numpy().view(np.uint32).astype(np.uint64), rowbits)
    assert np.array_equal(kc.cpu().numpy().view(np.uint32).astype(np.uint64), colbits)


def test_attention_deterministic():
    B, NH, S = 2, 4, 512
    qkv, am, keep, dctx = _case(B, NH, S, seed=3)
    a = _run(qkv, am, keep, dctx, B, S, NH)
    b = _run(qkv, am, keep, dctx, B, S, NH)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[2], b[2])


def test_attention_rejects_bad_shapes():
    from paper_2110_10802_b200.errors import UnsupportedOp

    k = K()
    qkv = torch.zeros(2 * 100, 3 * 128, dtype=torch.bfloat16, device="cuda")
    ctx = torch.zeros(200, 128, dtype=torch.bfloat16, device="cuda")
    lse = torch.zeros(2, 2, 100, device="cuda")
    with pytest.raises(UnsupportedOp):
        k.attn_fwd(qkv, 2, 100, 2, None, None, 1.0, 0.125, ctx, lse)


def test_layer_fused_matches_unfused():
    """The fused and the unfused attention paths of the encoder layer agree."""
    from paper_2110_10802_b200.bert import BertEncoderLayer, BertLayerConfig

    B, S, NH, H = 2, 256, 12, 768
    rng = np.random.default_rng(5)
    x = torch.as_tensor(rng.standard_normal((B * S, H)), dtype=torch.float32).bfloat16().cuda()
    dout = torch.as_tensor(rng.standard_normal((B * S, H)), dtype=torch.float32).bfloat16().cuda()
    am = torch.as_tensor(np.where(rng.random((B, S)) < 0.1, -10000.0, 0.0), dtype=torch.float32).cuda()
    keeps = [torch.as_tensor((rng.random(s) >= 0.1).astype(np.uint8)).cuda()
             for s in ((B, NH, S, S), (B * S, H), (B * S, H))]
    outs = []
    for fused in (True, False):
        layer = BertEncoderLayer(BertLayerConfig(fused_attention=fused), seed=3)
        out = layer.forward(x, am, *keeps).float().cpu().numpy()
        dx = layer.backward(dout).float().cpu().numpy()
        outs.append((out, dx, layer.grads_numpy()))
    (o1, d1, g1), (o2, d2, g2) = outs
    assert O.compare(o1, o2) <= 2e-2
    assert O.compare_scaled(d1, d2) <= 2e-2
    for name in ("wq", "wk", "wv", "bq", "wo", "w1"):
        assert O.compare_scaled(g1[name], g2[name]) <= 2e-2, name


def test_packed_keep_input_matches_u8():
    """The attention dropout mask supplied bit-packed (kernels.pack_keep_bits,
    the bench / e2e input form) gives bitwise the same layer outputs and
    gradients as the u8 keep flags."""
    import torch

    from paper_2110_10802_b200 import kernels as K
    from paper_2110_10802_b200.bert import BertEncoderLayer, BertLayerConfig

    B, S, H, NH = 2, 256, 768, 12
    g = torch.Generator(device="cpu").manual_seed(4)
    x = torch.randn(B * S, H, generator=g).bfloat16().cuda()
    dout = torch.randn(B * S, H, generator=g).bfloat16().cuda()
    am = torch.where(torch.rand(B, S, generator=g) < 0.1, -10000.0, 0.0).cuda()
    ka = (torch.rand(B, NH, S, S, generator=g) >= 0.1).to(torch.uint8).cuda()
    k1 = (torch.rand(B * S, H, generator=g) >= 0.1).to(torch.uint8).cuda()
    k2 = (torch.rand(B * S, H, generator=g) >= 0.1).to(torch.uint8).cuda()
    outs = []
    for keep in (ka, K.pack_keep_bits(ka)):
        layer = BertEncoderLayer(BertLayerConfig(dtype=torch.bfloat16), seed=9)
        out = layer.forward(x, am, keep, k1, k2).clone()
        dx = layer.backward(dout).clone()
        torch.cuda.synchronize()
        outs.append((out, dx, layer.grad.flat.clone()))
    for a, b in zip(*outs):
        assert torch.equal(a, b)
