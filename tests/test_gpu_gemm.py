"""GPU parity of the contraction paths (tcgen05 bf16 and CUDA-core f32).

Reference: Gemm/Einsum (frontend.py:369-481) evaluated by the oracle
(oracle.gemm, f64).  bf16 operands are exactly representable in f64, so the
only error is fp32 accumulation + output rounding."""

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def K():
    from paper_2110_10802_b200 import kernels

    return kernels


def _rand(shape, dtype, seed, scale=1.0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return (scale * torch.randn(shape, generator=g)).to(dtype).cuda()


def _ref(a, b):
    """f64 A @ B^T over the trailing two dims."""
    A = a.double().cpu().numpy()
    B = b.double().cpu().numpy()
    return np.einsum("...mk,...nk->...mn", A, B)


def _check(got, want, tol):
    err = O.compare(got.double().cpu().numpy(), want)
    assert err <= tol, f"max rel err {err:.3e} > {tol}"


LAYOUTS = [("k", "k"), ("k", "n"), ("m", "n"), ("m", "k")]


def _operands(m, n, k, la, lb, dtype, seed):
    a = _rand((m, k), dtype, seed) if la == "k" else _rand((k, m), dtype, seed).t()
    b = _rand((n, k), dtype, seed + 1) if lb == "k" else _rand((k, n), dtype, seed + 1).t()
    return a, b


@pytest.mark.parametrize("la,lb", LAYOUTS)
@pytest.mark.parametrize("m,n,k", [(256, 768, 768), (128, 64, 512), (512, 2304, 128), (384, 96, 64),
                                   (256, 320, 192)])
def test_tc_gemm_layouts(la, lb, m, n, k):
    kk = K()
    a, b = _operands(m, n, k, la, lb, torch.bfloat16, m + n + k)
    for out_dtype in (torch.bfloat16, torch.float32):
        d = torch.empty(m, n, dtype=out_dtype, device="cuda")
        assert kk.gemm_uses_tensor_cores(a, b, d)
        kk.gemm(a, b, d)
        torch.cuda.synchronize()
        _check(d, _ref(a, b), 1e-2 if out_dtype == torch.bfloat16 else 1e-4)


@pytest.mark.parametrize("epi", ["bias", "bias_gelu", "gelu_bwd", "add"])
@pytest.mark.parametrize("simt", [False, True])
def test_gemm_epilogues(epi, simt):
    kk = K()
    from paper_2110_10802_b200 import _lib

    m, n, k = 256, 512, 256
    a, b = _operands(m, n, k, "k", "k", torch.bfloat16, 7)
    bias = _rand((n,), torch.float32, 8, 0.1)
    aux = _rand((m, n), torch.bfloat16, 9)
    d = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
    pre = torch.empty_like(d)
    acc = 0.5 * _ref(a, b)
    bn = bias.double().cpu().numpy()
    ax = aux.double().cpu().numpy()
    if epi == "bias":
        kk.gemm(a, b, d, _lib.EPI_BIAS, alpha=0.5, bias=bias, force_simt=simt)
        want = acc + bn
    elif epi == "bias_gelu":
        kk.gemm(a, b, d, _lib.EPI_BIAS_GELU, alpha=0.5, bias=bias, aux_out=pre, force_simt=simt)
        want = O.gelu(acc + bn)
        torch.cuda.synchronize()
        _check(pre, acc + bn, 1e-2)
    elif epi == "gelu_bwd":
        kk.gemm(a, b, d, _lib.EPI_GELU_BWD, alpha=0.5, aux=aux, force_simt=simt)
        want = acc * O.gelu_grad(ax)
    else:
        kk.gemm(a, b, d, _lib.EPI_ADD, alpha=0.5, beta=2.0, aux=aux, force_simt=simt)
        want = acc + 2.0 * ax
    torch.cuda.synchronize()
    _check(d, want, 1e-2)


def test_tc_batched_attention_views():
    """The strided [B, NH, S, dh] views of a fused QKV buffer (bert.py)."""
    kk = K()
    B, NH, S, dh = 2, 4, 256, 64
    H = NH * dh
    qkv = _rand((B * S, 3 * H), torch.bfloat16, 3)
    view = lambda i: qkv.as_strided((B, NH, S, dh), (S * 3 * H, dh, 3 * H, 1), i * H)  # noqa: E731
    q, k_, v = view(0), view(1), view(2)
    sc = torch.empty(B, NH, S, S, dtype=torch.bfloat16, device="cuda")
    assert kk.gemm_uses_tensor_cores(q, k_, sc)
    kk.gemm(q, k_, sc)
    ctx = torch.empty(B * S, H, dtype=torch.bfloat16, device="cuda")
    cv = ctx.as_strided((B, NH, S, dh), (S * H, dh, H, 1), 0)
    assert kk.gemm_uses_tensor_cores(sc, v.transpose(-1, -2), cv)
    kk.gemm(sc, v.transpose(-1, -2), cv)
    dv = torch.empty_like(cv)
    kk.gemm(sc.transpose(-1, -2), cv.transpose(-1, -2), dv)
    torch.cuda.synchronize()
    _check(sc, _ref(q, k_), 1e-2)
    _check(cv, _ref(sc, v.transpose(-1, -2)), 1e-2)
    _check(dv, _ref(sc.transpose(-1, -2), cv.transpose(-1, -2)), 1e-2)


@pytest.mark.parametrize("m,n,k", [(7, 5, 3), (130, 70, 33), (256, 768, 768)])
def test_simt_f32(m, n, k):
    kk = K()
    a, b = _operands(m, n, k, "k", "n", torch.float32, 11)
    d = torch.empty(m, n, dtype=torch.float32, device="cuda")
    assert not kk.gemm_uses_tensor_cores(a, b, d)
    kk.gemm(a, b, d)
    torch.cuda.synchronize()
    _check(d, _ref(a, b), 1e-4)


def test_tc_large_wgrad_fp32_out():
    """wgrad shape of FFN1 at the C2 config: M-major A, N-major B, f32 out."""
    kk = K()
    T, F, H = 4096, 3072, 768
    dpre = _rand((T, F), torch.bfloat16, 21)
    ln1 = _rand((T, H), torch.bfloat16, 22)
    dw = torch.empty(F, H, dtype=torch.float32, device="cuda")
    assert kk.gemm_uses_tensor_cores(dpre.t(), ln1.t(), dw)
    kk.gemm(dpre.t(), ln1.t(), dw)
    torch.cuda.synchronize()
    want = (dpre.float().t() @ ln1.float()).double().cpu().numpy()
    _check(dw, want, 1e-3)


@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_tc_split_k(out_dtype):
    """Few-tile GEMMs (the 768x768 out-proj weight gradient) split K into f32
    partials reduced in fixed order."""
    kk = K()
    T, H = 4096, 768
    a = _rand((T, H), torch.bfloat16, 31)
    b = _rand((T, H), torch.bfloat16, 32)
    d = torch.empty(H, H, dtype=out_dtype, device="cuda")
    from paper_2110_10802_b200 import _lib

    g = kk.gemm_args(a.t(), b.t(), d)
    assert _lib.load().dfx_gemm_workspace(g) > 0  # the split-K plan is taken
    kk.gemm(a.t(), b.t(), d)
    d2 = torch.empty_like(d)
    kk.gemm(a.t(), b.t(), d2)
    torch.cuda.synchronize()
    assert torch.equal(d, d2)  # deterministic
    want = (a.float().t() @ b.float()).double().cpu().numpy()
    _check(d, want, 1e-2 if out_dtype == torch.bfloat16 else 1e-3)


@pytest.mark.parametrize("n", [8, 40, 200])
def test_tc_ragged_n(n):
    """N not a multiple of the tile: TMA loads zero-fill, TMA stores clip."""
    kk = K()
    a, b = _operands(256, n, 128, "k", "k", torch.bfloat16, n)
    bias = _rand((n,), torch.float32, 5, 0.1)
    d = torch.full((256, n), 7.0, dtype=torch.bfloat16, device="cuda")
    from paper_2110_10802_b200 import _lib

    assert kk.gemm_uses_tensor_cores(a, b, d)
    kk.gemm(a, b, d, _lib.EPI_BIAS, bias=bias)
    torch.cuda.synchronize()
    _check(d, _ref(a, b) + bias.double().cpu().numpy(), 1e-2)


@pytest.mark.parametrize("m,n,k,la,lb", [(4704, 40, 24, "k", "k"), (300, 96, 16, "k", "k"), (1000, 144, 24, "m", "k"),
                                         (24, 40, 4704, "m", "m"), (130, 1152, 192, "k", "k")])
def test_tc_ragged_m_k(m, n, k, la, lb):
    """M and K not multiples of the 128 x 64 tile (the EfficientNet-B0 1x1
    convolutions: K = 16/24/40 channels, M = N*H*W pixels, wgrad K = pixels)."""
    kk = K()
    a, b = _operands(m, n, k, la, lb, torch.bfloat16, m + n + k)
    d = torch.full((m, n), 7.0, dtype=torch.bfloat16, device="cuda")
    assert kk.gemm_uses_tensor_cores(a, b, d)
    kk.gemm(a, b, d)
    torch.cuda.synchronize()
    _check(d, _ref(a, b), 1e-2)


@pytest.mark.parametrize("force", ["2,192", "1,192"])
@pytest.mark.parametrize("la,lb,epi", [("k", "k", "none"), ("k", "n", "none"), ("m", "k", "bias"), ("k", "k", "gelu")])
def test_tc_192_tiles(force, la, lb, epi, monkeypatch):
    """The 192-column tiles (768-wide BERT outputs) on every epilogue path with
    K- and MN-major operands, forced through DFX_GEMM_FORCE (read per call)."""
    from paper_2110_10802_b200 import _lib

    monkeypatch.setenv("DFX_GEMM_FORCE", force)
    kk = K()
    a, b = _operands(512, 768, 320, la, lb, torch.bfloat16, 11)
    d = torch.empty(512, 768, dtype=torch.bfloat16, device="cuda")
    bias = _rand((768,), torch.float32, 3, 0.1)
    e = {"none": _lib.EPI_NONE, "bias": _lib.EPI_BIAS, "gelu": _lib.EPI_BIAS_GELU}[epi]
    kk.gemm(a, b, d, e, bias=bias if e != _lib.EPI_NONE else None)
    torch.cuda.synchronize()
    want = _ref(a, b)
    if e != _lib.EPI_NONE:
        want = want + bias.double().cpu().numpy()
    if e == _lib.EPI_BIAS_GELU:
        want = 0.5 * want * (1 + np.tanh(0.7978845608028654 * (want + 0.044715 * want ** 3)))
    _check(d, want, 2e-2)
