"""GPU parity of the HBM-bound row kernels against the numpy oracle.

Tolerances (north star): 1e-4 for f32, 2e-2 for bf16 (oracle fed the same
bf16-rounded inputs), with the interp.compare_outputs metric
max|a-b|/max(|b|,1) (interp.py:1332-1352)."""

import numpy as np
import pytest
import torch

from oracle import oracle as O
from golden_util import golden

pytestmark = pytest.mark.gpu

TOL = {torch.float32: 1e-4, torch.bfloat16: 2e-2}


def K():
    from paper_2110_10802_b200 import kernels

    return kernels


def dev(a, dtype):
    return torch.as_tensor(np.asarray(a), dtype=torch.float32).to("cuda").to(dtype).contiguous()


def host(t):
    return t.float().cpu().numpy().astype(np.float64)


def rounded(a, dtype):
    return O.round_bf16(a).astype(np.float64) if dtype == torch.bfloat16 else np.asarray(a, np.float64)


def assert_close(got, want, tol, what=""):
    err = O.compare(got, want)
    assert err <= tol, f"{what}: max rel err {err:.3e} > {tol:.1e}"


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("rows,cols", [(256, 768), (37, 64), (8, 1024), (1, 768), (300, 2048)])
def test_bdrln(dtype, rows, cols):
    k = K()
    rng = np.random.default_rng(rows * 7 + cols)
    h, r = rng.standard_normal((rows, cols)), rng.standard_normal((rows, cols))
    bias, g, be = 0.1 * rng.standard_normal(cols), 1 + 0.1 * rng.standard_normal(cols), 0.1 * rng.standard_normal(cols)
    p = 0.1
    keep = rng.random((rows, cols)) >= p
    h, r = rounded(h, dtype), rounded(r, dtype)
    mask = O.mask_values(keep, p, np.float64)
    want = O.bdrln_fwd(h, bias, mask, r, g, be, 1e-12)
    th, tr = dev(h, dtype), dev(r, dtype)
    tk = torch.as_tensor(keep.astype(np.uint8)).cuda()
    tb, tg, tbe = (dev(v, torch.float32) for v in (bias, g, be))
    y, s = torch.empty_like(th), torch.empty_like(th)
    mean = torch.empty(rows, device="cuda")
    rstd = torch.empty(rows, device="cuda")
    ks = 1.0 / (1.0 - p)
    k.bdrln_fwd(th, tb, tk, ks, tr, tg, tbe, 1e-12, y=y, s=s, mean=mean, rstd=rstd)
    torch.cuda.synchronize()
    tol = TOL[dtype]
    assert_close(host(y), want["y"], tol, "y")
    assert_close(host(s), want["s"], tol, "s")
    assert_close(host(mean), want["mean"], tol, "mean")
    dy = rounded(rng.standard_normal((rows, cols)), dtype)
    s_used = host(s)  # backward consumes the stash the GPU wrote
    wb = O.bdrln_bwd(dy, s_used, g, mask, 1e-12)
    ds, dh = torch.empty_like(th), torch.empty_like(th)
    dg, dbe, dbi = (torch.empty(cols, device="cuda") for _ in range(3))
    k.bdrln_bwd(dev(dy, dtype), s, tg, tk, ks, 1e-12, ds=ds, dh=dh, dgamma=dg, dbeta=dbe, dbias=dbi)
    torch.cuda.synchronize()
    assert_close(host(ds), wb["ds"], tol, "ds")
    assert_close(host(dh), wb["dh"], tol, "dh")
    assert_close(host(dg), wb["dgamma"], tol, "dgamma")
    assert_close(host(dbe), wb["dbeta"], tol, "dbeta")
    assert_close(host(dbi), wb["dbias"], tol, "dbias")


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("rows,cols", [(4096, 768), (37, 64), (300, 2048), (5, 96)])
def test_bdrln_packed_keep_identical(dtype, rows, cols):
    """Bit-packed keep flags (dfx_bdrln_{fwd,bwd}_kb) give bitwise the u8 results."""
    from paper_2110_10802_b200 import kernels as KK
    k = K()
    g = torch.Generator(device="cpu").manual_seed(rows + cols)
    h, r, dy = (torch.randn(rows, cols, generator=g).to(dtype).cuda() for _ in range(3))
    bias, gm, be = (torch.randn(cols, generator=g).cuda() for _ in range(3))
    keep = (torch.rand(rows, cols, generator=g) >= 0.1).to(torch.uint8).cuda()
    kb = KK.pack_keep_bits(keep)
    outs = []
    for kk in (keep, kb):
        y, s = torch.empty_like(h), torch.empty_like(h)
        k.bdrln_fwd(h, bias, kk, 1 / 0.9, r, gm, be, 1e-12, y=y, s=s)
        ds, dh = torch.empty_like(h), torch.empty_like(h)
        dg, dbe, dbi = (torch.empty(cols, device="cuda") for _ in range(3))
        k.bdrln_bwd(dy, s, gm, kk, 1 / 0.9, 1e-12, ds=ds, dh=dh, dgamma=dg, dbeta=dbe, dbias=dbi)
        outs.append((y, s, ds, dh, dg, dbe, dbi))
    torch.cuda.synchronize()
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def test_bdrln_golden_f32():
    """Straight against the reference's own outputs (tests/golden)."""
    k = K()
    g = golden("bdrln_f32")
    p = float(g["p"])
    keep = torch.as_tensor(g["keep"].astype(np.uint8)).cuda()
    f = lambda a: dev(a, torch.float32)  # noqa: E731
    s = torch.empty_like(f(g["h"]))
    y = k.bdrln_fwd(f(g["h"]), f(g["b"]), keep, 1 / (1 - p), f(g["r"]), f(g["g"]), f(g["be"]),
                    float(g["eps"]), s=s)
    ds, dh = torch.empty_like(y), torch.empty_like(y)
    H = y.shape[1]
    dgm, dbe, dbi = (torch.empty(H, device="cuda") for _ in range(3))
    k.bdrln_bwd(f(g["dy"]), s, f(g["g"]), keep, 1 / (1 - p), float(g["eps"]), ds=ds, dh=dh, dgamma=dgm,
                dbeta=dbe, dbias=dbi)
    torch.cuda.synchronize()
    for got, key in ((y, "y"), (dh, "dh"), (ds, "dr"), (dgm, "dg"), (dbe, "dbe"), (dbi, "db")):
        assert_close(host(got), g[key], 1e-4, key)


def test_bdrln_deterministic():
    k = K()
    rng = np.random.default_rng(5)
    rows, cols = 4096, 768
    x = dev(rng.standard_normal((rows, cols)), torch.bfloat16)
    g = dev(1 + 0.1 * rng.standard_normal(cols), torch.float32)
    outs = []
    for _ in range(2):
        ds, dh = torch.empty_like(x), torch.empty_like(x)
        dg = torch.empty(cols, device="cuda")
        k.bdrln_bwd(x, x, g, None, 1.0, 1e-12, ds=ds, dh=dh, dgamma=dg)
        outs.append(dg.clone())
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("B,NH,Q,Kc", [(2, 12, 128, 128), (1, 2, 5, 512), (2, 3, 16, 64), (1, 1, 3, 1024)])
def test_softmax(dtype, B, NH, Q, Kc):
    k = K()
    rng = np.random.default_rng(B * 100 + Kc)
    sc = rounded(3 * rng.standard_normal((B, NH, Q, Kc)), dtype)
    am = np.where(rng.random((B, 1, 1, Kc)) < 0.1, -10000.0, 0.0)
    p_ = 0.1
    keep = rng.random((B, NH, Q, Kc)) >= p_
    dm = O.mask_values(keep, p_, np.float64)
    pw, pdw = O.scaled_masked_softmax_fwd(sc, 8.0, am, dm)
    tsc = dev(sc, dtype)
    tk = torch.as_tensor(keep.astype(np.uint8)).cuda()
    tam = dev(am.reshape(B, Kc), torch.float32)
    p, pd = torch.empty_like(tsc), torch.empty_like(tsc)
    k.softmax_fwd(tsc, 1 / 8.0, tam, tk, 1 / (1 - p_), p, pd)
    torch.cuda.synchronize()
    tol = TOL[dtype]
    assert_close(host(p), pw, tol, "p")
    assert_close(host(pd), pdw, tol, "pd")
    dpd = rounded(rng.standard_normal((B, NH, Q, Kc)), dtype)
    want = O.scaled_masked_softmax_bwd(dpd, host(p), dm, 8.0)
    got = k.softmax_bwd(dev(dpd, dtype), p, tk, 1 / (1 - p_), 1 / 8.0)
    torch.cuda.synchronize()
    assert_close(host(got), want, tol, "dsc")


def test_softmax_golden_f32():
    k = K()
    g = golden("softmax_f32")
    B, NH, S, _ = g["sc"].shape
    pdrop = float(g["p"])
    keep = torch.as_tensor(g["keep"].astype(np.uint8)).cuda()
    tsc = dev(g["sc"], torch.float32)
    p, pd = torch.empty_like(tsc), torch.empty_like(tsc)
    k.softmax_fwd(tsc, 1 / float(g["divisor"]), dev(g["am"].reshape(B, S), torch.float32), keep,
                  1 / (1 - pdrop), p, pd)
    dsc = k.softmax_bwd(dev(g["dy"], torch.float32), p, keep, 1 / (1 - pdrop), 1 / float(g["divisor"]))
    torch.cuda.synchronize()
    assert_close(host(p), g["p_out"], 1e-4, "p")
    assert_close(host(pd), g["pd"], 1e-4, "pd")
    assert_close(host(dsc), g["dsc"], 1e-4, "dsc")


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_bias_gelu(dtype):
    k = K()
    rng = np.random.default_rng(3)
    f = rounded(2 * rng.standard_normal((96, 3072)), dtype)
    b = 0.1 * rng.standard_normal(3072)
    pre_w, y_w = O.bias_gelu_fwd(f, b)
    tf = dev(f, dtype)
    pre = torch.empty_like(tf)
    y = k.bias_gelu_fwd(tf, dev(b, torch.float32), pre=pre)
    dy = rounded(rng.standard_normal(f.shape), dtype)
    db = torch.empty(3072, device="cuda")
    dpre = k.bias_gelu_bwd(dev(dy, dtype), pre, dbias=db)
    torch.cuda.synchronize()
    dpre_w, db_w = O.bias_gelu_bwd(dy, host(pre))
    tol = TOL[dtype]
    assert_close(host(y), y_w, tol, "y")
    assert_close(host(pre), pre_w, tol, "pre")
    assert_close(host(dpre), dpre_w, tol, "dpre")
    assert_close(host(db), db_w, tol * 10 if dtype == torch.bfloat16 else tol, "dbias")


def test_colsum_strided():
    k = K()
    rng = np.random.default_rng(9)
    x = rng.standard_normal((777, 2304))
    t = dev(x, torch.float32)
    out = torch.zeros(768, device="cuda")
    k.colsum(t[:, 768:1536], out)
    torch.cuda.synchronize()
    assert_close(host(out), x[:, 768:1536].sum(0), 1e-4)


def test_errors_raise():
    """Host-side validation mirrors the reference's ShapeError behaviour."""
    from paper_2110_10802_b200.errors import ShapeError

    k = K()
    x = torch.zeros(4, 1001, device="cuda")  # odd width beyond the scalar-lane limit
    g = torch.ones(1001, device="cuda")
    with pytest.raises(ShapeError):
        k.bdrln_fwd(x, None, None, 1.0, None, g, g, 1e-5)
    with pytest.raises(ShapeError):  # f64 is not a B200 activation dtype
        k.bdrln_fwd(x.double(), None, None, 1.0, None, g, g, 1e-5)
    a = torch.zeros(64, 32, device="cuda")
    with pytest.raises(ShapeError):  # contracted dims differ
        k.gemm(a, torch.zeros(16, 48, device="cuda"), torch.zeros(64, 16, device="cuda"))


def test_odd_widths_scalar_lanes():
    """Widths that are not a multiple of the vector width take scalar lanes
    (the reference accepts any extent)."""
    k = K()
    rng = np.random.default_rng(1)
    for cols in (5, 7, 33, 500):
        x = rng.standard_normal((9, cols))
        g, b = 1 + 0.1 * rng.standard_normal(cols), 0.1 * rng.standard_normal(cols)
        y = k.bdrln_fwd(dev(x, torch.float32), None, None, 1.0, None, dev(g, torch.float32),
                        dev(b, torch.float32), 1e-5)
        torch.cuda.synchronize()
        assert_close(host(y), O.layernorm(x, g, b, 1e-5), 1e-4, f"cols={cols}")


@pytest.mark.parametrize("n,off", [(7_087_872, 0), (4096 * 3 + 4, 0), (1001, 0), (4096, 1)])
def test_sgd_update_vector_and_scalar_paths(n, off):
    """dfx_sgd_update: the 16-byte path (n % 4 == 0, aligned) and the scalar
    path (odd n / misaligned views) give w - lr*g as one fma, and the bf16
    shadow is its round-to-nearest copy."""
    from paper_2110_10802_b200 import kernels as KK
    g = torch.Generator(device="cpu").manual_seed(n)
    w0 = torch.randn(n + off, generator=g).cuda()
    gr = torch.randn(n + off, generator=g).cuda()
    w, gg = w0[off:], gr[off:]
    ref = torch.addcmul(w.double(), gg.double(), torch.full_like(gg.double(), -1e-3)).float()
    wb = torch.empty(n + off, dtype=torch.bfloat16, device="cuda")[off:]
    wk = w.clone() if off == 0 else w  # misaligned view stays a view
    KK.sgd_update(wk, gg, 1e-3, wb)
    torch.cuda.synchronize()
    assert torch.allclose(wk, ref, rtol=0, atol=1e-6 * max(1.0, ref.abs().max().item()))
    assert torch.equal(wb, wk.bfloat16())
