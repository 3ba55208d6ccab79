"""CPU oracle for the fused training hot path — TEST INFRASTRUCTURE ONLY.

This module is a plain-numpy (float64) restatement of the reference ``dfir``
semantics for every function on the north-star path.  It is
*the checker*, never the product: only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.
The product path (``paper_2110_10802_b200``) never imports this file and has
no CPU fallback.

Parity pin: ``tests/test_oracle_golden.py`` checks every function here against
golden vectors produced by the *real* reference (``oracle/make_golden.py``
imports ``/root/reference/pkg/src/dfir`` and runs ``interp.execute`` +
``autodiff.differentiate_graph``); fixtures live in ``tests/golden/``.

Semantics followed (reference file:line, under /root/reference/pkg/src/dfir):

* every operator evaluates in float64 and casts back to the input dtype at the
  op boundary (frontend.py:146-150, 216-218, 240-242) — here everything stays
  float64 and callers cast once at the end;
* LayerNormalization: biased variance over axes [axis, rank)
  (frontend.py:519-529), VJP recomputes mu/var/xhat from the stashed input
  (autodiff.py:1490-1545);
* Softmax: max-subtracted exp / sum (frontend.py:493-501), VJP
  ``(dy - sum(dy*y)) * y`` from the stashed output (autodiff.py:1465-1484);
* Div by the folded ``divisor`` attribute (frontend.py:294, 1034-1040), Add
  with ONNX broadcasting (frontend.py:175-188, 291), Mul by an explicit
  dropout-mask tensor (frontend.py:293; there is no Dropout op);
* tanh-GELU assembled from Pow/Mul/Add/Tanh (frontend.py:223-295); its
  derivative is the symexpr derivative of the same chain (symexpr.py:672-738);
* Gemm ``alpha*op(A)@op(B) + beta*C`` (frontend.py:369-405) with the Einsum
  VJPs (autodiff.py:1363-1459);
* depthwise Conv (group = C, weight (C,1,kh,kw), symmetric/asymmetric pads,
  strides) via padded taps (frontend.py:645-666); its backward is the
  transposed scatter that the lowered loop nest differentiates to
  (lowering.py:930-1004, autodiff.py:1623-1629);
* BatchNormalization training mode: batch statistics over all axes but 1,
  biased variance, running stats ``run*m + batch*(1-m)`` (frontend.py:558-591);
  VJP ``scale*rstd*(dy - mean(dy) - xhat*mean(dy*xhat))`` (autodiff.py:1557-1617);
* Sigmoid ``1/(1+exp(-x))`` (frontend.py:229), GlobalAveragePool = mean over
  spatial axes (frontend.py:681-706).
"""

from __future__ import annotations

import numpy as np

GELU_C0 = 0.044715
GELU_C1 = 0.7978845608028654

f64 = np.float64


def _a(x):
    return np.asarray(x, dtype=f64)


# ---------------------------------------------------------------------------
# dtype helpers


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round to the nearest bfloat16 (ties to even), returned as float32.

    The reference has no bf16 (ir.py:49-56); SURVEY.md §8c defines the bf16
    oracle as the f64 oracle run on bf16-rounded inputs."""
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    u = a.view(np.uint32).astype(np.uint64)
    rounded = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    out = rounded.astype(np.uint32).view(np.float32)
    return np.where(np.isnan(a), a, out)


def mask_values(keep: np.ndarray, p: float, dtype=np.float32) -> np.ndarray:
    """Float dropout mask as fed to the reference ``Mul``: keep/(1-p)."""
    return (keep.astype(f64) * (1.0 / (1.0 - p))).astype(dtype)


def compare(got, want) -> float:
    """``interp.compare_outputs`` metric: max|a-b|/max(|b|,1)
    (interp.py:1332-1352)."""
    a, b = _a(got), _a(want)
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch {a.shape} vs {b.shape}")
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1.0)))


def compare_scaled(got, want) -> float:
    """max|a-b| / max(max|b|, 1): the compare metric normalised by the
    tensor's scale instead of per element.  Used for bf16 *reduction* outputs
    (parameter gradients = sums over T rows), whose near-zero elements are
    dominated by bf16 rounding-boundary flips: perturbing the oracle's own
    bf16 storage model by 1e-6 relative moves them by several percent
    element-wise but by <1e-2 on this metric (tests/test_oracle_golden.py::
    test_bf16_flip_sensitivity)."""
    a, b = _a(got), _a(want)
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch {a.shape} vs {b.shape}")
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))), 1.0))


# ---------------------------------------------------------------------------
# a1-a3: bias + dropout + residual + LayerNorm


def layernorm(x, gamma, beta=None, eps=1e-5, axis=-1):
    """frontend.py:519-529."""
    x = _a(x)
    axis = axis % x.ndim
    axes = tuple(range(axis, x.ndim))
    mu = x.mean(axis=axes, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=axes, keepdims=True)
    y = (x - mu) / np.sqrt(var + eps) * _a(gamma)
    if beta is not None:
        y = y + _a(beta)
    return y


def layernorm_bwd(dy, x, gamma, eps=1e-5, axis=-1):
    """autodiff.py:1490-1545 (recompute mu/var/xhat from the stashed x)."""
    dy, x, gamma = _a(dy), _a(x), _a(gamma)
    axis = axis % x.ndim
    axes = tuple(range(axis, x.ndim))
    lead = tuple(range(axis))
    mu = x.mean(axis=axes, keepdims=True)
    xc = x - mu
    var = (xc * xc).mean(axis=axes, keepdims=True)
    rstd = 1.0 / np.sqrt(var + eps)
    xhat = xc * rstd
    dyg = dy * gamma
    m1 = dyg.mean(axis=axes, keepdims=True)
    m2 = (dyg * xhat).mean(axis=axes, keepdims=True)
    dx = rstd * (dyg - m1 - xhat * m2)
    dgamma = (dy * xhat).sum(axis=lead) if lead else dy * xhat
    dbeta = dy.sum(axis=lead) if lead else dy
    return dx, dgamma, dbeta


def bdrln_fwd(h, bias, mask, residual, gamma, beta, eps):
    """s = (h + b) * mask + r ; y = LN(s).  Add/Mul/Add/LayerNormalization
    (frontend.py:291, 293, 519-529).  ``mask`` holds keep/(1-p) values."""
    s = (_a(h) + _a(bias)) * _a(mask) + _a(residual)
    mu = s.mean(axis=-1, keepdims=True)
    var = ((s - mu) ** 2).mean(axis=-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + eps)
    y = (s - mu) * rstd * _a(gamma) + _a(beta)
    return {"y": y, "s": s, "mean": mu[..., 0], "rstd": rstd[..., 0]}


def bdrln_bwd(dy, s, gamma, mask, eps):
    """VJP of bdrln_fwd: LN VJP (autodiff.py:1490-1545) then the Mul/Add
    VJPs.  Returns ds (= grad of residual), dh, dbias, dgamma, dbeta."""
    ds, dgamma, dbeta = layernorm_bwd(dy, s, gamma, eps)
    dh = ds * _a(mask)
    return {"ds": ds, "dh": dh, "dbias": dh.reshape(-1, dh.shape[-1]).sum(0),
            "dgamma": dgamma.reshape(-1, dgamma.shape[-1]).sum(0) if dgamma.ndim > 1 else dgamma,
            "dbeta": dbeta.reshape(-1, dbeta.shape[-1]).sum(0) if dbeta.ndim > 1 else dbeta}


# ---------------------------------------------------------------------------
# a4-a6: scaled + masked softmax + dropout


def softmax(x, axis=-1):
    """frontend.py:493-501."""
    x = _a(x)
    z = x - x.max(axis=axis, keepdims=True)
    e = np.exp(z)
    return e / e.sum(axis=axis, keepdims=True)


def softmax_bwd(dy, y, axis=-1):
    """autodiff.py:1465-1484."""
    dy, y = _a(dy), _a(y)
    return (dy - (dy * y).sum(axis=axis, keepdims=True)) * y


def scaled_masked_softmax_fwd(scores, divisor, add_mask, drop_mask):
    """P = softmax(scores/divisor + add_mask); Pd = P * drop_mask."""
    p = softmax(_a(scores) / divisor + _a(add_mask))
    return p, p * _a(drop_mask)


def scaled_masked_softmax_bwd(dpd, p, drop_mask, divisor):
    return softmax_bwd(_a(dpd) * _a(drop_mask), p) / divisor


# ---------------------------------------------------------------------------
# a7: bias + tanh-GELU


def gelu(x):
    x = _a(x)
    return 0.5 * x * (1.0 + np.tanh(GELU_C1 * (x + GELU_C0 * x ** 3)))


def gelu_grad(x):
    """d/dx of the Pow/Mul/Add/Tanh chain (symexpr.py:672-738)."""
    x = _a(x)
    t = np.tanh(GELU_C1 * (x + GELU_C0 * x ** 3))
    return 0.5 * (1.0 + t) + 0.5 * x * (1.0 - t * t) * GELU_C1 * (1.0 + 3.0 * GELU_C0 * x * x)


def bias_gelu_fwd(f, b):
    pre = _a(f) + _a(b)
    return pre, gelu(pre)


def bias_gelu_bwd(dy, pre):
    dpre = _a(dy) * gelu_grad(pre)
    return dpre, dpre.reshape(-1, dpre.shape[-1]).sum(0)


# ---------------------------------------------------------------------------
# a8: contractions


def gemm(a, b, c=None, alpha=1.0, beta=1.0, trans_a=False, trans_b=False):
    """frontend.py:384-394."""
    a, b = _a(a), _a(b)
    if trans_a:
        a = a.T
    if trans_b:
        b = b.T
    y = alpha * (a @ b)
    if c is not None:
        y = y + beta * _a(c)
    return y


# ---------------------------------------------------------------------------
# BERT encoder layer (SURVEY.md:500-511) built from the functions above.

BERT_WEIGHTS = ("wq", "wk", "wv", "wo", "w1", "w2", "bq", "bk", "bv", "bo", "b1", "b2",
                "g1", "be1", "g2", "be2")


def _ident(a):
    return a


def bert_layer_fwd(prm, x, am, dm, m1, m2, B, S, NH, eps=1e-12, rnd=None):
    """Forward of one post-LN encoder layer with explicit dropout masks.

    prm: dict of weights (Linear layout [out, in]); x [T,H]; am [B,1,1,S]
    additive mask; dm [B,NH,S,S], m1/m2 [T,H] dropout mask values.

    ``rnd`` (default: identity) is the storage model: it is applied to every
    intermediate the B200 path materialises in HBM, at the point it is
    stored (``round_bf16`` emulates the bf16 pipeline; the arithmetic itself
    stays float64).  With the identity this is exactly the reference chain."""
    R = rnd or _ident
    x = _a(x)
    T, H = x.shape
    dh = H // NH
    P = {k: _a(v) for k, v in prm.items()}

    def heads(t):
        return t.reshape(B, S, NH, dh)

    q = heads(R(gemm(x, P["wq"], P["bq"], trans_b=True)))
    k = heads(R(gemm(x, P["wk"], P["bk"], trans_b=True)))
    v = heads(R(gemm(x, P["wv"], P["bv"], trans_b=True)))
    sc = R(np.einsum("bsnd,btnd->bnst", q, k))
    p_exact, pd = scaled_masked_softmax_fwd(sc, float(np.sqrt(dh)), am, dm)
    p, pd = R(p_exact), R(pd)
    ctx = R(np.einsum("bnst,btnd->bsnd", pd, v).reshape(T, H))
    a1 = R(gemm(ctx, P["wo"], trans_b=True))
    r1 = bdrln_fwd(a1, P["bo"], m1, x, P["g1"], P["be1"], eps)
    ln1 = R(r1["y"])
    pre_exact, g = bias_gelu_fwd(gemm(ln1, P["w1"], trans_b=True), P["b1"])
    pre, g = R(pre_exact), R(g)
    a2 = R(gemm(g, P["w2"], trans_b=True))
    r2 = bdrln_fwd(a2, P["b2"], m2, ln1, P["g2"], P["be2"], eps)
    cache = dict(x=x, q=q, k=k, v=v, p=p, pd=pd, ctx=ctx, s1=R(r1["s"]), ln1=ln1, pre=pre, g=g,
                 s2=R(r2["s"]), dm=_a(dm), m1=_a(m1), m2=_a(m2), B=B, S=S, NH=NH, eps=eps, rnd=R)
    return R(r2["y"]), cache


def bert_layer_bwd(prm, cache, dout):
    """Reverse pass of bert_layer_fwd; returns grads keyed like prm plus 'x'.
    Stored gradient activations go through the same storage model."""
    P = {k: _a(v) for k, v in prm.items()}
    c = cache
    R = c.get("rnd") or _ident
    B, S, NH, eps = c["B"], c["S"], c["NH"], c["eps"]
    T, H = c["x"].shape
    dh = H // NH
    gr = {}
    r2 = bdrln_bwd(dout, c["s2"], P["g2"], c["m2"], eps)
    gr["g2"], gr["be2"], gr["b2"] = r2["dgamma"], r2["dbeta"], r2["dbias"]
    ds2, da2 = R(r2["ds"]), R(r2["dh"])
    gr["w2"] = da2.T @ c["g"]
    dpre, _ = bias_gelu_bwd(da2 @ P["w2"], c["pre"])
    dpre = R(dpre)
    gr["b1"] = dpre.sum(0)
    gr["w1"] = dpre.T @ c["ln1"]
    dln1 = R(dpre @ P["w1"] + ds2)
    r1 = bdrln_bwd(dln1, c["s1"], P["g1"], c["m1"], eps)
    gr["g1"], gr["be1"], gr["bo"] = r1["dgamma"], r1["dbeta"], r1["dbias"]
    ds1, da1 = R(r1["ds"]), R(r1["dh"])
    gr["wo"] = da1.T @ c["ctx"]
    dctx = R(da1 @ P["wo"]).reshape(B, S, NH, dh)
    dpd = R(np.einsum("bsnd,btnd->bnst", dctx, c["v"]))
    dv = R(np.einsum("bnst,bsnd->btnd", c["pd"], dctx))
    dsc = R(scaled_masked_softmax_bwd(dpd, c["p"], c["dm"], float(np.sqrt(dh))))
    dq = R(np.einsum("bnst,btnd->bsnd", dsc, c["k"]))
    dk = R(np.einsum("bnst,bsnd->btnd", dsc, c["q"]))
    dx = ds1.copy()
    for t, d in (("q", dq), ("k", dk), ("v", dv)):
        d2 = d.reshape(T, H)
        gr["w" + t] = d2.T @ c["x"]
        gr["b" + t] = d2.sum(0)
        dx += d2 @ P["w" + t]
    gr["x"] = R(dx)
    return gr


def bert_layer_flops(B, S, H, NH, FF):
    """Algorithmic GEMM FLOPs of one fwd+bwd step."""
    T = B * S
    fwd = 2 * T * H * (3 * H) + 2 * 2 * B * NH * S * S * (H // NH) + 2 * T * H * H \
        + 2 * 2 * T * H * FF
    return 3 * fwd


# ---------------------------------------------------------------------------
# a9-a13: MBConv (NCHW, as the reference)


def dwconv(x, w, stride=1, pads=(1, 1, 1, 1)):
    """Depthwise Conv, group=C, weight (C,1,kh,kw) (frontend.py:645-666)."""
    x, w = _a(x), _a(w)
    n, c, h, wi = x.shape
    _, _, kh, kw = w.shape
    pt, pl, pb, pr = pads
    xp = np.pad(x, ((0, 0), (0, 0), (pt, pb), (pl, pr)))
    oh = (h + pt + pb - kh) // stride + 1
    ow = (wi + pl + pr - kw) // stride + 1
    out = np.zeros((n, c, oh, ow))
    for i in range(kh):
        for j in range(kw):
            win = xp[:, :, i:i + oh * stride:stride, j:j + ow * stride:stride]
            out += win * w[:, 0, i, j].reshape(1, -1, 1, 1)
    return out


def dwconv_bwd(dz, x, w, stride=1, pads=(1, 1, 1, 1)):
    """Transposed scatter of the lowered conv loop nest (lowering.py:930-1004
    differentiated by tasklet VJPs): dx[.., i*s+ky-pt, j*s+kx-pl] += dz*w,
    dw[c,ky,kx] += dz * xpad window."""
    dz, x, w = _a(dz), _a(x), _a(w)
    n, c, h, wi = x.shape
    _, _, kh, kw = w.shape
    pt, pl, pb, pr = pads
    _, _, oh, ow = dz.shape
    xp = np.pad(x, ((0, 0), (0, 0), (pt, pb), (pl, pr)))
    dxp = np.zeros_like(xp)
    dw = np.zeros_like(w)
    for i in range(kh):
        for j in range(kw):
            sl = (slice(None), slice(None), slice(i, i + oh * stride, stride),
                  slice(j, j + ow * stride, stride))
            dxp[sl] += dz * w[:, 0, i, j].reshape(1, -1, 1, 1)
            dw[:, 0, i, j] = (dz * xp[sl]).sum(axis=(0, 2, 3))
    dx = dxp[:, :, pt:pt + h, pl:pl + wi]
    return dx, dw


def batchnorm_train(x, scale, bias, run_mean, run_var, eps=1e-5, momentum=0.9):
    """Training-mode BatchNormalization (frontend.py:558-591)."""
    x = _a(x)
    axes = tuple(a for a in range(x.ndim) if a != 1)
    shp = (1, -1) + (1,) * (x.ndim - 2)
    mu = x.mean(axis=axes)
    var = ((x - mu.reshape(shp)) ** 2).mean(axis=axes)
    y = (x - mu.reshape(shp)) / np.sqrt(var.reshape(shp) + eps)
    y = y * _a(scale).reshape(shp) + _a(bias).reshape(shp)
    new_mean = _a(run_mean) * momentum + mu * (1.0 - momentum)
    new_var = _a(run_var) * momentum + var * (1.0 - momentum)
    return y, new_mean, new_var, mu, var


def batchnorm_train_bwd(dy, x, scale, eps=1e-5):
    """autodiff.py:1557-1617."""
    dy, x = _a(dy), _a(x)
    axes = tuple(a for a in range(x.ndim) if a != 1)
    shp = (1, -1) + (1,) * (x.ndim - 2)
    mu = x.mean(axis=axes, keepdims=True)
    xc = x - mu
    var = (xc * xc).mean(axis=axes, keepdims=True)
    rstd = 1.0 / np.sqrt(var + eps)
    xhat = xc * rstd
    m1 = dy.mean(axis=axes, keepdims=True)
    m2 = (dy * xhat).mean(axis=axes, keepdims=True)
    dx = _a(scale).reshape(shp) * rstd * (dy - m1 - xhat * m2)
    return dx, (dy * xhat).sum(axis=axes), dy.sum(axis=axes)


def sigmoid(x):
    """frontend.py:229."""
    return 1.0 / (1.0 + np.exp(-_a(x)))


def swish(x):
    x = _a(x)
    return x * sigmoid(x)


def swish_grad(x):
    s = sigmoid(x)
    return s + _a(x) * s * (1.0 - s)


MBCONV_WEIGHTS = ("wdw", "g", "b", "rm", "rv", "wr", "br", "we", "be")


def mbconv_fwd(prm, x, stride=1, eps=1e-3, momentum=0.99, rnd=None, pads=(1, 1, 1, 1)):
    """dw3x3 + BN(train) + swish + squeeze-excite (SURVEY.md:512-514).

    ``rnd`` is the storage model (see bert_layer_fwd): applied to z, the only
    full-size intermediate the B200 path stores; BN statistics come from the
    unrounded z, as on the GPU."""
    R = rnd or _ident
    P = {k: _a(v) for k, v in prm.items()}
    x = _a(x)
    n, c = x.shape[:2]
    z_exact = dwconv(x, P["wdw"], stride, pads)
    _, new_rm, new_rv, mu, var = batchnorm_train(z_exact, P["g"], P["b"], P["rm"], P["rv"], eps, momentum)
    z = R(z_exact)
    shp = (1, -1, 1, 1)
    u = (z - mu.reshape(shp)) / np.sqrt(var.reshape(shp) + eps) * P["g"].reshape(shp) + P["b"].reshape(shp)
    a = swish(u)
    pooled = a.mean(axis=(2, 3))
    r = gemm(pooled, P["wr"], P["br"], trans_b=True)
    r2 = swish(r)
    e = gemm(r2, P["we"], P["be"], trans_b=True)
    s = sigmoid(e)
    y = R(a * s.reshape(n, c, 1, 1))
    cache = dict(x=x, z=z, u=u, a=a, pooled=pooled, r=r, r2=r2, e=e, s=s, stride=stride, eps=eps,
                 mu=mu, var=var, rnd=R, pads=pads)
    return y, new_rm, new_rv, cache


def mbconv_bwd(prm, cache, dy):
    P = {k: _a(v) for k, v in prm.items()}
    c = cache
    R = c.get("rnd") or _ident
    dy = _a(dy)
    n, ch, oh, ow = dy.shape
    gr = {}
    s4 = c["s"].reshape(n, ch, 1, 1)
    ds = (dy * c["a"]).sum(axis=(2, 3))
    de = ds * c["s"] * (1.0 - c["s"])
    gr["we"] = de.T @ c["r2"]
    gr["be"] = de.sum(0)
    dr2 = de @ P["we"]
    dr = dr2 * swish_grad(c["r"])
    gr["wr"] = dr.T @ c["pooled"]
    gr["br"] = dr.sum(0)
    dpooled = dr @ P["wr"]
    da = dy * s4 + dpooled.reshape(n, ch, 1, 1) / (oh * ow)
    du = da * swish_grad(c["u"])
    # BN VJP (autodiff.py:1557-1617) with the forward batch statistics
    shp = (1, -1, 1, 1)
    rstd = 1.0 / np.sqrt(c["var"] + c["eps"])
    xhat = (c["z"] - c["mu"].reshape(shp)) * rstd.reshape(shp)
    m1 = du.mean(axis=(0, 2, 3), keepdims=True)
    m2 = (du * xhat).mean(axis=(0, 2, 3), keepdims=True)
    dz = P["g"].reshape(shp) * rstd.reshape(shp) * (du - m1 - xhat * m2)
    gr["g"] = (du * xhat).sum(axis=(0, 2, 3))
    gr["b"] = du.sum(axis=(0, 2, 3))
    dx, gr["wdw"] = dwconv_bwd(dz, c["x"], P["wdw"], c["stride"], c.get("pads", (1, 1, 1, 1)))
    gr["x"] = R(dx)
    return gr


# ---------------------------------------------------------------------------
# C4: normalisation sweep (LN over last axis / BN over channel axis, + swish)


def ln_swish_fwd(x, g, b, eps=1e-5):
    u = layernorm(x, g, b, eps)
    return swish(u), u


def ln_swish_bwd(dy, x, g, b, eps=1e-5):
    u = layernorm(x, g, b, eps)
    du = _a(dy) * swish_grad(u)
    dx, dg, db = layernorm_bwd(du, x, g, eps)
    red = tuple(range(_a(x).ndim - 1))
    return dx, dg.sum(axis=red) if dg.ndim > 1 else dg, db.sum(axis=red) if db.ndim > 1 else db


def bn_swish_fwd(x, g, b, rm, rv, eps=1e-5, momentum=0.9):
    u, nrm, nrv, mu, var = batchnorm_train(x, g, b, rm, rv, eps, momentum)
    return swish(u), nrm, nrv


def bn_swish_bwd(dy, x, g, b, eps=1e-5):
    u = batchnorm_train(x, g, b, np.zeros_like(_a(g)), np.ones_like(_a(g)), eps)[0]
    du = _a(dy) * swish_grad(u)
    return batchnorm_train_bwd(du, x, g, eps)
