"""Device-resident operator implementations (torch tensors in, torch tensors out).

One implementation of every operator the B200 path executes, on CUDA tensors
and on the current stream, with no host round trip: ``library_eval`` (the
reference interpreter's host-array seam, library_eval.py) wraps these with
host<->device copies, and ``dfm.DeviceGraph`` runs whole ``dfm-0.1`` models
through them with every intermediate resident in HBM.

Semantics follow the reference evaluators (frontend.py:302-829) and the fused
operator specs (registry.py); arithmetic is fp32 (CUDA-core fp32 GEMMs: TF32
would miss the reference's 1e-4 bar) except where a bf16 tensor is passed in.
Operators outside the hot path raise ``UnsupportedOp`` — no CPU fallback.
"""

from __future__ import annotations

import ctypes
import string

import torch

from . import _lib
from . import kernels as K
from ._lib import EPI_ADD, EPI_NONE
from .errors import ShapeError, UnsupportedOp

__all__ = ["DEVICE_OPS", "run_op", "keep_of"]


def _f32(t):
    if not t.is_cuda:
        raise ShapeError("device op: operands must be CUDA tensors")
    return t.contiguous() if t.dtype == torch.float32 else t.float().contiguous()


def keep_of(mask):
    """Reference float dropout mask (keep/(1-p)) -> (u8 keep flags, scale).
    The scale is read back once (one host sync per masked operator)."""
    m = _f32(mask)
    keep = (m != 0).to(torch.uint8)
    nz = m[m != 0]
    if nz.numel() == 0:
        return keep, 1.0
    lo, hi = float(nz.amin()), float(nz.amax())
    if lo != hi:
        raise ShapeError("dropout mask must hold a single non-zero value (keep / (1 - p))")
    return keep, hi


# ---------------------------------------------------------------------------
# contractions


def gemm_nt(a, b, alpha=1.0, c=None, beta=1.0):
    """a [nb, m, k], b [nb, n, k] -> alpha * a b^T (+ beta c)."""
    ta, tb = _f32(a), _f32(b)
    d = torch.empty(ta.shape[0], ta.shape[1], tb.shape[1], device=ta.device)
    if c is None:
        K.gemm(ta, tb, d, EPI_NONE, alpha=alpha)
    else:
        K.gemm(ta, tb, d, EPI_ADD, alpha=alpha, beta=beta, aux=_f32(c).expand(d.shape).contiguous())
    return d


def _parse_einsum(eq, n):
    eq = eq.replace(" ", "")
    if "." in eq:
        raise ShapeError("Einsum: ellipsis is not supported")
    lhs, rhs = eq.split("->") if "->" in eq else (eq, None)
    terms = lhs.split(",")
    if len(terms) != n:
        raise ShapeError(f"Einsum: equation {eq!r} names {len(terms)} operands, got {n}")
    if rhs is None:
        cnt = {}
        for t in terms:
            for ch in t:
                cnt[ch] = cnt.get(ch, 0) + 1
        rhs = "".join(sorted(ch for ch, v in cnt.items() if v == 1))
    for t in terms + [rhs]:
        if any(ch not in string.ascii_lowercase for ch in t):
            raise ShapeError("Einsum: only lowercase index letters allowed")
    return terms, rhs


def einsum(attrs, inputs):
    """Two-operand Einsum as one batched GEMM: batch letters (A, B, out),
    m letters (A, out), n letters (B, out), k letters (A, B)."""
    (ta, tb), out = _parse_einsum(attrs["equation"], 2)
    a, b = inputs
    for t, x in ((ta, a), (tb, b)):
        if len(set(t)) != len(t):
            raise UnsupportedOp("Einsum with a repeated index inside one operand")
        if len(t) != x.dim():
            raise ShapeError(f"Einsum: term {t!r} has {len(t)} indices for rank {x.dim()} operand")
    ext = {}
    for t, x in ((ta, a), (tb, b)):
        for ch, d in zip(t, x.shape):
            if ext.setdefault(ch, d) != d:
                raise ShapeError(f"Einsum: index {ch!r} bound to both {ext[ch]} and {d}")
    bl = [c for c in out if c in ta and c in tb]
    ml = [c for c in out if c in ta and c not in tb]
    nl = [c for c in out if c in tb and c not in ta]
    kl = [c for c in ta if c in tb and c not in out]
    if any(c not in out and c not in tb for c in ta) or any(c not in out and c not in ta for c in tb):
        raise UnsupportedOp("Einsum summing an index of a single operand (a reduction, not a contraction)")

    def size(ls):
        n = 1
        for c in ls:
            n *= ext[c]
        return n

    A = _f32(a).permute([ta.index(c) for c in bl + ml + kl]).reshape(size(bl), size(ml), size(kl))
    B = _f32(b).permute([tb.index(c) for c in bl + nl + kl]).reshape(size(bl), size(nl), size(kl))
    d = gemm_nt(A, B).reshape([ext[c] for c in bl + ml + nl])
    return [d.permute([(bl + ml + nl).index(c) for c in out]).contiguous()]


def gemm(attrs, inputs):
    a, b = inputs[0], inputs[1]
    if a.dim() != 2 or b.dim() != 2:
        raise ShapeError("Gemm: A and B must be rank 2")
    A = a.t() if attrs["transA"] else a
    Bn = b if attrs["transB"] else b.t()  # [n, k]
    if A.shape[1] != Bn.shape[1]:
        raise ShapeError(f"Gemm: contracted dims differ: {A.shape[1]} vs {Bn.shape[1]}")
    c = inputs[2] if len(inputs) == 3 else None
    d = gemm_nt(A.unsqueeze(0), Bn.unsqueeze(0), float(attrs["alpha"]), c, float(attrs["beta"]))
    return [d[0]]


def matmul(attrs, inputs):
    a, b = inputs
    a2 = a.unsqueeze(0) if a.dim() == 1 else a
    b2 = b.unsqueeze(-1) if b.dim() == 1 else b
    if a2.shape[-1] != b2.shape[-2]:
        raise ShapeError(f"MatMul: contracted dims differ: {a2.shape[-1]} vs {b2.shape[-2]}")
    batch = torch.broadcast_shapes(a2.shape[:-2], b2.shape[:-2])
    A = a2.expand(*batch, *a2.shape[-2:]).reshape(-1, *a2.shape[-2:])
    B = b2.expand(*batch, *b2.shape[-2:]).reshape(-1, *b2.shape[-2:]).transpose(-1, -2)
    y = gemm_nt(A, B).reshape(*batch, a2.shape[-2], b2.shape[-1])
    if a.dim() == 1:
        y = y[..., 0, :]
    if b.dim() == 1:
        y = y[..., 0]
    return [y]


# ---------------------------------------------------------------------------
# reductions and layout


def _norm_axes(axes, rank):
    if axes is None or (not isinstance(axes, int) and len(list(axes)) == 0):
        return tuple(range(rank))
    axes = [axes] if isinstance(axes, int) else list(axes)
    out = sorted({int(a) % rank for a in axes})
    if len(out) != len(axes):
        raise ShapeError(f"repeated axis in {axes}")
    return tuple(out)


def reduce(attrs, inputs, mean=False):
    """ReduceSum / ReduceMean (frontend.py:302-328): the reduced axes are moved
    to the front and summed by the fixed-order column-sum kernel."""
    x = _f32(inputs[0])
    axes = _norm_axes(attrs["axes"], x.dim())
    kept = [a for a in range(x.dim()) if a not in axes]
    rows = 1
    for a in axes:
        rows *= x.shape[a]
    cols = x.numel() // max(rows, 1)
    xt = x.permute(list(axes) + kept).reshape(rows, cols)
    pad = -cols % 8  # the column-sum kernel reads 16-byte vectors: pad with zero columns
    if pad:
        xt = torch.nn.functional.pad(xt, (0, pad))
    xt = xt.contiguous()
    out = torch.empty(cols + pad, device=x.device)
    K.colsum(xt, out)
    if mean:
        K.scale_(out, 1.0 / max(rows, 1))
    shape = [1 if a in axes else x.shape[a] for a in range(x.dim())] if attrs["keepdims"] else \
        [x.shape[a] for a in kept]
    return [out[:cols].reshape(shape)]


def reshape(attrs, inputs):
    """Reshape / Flatten are metadata on row-major storage (frontend.py:713-829)."""
    x = inputs[0]
    if "axis" in attrs:  # Flatten
        ax = int(attrs["axis"]) % max(x.dim(), 1)
        lead = 1
        for d in x.shape[:ax]:
            lead *= d
        return [x.reshape(lead, -1)]
    shape = [int(v) for v in attrs["shape"]]
    shape = [x.shape[i] if v == 0 else v for i, v in enumerate(shape)]
    return [x.reshape(shape)]


# ---------------------------------------------------------------------------
# normalisations


def layernorm(attrs, inputs, act=0):
    x = _f32(inputs[0])
    axis = int(attrs["axis"]) % x.dim()
    cols = 1
    for d in x.shape[axis:]:
        cols *= d
    g = _f32(inputs[1]).reshape(-1)
    be = _f32(inputs[2]).reshape(-1) if len(inputs) == 3 else torch.zeros(cols, device=x.device)
    if g.numel() != cols or be.numel() != cols:
        raise ShapeError("LayerNormalization: scale/bias must match the normalized shape")
    y = torch.empty_like(x)
    _lib.call("dfx_layernorm_act_fwd", _lib.DFX_F32, x.numel() // cols, cols, x.data_ptr(), g.data_ptr(),
              be.data_ptr(), float(attrs["epsilon"]), act, y.data_ptr(), K._stream())
    return [y]


def softmax(attrs, inputs):
    x = _f32(inputs[0])
    axis = int(attrs["axis"]) % x.dim()
    xm = x.movedim(axis, -1).contiguous()
    t = xm.reshape(1, 1, -1, xm.shape[-1])
    p = torch.empty_like(t)
    K.softmax_fwd(t, 1.0, None, None, 1.0, p=p)
    return [p.reshape(xm.shape).movedim(-1, axis).contiguous()]


def batchnorm(attrs, inputs, act=0):
    x, g, b, rm, rv = (_f32(v) for v in inputs)
    if x.dim() < 2:
        raise ShapeError("BatchNormalization: input must have a channel dim")
    C = x.shape[1]
    xl = x.movedim(1, -1).contiguous()
    rows = xl.numel() // C
    f = lambda *s: torch.empty(s, device=x.device)  # noqa: E731
    local, mean, var, rstd = f(3, C), f(C), f(C), f(C)
    nrm, nrv = rm.clone(), rv.clone()
    ws = K.WORKSPACE.get(_lib.load().dfx_batchnorm_workspace(rows, C))
    st = K._stream()
    _lib.call("dfx_batchnorm_stats", _lib.DFX_F32, rows, C, xl.data_ptr(), local.data_ptr(), ws.data_ptr(),
              ws.numel(), st)
    _lib.call("dfx_bn_finalize", C, 1, local.data_ptr(), float(attrs["epsilon"]), float(attrs["momentum"]),
              mean.data_ptr(), var.data_ptr(), rstd.data_ptr(), nrm.data_ptr(), nrv.data_ptr(), st)
    y = torch.empty_like(xl)
    _lib.call("dfx_batchnorm_act_apply", _lib.DFX_F32, rows, C, xl.data_ptr(), mean.data_ptr(), rstd.data_ptr(),
              g.data_ptr(), b.data_ptr(), act, y.data_ptr(), st)
    return [y.movedim(-1, 1).contiguous(), nrm, nrv]


def _act_code(attrs):
    a = attrs["activation"]
    if a not in ("none", "swish"):
        raise UnsupportedOp(f"activation {a!r}")
    return 1 if a == "swish" else 0


def ln_act(attrs, inputs):
    return layernorm({"axis": -1, "epsilon": attrs["epsilon"]}, inputs, act=_act_code(attrs))


def bn_act(attrs, inputs):
    return batchnorm(attrs, inputs, act=_act_code(attrs))


def ln_act_grad(attrs, inputs):
    from .norms import LayerNormAct

    dy, x, g, b = (_f32(v) for v in inputs)
    m = LayerNormAct(x.shape[-1], eps=float(attrs["epsilon"]), act=attrs["activation"], device=x.device)
    m.gamma.copy_(g)
    m.beta.copy_(b)
    m.forward(x)
    dx = m.backward(dy)
    return [dx, m.dgamma, m.dbeta]


def bn_act_grad(attrs, inputs):
    """BN(+act) VJP with the batch statistics recomputed from x (as the
    reference's _bwd_batchnorm does, autodiff.py:1569-1574)."""
    from .norms import BatchNormAct

    dy, x, g, b = (_f32(v) for v in inputs)
    if x.dim() < 2:
        raise ShapeError("BatchNormActGrad: input must have a channel dim")
    m = BatchNormAct(x.shape[1], eps=float(attrs["epsilon"]), act=attrs["activation"], device=x.device)
    m.gamma.copy_(g)
    m.beta.copy_(b)
    m.forward(x.movedim(1, -1).contiguous())
    dx = m.backward(dy.movedim(1, -1).contiguous())
    return [dx.movedim(-1, 1).contiguous(), m.dgamma, m.dbeta]


# ---------------------------------------------------------------------------
# depthwise conv / MBConv


def _pads_strides(attrs):
    strides = [int(s) for s in (attrs.get("strides") or [1, 1])]
    pads = [int(p) for p in (attrs.get("pads") or [0, 0, 0, 0])]
    if len(strides) != 2 or strides[0] != strides[1] or strides[0] not in (1, 2):
        raise UnsupportedOp("Conv: the B200 depthwise path takes equal strides of 1 or 2")
    return strides[0], pads


def conv(attrs, inputs):
    x, w = _f32(inputs[0]), _f32(inputs[1])
    if x.dim() != 4 or w.dim() != 4:
        raise ShapeError("Conv: X and W must be rank 4 (N, C, H, W)")
    N, C, H, W = x.shape
    k = w.shape[-1]
    if int(attrs["group"]) != C or tuple(w.shape) != (C, 1, k, k) or k not in (3, 5):
        raise UnsupportedOp("Conv: only depthwise 3x3 / 5x5 (group = C, weight (C,1,k,k)) runs on the B200 path")
    stride, pads = _pads_strides(attrs)
    tx = x.movedim(1, -1).contiguous()
    tw = w.reshape(C, k * k).t().contiguous()
    Ho = (H + pads[0] + pads[2] - k) // stride + 1
    Wo = (W + pads[1] + pads[3] - k) // stride + 1
    z = torch.empty(N, Ho, Wo, C, device=x.device)
    local = torch.empty(3, C, device=x.device)
    pc = (ctypes.c_int * 4)(*pads)
    ws = K.WORKSPACE.get(_lib.load().dfx_mbconv_workspace(N, H, W, C, stride, k, pc, 1))
    _lib.call("dfx_mbconv_fwd_stats", _lib.DFX_F32, N, H, W, C, stride, k, pc, tx.data_ptr(), tw.data_ptr(),
              z.data_ptr(), local.data_ptr(), ws.data_ptr(), ws.numel(), K._stream())
    return [z.movedim(-1, 1).contiguous()]


def mbconv_block(attrs, inputs, grad=False):
    from .mbconv import MBConvBlock, MBConvConfig

    if grad:
        dy, x, rest = _f32(inputs[0]), _f32(inputs[1]), inputs[2:]
    else:
        x, rest = _f32(inputs[0]), inputs[1:]
    wdw, g, b, rm, rv, wr, br, we, be = (_f32(v) for v in rest)
    stride, pads = _pads_strides(attrs)
    N, C, H, W = x.shape
    blk = MBConvBlock(MBConvConfig(channels=C, se=wr.shape[0], stride=stride, pads=tuple(pads),
                                   eps=float(attrs["epsilon"]), momentum=float(attrs["momentum"]),
                                   dtype=torch.float32), device=x.device)
    blk.load_params(dict(wdw=wdw, g=g, b=b, rm=rm, rv=rv, wr=wr, br=br, we=we, be=be))
    y = blk.forward(x.movedim(1, -1).contiguous())
    if not grad:
        return [y.movedim(-1, 1).contiguous(), blk.running_mean.clone(), blk.running_var.clone()]
    dx = blk.backward(dy.movedim(1, -1).contiguous())
    G = blk.grad
    k = blk.cfg.ksize
    dwdw = G["wdw"].permute(2, 0, 1).reshape(C, 1, k, k).contiguous()
    return [dx.movedim(-1, 1).contiguous(), dwdw, G["g"].clone(), G["b"].clone(), G["wr"].clone(),
            G["br"].clone(), G["we"].clone(), G["be"].clone()]


# ---------------------------------------------------------------------------
# fused BERT row operators


def bdrln(attrs, inputs):
    h, bias, mask, res, g, be = inputs
    keep, ks = keep_of(mask)
    th = _f32(h)
    y, s = torch.empty_like(th), torch.empty_like(th)
    K.bdrln_fwd(th, _f32(bias), keep, ks, _f32(res), _f32(g), _f32(be), float(attrs["epsilon"]), y=y, s=s)
    return [y, s]


def bdrln_grad(attrs, inputs):
    dy, s, g, mask = inputs
    keep, ks = keep_of(mask)
    tdy = _f32(dy)
    H = tdy.shape[-1]
    ds, dh = torch.empty_like(tdy), torch.empty_like(tdy)
    dg, dbe, dbi = (torch.empty(H, device=tdy.device) for _ in range(3))
    K.bdrln_bwd(tdy, _f32(s), _f32(g), keep, ks, float(attrs["epsilon"]), ds=ds, dh=dh, dgamma=dg, dbeta=dbe,
                dbias=dbi)
    return [ds, dh, dbi, dg, dbe]


def sm_fused(attrs, inputs):
    sc, am, dm = inputs
    if sc.dim() != 4:
        raise ShapeError("ScaledMaskedSoftmax: scores must be [B, NH, Q, K]")
    B, NH, Q, Kc = sc.shape
    keep, ks = keep_of(dm)
    t = _f32(sc)
    p, pd = torch.empty_like(t), torch.empty_like(t)
    am2 = _f32(am).expand(B, 1, 1, Kc).reshape(B, Kc).contiguous()
    K.softmax_fwd(t, 1.0 / float(attrs["divisor"]), am2, keep, ks, p, pd)
    return [pd, p]


def sm_fused_grad(attrs, inputs):
    dpd, p, dm = inputs
    keep, ks = keep_of(dm)
    return [K.softmax_bwd(_f32(dpd), _f32(p), keep, ks, 1.0 / float(attrs["divisor"]))]


def bias_gelu(attrs, inputs):
    f, b = (_f32(v) for v in inputs)
    pre = torch.empty_like(f)
    y = K.bias_gelu_fwd(f, b, pre=pre)
    return [y, pre]


def bias_gelu_grad(attrs, inputs):
    dy, pre = (_f32(v) for v in inputs)
    db = torch.empty(dy.shape[-1], device=dy.device)
    dpre = K.bias_gelu_bwd(dy, pre, dbias=db)
    return [dpre, db]


DEVICE_OPS = {
    "Gemm": gemm, "MatMul": matmul, "Einsum": einsum, "LayerNormalization": layernorm,
    "Softmax": softmax, "BatchNormalization": batchnorm, "Conv": conv,
    "BiasDropoutResidualLayerNorm": bdrln, "BiasDropoutResidualLayerNormGrad": bdrln_grad,
    "ScaledMaskedSoftmax": sm_fused, "ScaledMaskedSoftmaxGrad": sm_fused_grad,
    "BiasGelu": bias_gelu, "BiasGeluGrad": bias_gelu_grad,
    "MBConvBlock": mbconv_block, "MBConvBlockGrad": lambda a, i: mbconv_block(a, i, grad=True),
    "LayerNormAct": ln_act, "BatchNormAct": bn_act,
    "LayerNormActGrad": ln_act_grad, "BatchNormActGrad": bn_act_grad,
    "ReduceSum": reduce, "ReduceMean": lambda a, i: reduce(a, i, mean=True),
    "Reshape": reshape, "Flatten": reshape,
}


def run_op(op: str, attrs: dict, inputs: list) -> list:
    """Evaluate one (normalised-attribute) operator on device tensors."""
    fn = DEVICE_OPS.get(op)
    if fn is None:
        raise UnsupportedOp(op)
    return fn(attrs, list(inputs))
