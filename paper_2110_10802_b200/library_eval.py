"""``library_eval`` — the drop-in execution seam of the reference interpreter.

The reference executes every LibraryNode through

    _Execution.run_library -> self.library_eval(node.op, node.attrs, inputs)
                                                        interp.py:337-368
    default: frontend.reference_apply(op, attrs, inputs) frontend.py:146-150

with ``inputs`` a list of numpy arrays (possibly views into interpreter
storage) and the result a list of arrays that the interpreter casts and
writes back.  ``library_eval`` below has exactly that signature, so

    dfir.interp.execute(g, inputs, bindings, library_eval=library_eval)

runs the hot-path operators of a dfir graph on the B200.  Each call copies
its host arrays to HBM, launches the sm_100a kernels through the C ABI
(include/dfx.h) and copies the results back.  Operators outside the hot path
raise ``UnsupportedOp`` — there is no CPU fallback.  Attribute
handling follows ``frontend.normalize_attrs`` (registry.py).

Arithmetic is fp32 (the tensor cores are used for bf16 only).  The reference
evaluates every operator in float64 and casts back to the input dtype
(frontend.py:146-150, 216-218); for f32 graphs that is what happens here too
(fp32 arithmetic, f32 results).  f64 graphs are REJECTED by default — the B200
path has no f64 arithmetic and silently computing in fp32 would change the
reference's numerics; ``make_library_eval(f64="as_f32")`` opts in explicitly
(results are cast back to f64).

``Reshape`` / ``Flatten`` are pure metadata in row-major storage (no bytes
move, no arithmetic); they are answered with a view of the input so a graph
that keeps them as library nodes still runs.
"""

from __future__ import annotations

import ctypes
import string

import numpy as np
import torch

from . import _lib
from . import kernels as K
from ._lib import EPI_ADD, EPI_NONE
from .errors import ShapeError, UnsupportedOp
from .registry import get_op, normalize_attrs

__all__ = ["library_eval", "SUPPORTED_OPS"]


_POLICY = {"f64": "reject"}


def _dev(a, dtype=torch.float32):
    arr = np.asarray(a)
    if arr.dtype == np.float64 and _POLICY["f64"] != "as_f32":
        raise ShapeError("B200 path computes in fp32: f64 operands are rejected (the reference evaluates f64; "
                         "use make_library_eval(f64='as_f32') to accept fp32 arithmetic explicitly)")
    if arr.dtype not in (np.float32, np.float64):
        raise ShapeError(f"B200 path takes f32 tensors, got {arr.dtype}")
    # a private, writable, contiguous fp32 copy: the interpreter hands in
    # read-only views of its storage (interp.py:348)
    host = torch.from_numpy(np.array(arr, dtype=np.float32, order="C", copy=True))
    return host.to("cuda", dtype=dtype)


def _host(t, like):
    return t.float().cpu().numpy().astype(np.asarray(like).dtype, copy=False)


def _keep(mask):
    """Reference float dropout mask (keep/(1-p)) -> (u8 keep flags, scale)."""
    m = np.asarray(mask)
    nz = m[m != 0]
    scale = float(nz.flat[0]) if nz.size else 1.0
    if nz.size and not np.all(nz == scale):
        raise ShapeError("dropout mask must hold a single non-zero value (keep / (1 - p))")
    return torch.from_numpy(np.ascontiguousarray((m != 0).astype(np.uint8))).cuda(), scale


# ---------------------------------------------------------------------------
# contractions


def _gemm_nt(a, b, alpha=1.0, c=None, beta=1.0):
    """a [nb, m, k], b [nb, n, k] (host) -> alpha * a b^T (+ beta c)."""
    ta, tb = _dev(a), _dev(b)
    d = torch.empty(ta.shape[0], ta.shape[1], tb.shape[1], device="cuda")
    if c is None:
        K.gemm(ta, tb, d, EPI_NONE, alpha=alpha)
    else:
        K.gemm(ta, tb, d, EPI_ADD, alpha=alpha, beta=beta, aux=_dev(np.broadcast_to(c, d.shape)))
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


def _einsum(attrs, inputs):
    """Two-operand Einsum as one batched GEMM: batch letters (A, B, out),
    m letters (A, out), n letters (B, out), k letters (A, B)."""
    (ta, tb), out = _parse_einsum(attrs["equation"], 2)
    a, b = (np.asarray(x) for x in inputs)
    for t, x in ((ta, a), (tb, b)):
        if len(set(t)) != len(t):
            raise UnsupportedOp("Einsum with a repeated index inside one operand")
        if len(t) != x.ndim:
            raise ShapeError(f"Einsum: term {t!r} has {len(t)} indices for rank {x.ndim} operand")
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
    size = lambda ls: int(np.prod([ext[c] for c in ls], dtype=np.int64)) if ls else 1  # noqa: E731
    A = np.transpose(a, [ta.index(c) for c in bl + ml + kl]).reshape(size(bl), size(ml), size(kl))
    B = np.transpose(b, [tb.index(c) for c in bl + nl + kl]).reshape(size(bl), size(nl), size(kl))
    d = _gemm_nt(A, B)
    res = _host(d, a).reshape([ext[c] for c in bl + ml + nl])
    return [np.transpose(res, [(bl + ml + nl).index(c) for c in out])]


def _gemm(attrs, inputs):
    a, b = np.asarray(inputs[0]), np.asarray(inputs[1])
    if a.ndim != 2 or b.ndim != 2:
        raise ShapeError("Gemm: A and B must be rank 2")
    A = a.T if attrs["transA"] else a
    Bn = b if attrs["transB"] else b.T  # [n, k]
    if A.shape[1] != Bn.shape[1]:
        raise ShapeError(f"Gemm: contracted dims differ: {A.shape[1]} vs {Bn.shape[1]}")
    c = np.asarray(inputs[2]) if len(inputs) == 3 else None
    d = _gemm_nt(A[None], Bn[None], float(attrs["alpha"]), None if c is None else c, float(attrs["beta"]))
    return [_host(d[0], a)]


def _matmul(attrs, inputs):
    a, b = np.asarray(inputs[0]), np.asarray(inputs[1])
    a2 = a[None] if a.ndim == 1 else a
    b2 = b[:, None] if b.ndim == 1 else b
    if a2.shape[-1] != b2.shape[-2]:
        raise ShapeError(f"MatMul: contracted dims differ: {a2.shape[-1]} vs {b2.shape[-2]}")
    batch = np.broadcast_shapes(a2.shape[:-2], b2.shape[:-2])
    A = np.broadcast_to(a2, batch + a2.shape[-2:]).reshape(-1, *a2.shape[-2:])
    B = np.swapaxes(np.broadcast_to(b2, batch + b2.shape[-2:]).reshape(-1, *b2.shape[-2:]), -1, -2)
    y = _host(_gemm_nt(A, B), a).reshape(batch + (a2.shape[-2], b2.shape[-1]))
    if a.ndim == 1:
        y = y[..., 0, :]
    if b.ndim == 1:
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


def _reduce(attrs, inputs, mean=False):
    """ReduceSum / ReduceMean (frontend.py:302-328): the reduced axes are moved
    to the front and summed by the fixed-order column-sum kernel."""
    x = np.asarray(inputs[0])
    axes = _norm_axes(attrs["axes"], x.ndim)
    kept = [a for a in range(x.ndim) if a not in axes]
    rows = int(np.prod([x.shape[a] for a in axes], dtype=np.int64))
    cols = int(np.prod([x.shape[a] for a in kept], dtype=np.int64))
    xt = np.transpose(x, list(axes) + kept).reshape(rows, cols)
    pad = -cols % 8  # the column-sum kernel reads 16-byte vectors: pad with zero columns
    t = _dev(np.pad(xt, ((0, 0), (0, pad))) if pad else xt)
    out = torch.empty(cols + pad, device="cuda")
    K.colsum(t, out)
    out = out[:cols]
    if mean:
        K.scale_(out, 1.0 / max(rows, 1))
    shape = [1 if a in axes else x.shape[a] for a in range(x.ndim)] if attrs["keepdims"] else \
        [x.shape[a] for a in kept]
    return [_host(out, x).reshape(shape)]


def _reshape(attrs, inputs):
    """Reshape / Flatten are metadata on row-major storage (frontend.py:713-829)."""
    x = np.asarray(inputs[0])
    if "axis" in attrs:  # Flatten
        ax = int(attrs["axis"]) % max(x.ndim, 1)
        return [x.reshape(int(np.prod(x.shape[:ax], dtype=np.int64)), -1)]
    shape = [int(v) for v in attrs["shape"]]
    shape = [x.shape[i] if v == 0 else v for i, v in enumerate(shape)]
    return [x.reshape(shape)]


# ---------------------------------------------------------------------------
# normalisations


def _layernorm(attrs, inputs, act=0):
    x = np.asarray(inputs[0])
    axis = int(attrs["axis"]) % x.ndim
    cols = int(np.prod(x.shape[axis:], dtype=np.int64))
    g = np.asarray(inputs[1]).reshape(-1)
    be = np.asarray(inputs[2]).reshape(-1) if len(inputs) == 3 else np.zeros(cols)
    if g.size != cols or be.size != cols:
        raise ShapeError("LayerNormalization: scale/bias must match the normalized shape")
    tx = _dev(x.reshape(-1, cols))
    tg, tb = _dev(g), _dev(be)  # keep the uploads alive until the launch is queued
    y = torch.empty_like(tx)
    _lib.call("dfx_layernorm_act_fwd", _lib.DFX_F32, tx.shape[0], cols, tx.data_ptr(), tg.data_ptr(),
              tb.data_ptr(), float(attrs["epsilon"]), act, y.data_ptr(), K._stream())
    return [_host(y, x).reshape(x.shape)]


def _softmax(attrs, inputs):
    x = np.asarray(inputs[0])
    axis = int(attrs["axis"]) % x.ndim
    xm = np.moveaxis(x, axis, -1)
    t = _dev(xm.reshape(1, 1, -1, xm.shape[-1]))
    p = torch.empty_like(t)
    K.softmax_fwd(t, 1.0, None, None, 1.0, p=p)
    return [np.moveaxis(_host(p, x).reshape(xm.shape), -1, axis)]


def _batchnorm(attrs, inputs, act=0):
    x, g, b, rm, rv = (np.asarray(v) for v in inputs)
    if x.ndim < 2:
        raise ShapeError("BatchNormalization: input must have a channel dim")
    C = x.shape[1]
    xl = np.moveaxis(x, 1, -1)
    tx = _dev(xl.reshape(-1, C))
    rows = tx.shape[0]
    f = lambda *s: torch.empty(s, device="cuda")  # noqa: E731
    local, mean, var, rstd = f(3, C), f(C), f(C), f(C)
    trm, trv = _dev(rm), _dev(rv)
    ws = K.WORKSPACE.get(_lib.load().dfx_batchnorm_workspace(rows, C))
    st = K._stream()
    _lib.call("dfx_batchnorm_stats", _lib.DFX_F32, rows, C, tx.data_ptr(), local.data_ptr(), ws.data_ptr(),
              ws.numel(), st)
    _lib.call("dfx_bn_finalize", C, 1, local.data_ptr(), float(attrs["epsilon"]), float(attrs["momentum"]),
              mean.data_ptr(), var.data_ptr(), rstd.data_ptr(), trm.data_ptr(), trv.data_ptr(), st)
    y = torch.empty_like(tx)
    tg, tb = _dev(g), _dev(b)
    _lib.call("dfx_batchnorm_act_apply", _lib.DFX_F32, rows, C, tx.data_ptr(), mean.data_ptr(), rstd.data_ptr(),
              tg.data_ptr(), tb.data_ptr(), act, y.data_ptr(), st)
    yo = np.moveaxis(_host(y, x).reshape(xl.shape), -1, 1)
    return [yo, _host(trm, rm), _host(trv, rv)]


# ---------------------------------------------------------------------------
# MBConv (depthwise conv) pieces


def _pads_strides(attrs):
    strides = [int(s) for s in (attrs.get("strides") or [1, 1])]
    pads = [int(p) for p in (attrs.get("pads") or [0, 0, 0, 0])]
    if len(strides) != 2 or strides[0] != strides[1] or strides[0] not in (1, 2):
        raise UnsupportedOp("Conv: the B200 depthwise path takes equal strides of 1 or 2")
    return strides[0], pads


def _conv(attrs, inputs):
    x, w = np.asarray(inputs[0]), np.asarray(inputs[1])
    if x.ndim != 4 or w.ndim != 4:
        raise ShapeError("Conv: X and W must be rank 4 (N, C, H, W)")
    N, C, H, W = x.shape
    k = w.shape[-1]
    if int(attrs["group"]) != C or w.shape != (C, 1, k, k) or k not in (3, 5):
        raise UnsupportedOp("Conv: only depthwise 3x3 / 5x5 (group = C, weight (C,1,k,k)) runs on the B200 path")
    stride, pads = _pads_strides(attrs)
    tx = _dev(np.moveaxis(x, 1, -1))
    tw = _dev(w.reshape(C, k * k).T)
    Ho = (H + pads[0] + pads[2] - k) // stride + 1
    Wo = (W + pads[1] + pads[3] - k) // stride + 1
    z = torch.empty(N, Ho, Wo, C, device="cuda")
    local = torch.empty(3, C, device="cuda")
    pc = (ctypes.c_int * 4)(*pads)
    ws = K.WORKSPACE.get(_lib.load().dfx_mbconv_workspace(N, H, W, C, stride, k, pc, 1))
    _lib.call("dfx_mbconv_fwd_stats", _lib.DFX_F32, N, H, W, C, stride, k, pc, tx.data_ptr(), tw.data_ptr(),
              z.data_ptr(), local.data_ptr(), ws.data_ptr(), ws.numel(), K._stream())
    return [np.moveaxis(_host(z, x), -1, 1)]


def _mbconv_block(attrs, inputs, grad=False):
    from .mbconv import MBConvBlock, MBConvConfig

    if grad:
        dy, x = np.asarray(inputs[0]), np.asarray(inputs[1])
        rest = inputs[2:]
    else:
        x = np.asarray(inputs[0])
        rest = inputs[1:]
    wdw, g, b, rm, rv, wr, br, we, be = (np.asarray(v) for v in rest)
    stride, pads = _pads_strides(attrs)
    N, C, H, W = x.shape
    blk = MBConvBlock(MBConvConfig(channels=C, se=wr.shape[0], stride=stride, pads=tuple(pads),
                                   eps=float(attrs["epsilon"]), momentum=float(attrs["momentum"]),
                                   dtype=torch.float32))
    blk.load_params(dict(wdw=wdw, g=g, b=b, rm=rm, rv=rv, wr=wr, br=br, we=we, be=be))
    y = blk.forward(_dev(np.moveaxis(x, 1, -1)))
    if not grad:
        return [np.moveaxis(_host(y, x), -1, 1), _host(blk.running_mean, rm), _host(blk.running_var, rv)]
    dx = blk.backward(_dev(np.moveaxis(dy, 1, -1)))
    gr = blk.grads_numpy()
    cast = lambda a: np.asarray(a).astype(x.dtype)  # noqa: E731
    return [np.moveaxis(_host(dx, x), -1, 1), cast(gr["wdw"]), cast(gr["g"]), cast(gr["b"]), cast(gr["wr"]),
            cast(gr["br"]), cast(gr["we"]), cast(gr["be"])]


# ---------------------------------------------------------------------------
# fused BERT row operators


def _bdrln(attrs, inputs):
    h, bias, mask, res, g, be = (np.asarray(v) for v in inputs)
    keep, ks = _keep(mask)
    th = _dev(h)
    y, s = torch.empty_like(th), torch.empty_like(th)
    K.bdrln_fwd(th, _dev(bias), keep, ks, _dev(res), _dev(g), _dev(be), float(attrs["epsilon"]), y=y, s=s)
    return [_host(y, h), _host(s, h)]


def _bdrln_grad(attrs, inputs):
    dy, s, g, mask = (np.asarray(v) for v in inputs)
    keep, ks = _keep(mask)
    tdy = _dev(dy)
    H = dy.shape[-1]
    ds, dh = torch.empty_like(tdy), torch.empty_like(tdy)
    dg, dbe, dbi = (torch.empty(H, device="cuda") for _ in range(3))
    K.bdrln_bwd(tdy, _dev(s), _dev(g), keep, ks, float(attrs["epsilon"]), ds=ds, dh=dh, dgamma=dg, dbeta=dbe,
                dbias=dbi)
    return [_host(ds, dy), _host(dh, dy), _host(dbi, dy), _host(dg, dy), _host(dbe, dy)]


def _sm_fused(attrs, inputs):
    sc, am, dm = (np.asarray(v) for v in inputs)
    if sc.ndim != 4:
        raise ShapeError("ScaledMaskedSoftmax: scores must be [B, NH, Q, K]")
    B, NH, Q, Kc = sc.shape
    keep, ks = _keep(dm)
    t = _dev(sc)
    p, pd = torch.empty_like(t), torch.empty_like(t)
    K.softmax_fwd(t, 1.0 / float(attrs["divisor"]), _dev(np.broadcast_to(am, (B, 1, 1, Kc)).reshape(B, Kc)),
                  keep, ks, p, pd)
    return [_host(pd, sc), _host(p, sc)]


def _sm_fused_grad(attrs, inputs):
    dpd, p, dm = (np.asarray(v) for v in inputs)
    keep, ks = _keep(dm)
    out = K.softmax_bwd(_dev(dpd), _dev(p), keep, ks, 1.0 / float(attrs["divisor"]))
    return [_host(out, dpd)]


def _bias_gelu(attrs, inputs):
    f, b = (np.asarray(v) for v in inputs)
    tf = _dev(f)
    pre = torch.empty_like(tf)
    y = K.bias_gelu_fwd(tf, _dev(b), pre=pre)
    return [_host(y, f), _host(pre, f)]


def _bias_gelu_grad(attrs, inputs):
    dy, pre = (np.asarray(v) for v in inputs)
    db = torch.empty(dy.shape[-1], device="cuda")
    dpre = K.bias_gelu_bwd(_dev(dy), _dev(pre), dbias=db)
    return [_host(dpre, dy), _host(db, dy)]


def _ln_act_grad(attrs, inputs):
    from .norms import LayerNormAct

    dy, x, g, b = (np.asarray(v) for v in inputs)
    H = x.shape[-1]
    m = LayerNormAct(H, eps=float(attrs["epsilon"]), act=attrs["activation"])
    m.gamma.copy_(_dev(g))
    m.beta.copy_(_dev(b))
    m.forward(_dev(x))
    dx = m.backward(_dev(dy))
    return [_host(dx, x), _host(m.dgamma, g), _host(m.dbeta, b)]


def _bn_act_grad(attrs, inputs):
    """BN(+act) VJP with the batch statistics recomputed from x (as the
    reference's _bwd_batchnorm does, autodiff.py:1569-1574)."""
    from .norms import BatchNormAct

    dy, x, g, b = (np.asarray(v) for v in inputs)
    if x.ndim < 2:
        raise ShapeError("BatchNormActGrad: input must have a channel dim")
    C = x.shape[1]
    m = BatchNormAct(C, eps=float(attrs["epsilon"]), act=attrs["activation"])
    m.gamma.copy_(_dev(g))
    m.beta.copy_(_dev(b))
    m.forward(_dev(np.moveaxis(x, 1, -1)))
    dx = m.backward(_dev(np.moveaxis(dy, 1, -1)))
    return [np.moveaxis(_host(dx, x).reshape(np.moveaxis(x, 1, -1).shape), -1, 1), _host(m.dgamma, g),
            _host(m.dbeta, b)]


def _ln_act(attrs, inputs):
    return _layernorm({"axis": -1, "epsilon": attrs["epsilon"]}, inputs, act=_act_code(attrs))


def _bn_act(attrs, inputs):
    return _batchnorm(attrs, inputs, act=_act_code(attrs))


def _act_code(attrs):
    a = attrs["activation"]
    if a not in ("none", "swish"):
        raise UnsupportedOp(f"activation {a!r}")
    return 1 if a == "swish" else 0


_DISPATCH = {
    "Gemm": _gemm, "MatMul": _matmul, "Einsum": _einsum, "LayerNormalization": _layernorm,
    "Softmax": _softmax, "BatchNormalization": _batchnorm, "Conv": _conv,
    "BiasDropoutResidualLayerNorm": _bdrln, "BiasDropoutResidualLayerNormGrad": _bdrln_grad,
    "ScaledMaskedSoftmax": _sm_fused, "ScaledMaskedSoftmaxGrad": _sm_fused_grad,
    "BiasGelu": _bias_gelu, "BiasGeluGrad": _bias_gelu_grad,
    "MBConvBlock": _mbconv_block, "MBConvBlockGrad": lambda a, i: _mbconv_block(a, i, grad=True),
    "LayerNormAct": _ln_act, "BatchNormAct": _bn_act,
    "LayerNormActGrad": _ln_act_grad, "BatchNormActGrad": _bn_act_grad,
    "ReduceSum": _reduce, "ReduceMean": lambda a, i: _reduce(a, i, mean=True),
    "Reshape": _reshape, "Flatten": _reshape,
}
SUPPORTED_OPS = sorted(_DISPATCH)


def library_eval(op: str, attrs, inputs):
    """Evaluate one operator on the B200 (same contract as
    frontend.reference_apply).  Raises UnsupportedOp for operators that are
    not on the hot path — never falls back to the CPU."""
    fn = _DISPATCH.get(op)
    if fn is None:
        raise UnsupportedOp(op)
    spec = get_op(op)
    if not (spec.min_inputs <= len(inputs) <= spec.max_inputs):
        raise ShapeError(f"{op}: takes {spec.min_inputs}..{spec.max_inputs} inputs, got {len(inputs)}")
    _lib.load(check_device=True)
    # results come back as host arrays (the seam's contract); the D2H copies
    # inside _host already order them after the kernels
    return fn(normalize_attrs(spec, attrs), list(inputs))


def make_library_eval(f64: str = "reject"):
    """A ``library_eval`` with an explicit f64 policy: ``"reject"`` (default,
    raise ShapeError) or ``"as_f32"`` (compute in fp32, cast results back)."""
    if f64 not in ("reject", "as_f32"):
        raise ValueError("f64 policy must be 'reject' or 'as_f32'")

    def evaluate(op, attrs, inputs):
        saved = _POLICY["f64"]
        _POLICY["f64"] = f64
        try:
            return library_eval(op, attrs, inputs)
        finally:
            _POLICY["f64"] = saved

    return evaluate
