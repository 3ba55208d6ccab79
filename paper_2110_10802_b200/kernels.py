"""Typed wrappers over the C ABI for tensors already resident on the GPU.

PyTorch is used only as the device-memory / stream plumbing: every function
here hands raw pointers, extents and ``torch.cuda.current_stream()`` to the
sm_100a library through ``_lib`` (ctypes) and launches nothing itself.
Shapes and dtypes are validated on the host before launch (dfx.h error
contract); violations raise ``ShapeError`` like the reference's
``frontend.infer_shapes`` (frontend.py:132-143).
"""

from __future__ import annotations

import torch

from . import _lib
from ._lib import GemmArgs
from .errors import ShapeError

_DT = {torch.float32: _lib.DFX_F32, torch.bfloat16: _lib.DFX_BF16}


def dfx_dtype(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError:
        raise ShapeError(f"dtype {t.dtype} is not supported on the B200 path (f32, bf16)") from None


def _ptr(t):
    return None if t is None else t.data_ptr()


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _contig(t: torch.Tensor, name: str):
    if not t.is_cuda:
        raise ShapeError(f"{name}: tensor must be on the GPU")
    if not t.is_contiguous():
        raise ShapeError(f"{name}: tensor must be contiguous")
    return t


def _vec(t, n, name):
    if t is None:
        return None
    if t.dtype != torch.float32 or t.numel() != n:
        raise ShapeError(f"{name}: expected f32 vector of {n} elements")
    return _contig(t, name)


def _keep_arg(t, numel, name):
    """(entry-point suffix, tensor): u8/bool flags, or int32 words bit-packed by
    pack_keep_bits (bit e % 32 of word e // 32 = flag of flat element e)."""
    if t is not None and t.dtype == torch.int32:
        if t.numel() * 32 != numel:
            raise ShapeError(f"{name}: expected {numel // 32} packed int32 keep words")
        return "_kb", _contig(t, name)
    return "", _u8(t, numel, name)


def _u8(t, numel, name):
    if t is None:
        return None
    if t.dtype not in (torch.uint8, torch.bool) or t.numel() != numel:
        raise ShapeError(f"{name}: expected a u8 keep mask with {numel} elements")
    return _contig(t, name)


class _Workspace:
    """Grow-only scratch buffer per (device, stream); stream-ordered reuse.

    A superseded (smaller) buffer is never freed: a CUDA graph captured
    earlier may have baked its address in and still write it on replay, and
    torch hands out side streams from a small pool, so two users can share a
    key.  The retired buffers are kept alive for the process lifetime (they
    only ever grow geometrically, so the total is bounded by ~2x the largest)."""

    def __init__(self):
        self.bufs = {}
        self.retired = []

    def get(self, nbytes: int) -> torch.Tensor:
        key = (torch.cuda.current_device(), torch.cuda.current_stream().cuda_stream)
        buf = self.bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            if buf is not None:
                self.retired.append(buf)
            size = max(nbytes, 1 << 20, 0 if buf is None else 2 * buf.numel())
            buf = torch.empty(size, dtype=torch.uint8, device="cuda")
            self.bufs[key] = buf
        return buf


WORKSPACE = _Workspace()


# ---------------------------------------------------------------------------
# optional per-call CUDA-event timing (bench.py roofline accounting)


class KernelTimer:
    """Records a CUDA event pair around every library call made while active,
    on the stream the call launches on, together with the call's algorithmic
    work: ``("hbm", bytes)`` for row kernels or ``("tensor"|"simt", flops)``
    for contractions.

    Works eagerly and under CUDA-graph capture (events are created with
    ``external=True`` so they become event-record nodes of the graph): call
    ``collect()`` after each synchronized replay to accumulate durations."""

    def __init__(self):
        self.records = []
        self.totals = {}

    def __enter__(self):
        global _TIMER
        _TIMER = self
        return self

    def __exit__(self, *exc):
        global _TIMER
        _TIMER = None

    def collect(self):
        torch.cuda.synchronize()
        for label, kind, work, nbytes, e0, e1 in self.records:
            a = self.totals.setdefault(label, {"label": label, "kind": kind, "calls": 0, "ms": 0.0,
                                               "work": 0.0, "bytes": 0.0})
            a["calls"] += 1
            a["ms"] += e0.elapsed_time(e1)
            a["work"] += work
            a["bytes"] += nbytes if nbytes is not None else (work if kind == "hbm" else 0.0)

    def reset_records(self):
        self.records = []

    def summary(self):
        if not self.totals:
            self.collect()
        return sorted(self.totals.values(), key=lambda r: -r["ms"])


_TIMER = None


class _Span:
    __slots__ = ("label", "kind", "work", "nbytes", "e0")

    def __init__(self, label, kind, work, nbytes=None):
        self.label, self.kind, self.work, self.nbytes = label, kind, work, nbytes

    def __enter__(self):
        self.e0 = torch.cuda.Event(enable_timing=True, external=True)
        self.e0.record()

    def __exit__(self, *exc):
        e1 = torch.cuda.Event(enable_timing=True, external=True)
        e1.record()
        if _TIMER is not None:
            _TIMER.records.append((self.label, self.kind, self.work, self.nbytes, self.e0, e1))


class _Null:
    def __enter__(self):
        return None

    def __exit__(self, *exc):
        return False


_NULL = _Null()
_LABEL = [None]


_LABEL_NEST = False  # profiling tools: "outer/inner" call-site labels


def _span(default_label, kind, work_fn, bytes_fn=None):
    """``work_fn``: algorithmic bytes (kind "hbm") or flops (contractions);
    ``bytes_fn`` (contractions): compulsory operand bytes, so a contraction
    whose arithmetic intensity is below the ridge point is judged against HBM."""
    if _TIMER is None:
        return _NULL
    nb = bytes_fn() if bytes_fn is not None else None
    if _LABEL_NEST and _LABEL[0]:
        return _Span(f"{_LABEL[0]}/{default_label}", kind, work_fn(), nb)
    return _Span(_LABEL[0] or default_label, kind, work_fn(), nb)


class label:
    """Context manager naming the calls made inside it (per-call-site rows)."""

    def __init__(self, name):
        self.name = name

    def __enter__(self):
        self.prev = _LABEL[0]
        _LABEL[0] = f"{self.prev}/{self.name}" if (_LABEL_NEST and self.prev) else self.name

    def __exit__(self, *exc):
        _LABEL[0] = self.prev


# ---------------------------------------------------------------------------
# bias + dropout + residual + LayerNorm


def bdrln_fwd(h, bias, keep, keep_scale, residual, gamma, beta, eps, y=None, s=None, mean=None,
              rstd=None):
    _contig(h, "h")
    cols = h.shape[-1]
    rows = h.numel() // cols
    y = torch.empty_like(h) if y is None else y
    if residual is not None and (residual.shape != h.shape or residual.dtype != h.dtype):
        raise ShapeError("bdrln: residual must match h")
    esz = h.element_size()
    sfx, keep = _keep_arg(keep, h.numel(), "keep")
    kbytes = 0 if keep is None else (1 if sfx == "" else 0.125)
    work = lambda: rows * cols * (esz * (2 + (residual is not None) + (s is not None))  # noqa: E731
                                  + kbytes) + rows * 8 * (mean is not None) + 3 * cols * 4
    with _span("bdrln_fwd", "hbm", work):
        _lib.call("dfx_bdrln_fwd" + sfx, dfx_dtype(h), rows, cols, h.data_ptr(), _ptr(_vec(bias, cols, "bias")),
                  _ptr(keep), float(keep_scale),
                  _ptr(None if residual is None else _contig(residual, "residual")),
                  _ptr(_vec(gamma, cols, "gamma")), _ptr(_vec(beta, cols, "beta")), float(eps),
                  _contig(y, "y").data_ptr(), _ptr(s), _ptr(mean), _ptr(rstd), _stream())
    return y


def bdrln_bwd(dy, s, gamma, keep, keep_scale, eps, ds=None, dh=None, dgamma=None, dbeta=None,
              dbias=None, ws=None):
    """``ws``: an explicit workspace (>= dfx_bdrln_bwd_workspace bytes) whose
    partial sums bdrln_bwd_finalize reduces later (dgamma/dbeta/dbias None)."""
    _contig(dy, "dy")
    cols = dy.shape[-1]
    rows = dy.numel() // cols
    if s.shape != dy.shape or s.dtype != dy.dtype:
        raise ShapeError("bdrln_bwd: stash must match dy")
    ws_n = _lib.load().dfx_bdrln_bwd_workspace(rows, cols)
    if ws is None:
        ws = WORKSPACE.get(ws_n)
    elif ws.numel() < ws_n:
        raise ShapeError("bdrln_bwd: workspace too small")
    esz = dy.element_size()
    sfx, keep = _keep_arg(keep, dy.numel(), "keep")
    kbytes = 0 if keep is None else (1 if sfx == "" else 0.125)
    work = lambda: rows * cols * (esz * (2 + (ds is not None) + (dh is not None))  # noqa: E731
                                  + kbytes) + 4 * cols * 4
    with _span("bdrln_bwd", "hbm", work):
        _lib.call("dfx_bdrln_bwd" + sfx, dfx_dtype(dy), rows, cols, dy.data_ptr(), _contig(s, "s").data_ptr(),
                  _vec(gamma, cols, "gamma").data_ptr(), _ptr(keep),
                  float(keep_scale), float(eps), _ptr(ds), _ptr(dh), _ptr(dgamma), _ptr(dbeta),
                  _ptr(dbias), ws.data_ptr(), ws.numel(), _stream())


def bdrln_bwd_finalize(dy_like, ws, dgamma, dbeta, dbias):
    """dgamma / dbeta / dbias from the partial sums a bdrln_bwd(..., ws=ws) left."""
    cols = dy_like.shape[-1]
    rows = dy_like.numel() // cols
    with _span("bdrln_bwd_finalize", "hbm", lambda: 3 * cols * 4 * 256):
        _lib.call("dfx_bdrln_bwd_finalize", dfx_dtype(dy_like), rows, cols, ws.data_ptr(), ws.numel(),
                  _ptr(dgamma), _ptr(dbeta), _ptr(dbias), _stream())


# ---------------------------------------------------------------------------
# scaled + masked softmax + dropout


def softmax_fwd(scores, inv_divisor, add_mask, keep, keep_scale, p=None, pd=None):
    """scores [B, NH, Q, K]; add_mask f32 [B, K] (or None)."""
    _contig(scores, "scores")
    if scores.dim() != 4:
        raise ShapeError("softmax_fwd: scores must be [B, NH, Q, K]")
    B, NH, Q, K = scores.shape
    if add_mask is not None:
        if add_mask.dtype != torch.float32 or add_mask.numel() != B * K:
            raise ShapeError("softmax_fwd: add_mask must be f32 with B*K elements")
        _contig(add_mask, "add_mask")
    n, esz = scores.numel(), scores.element_size()
    work = lambda: n * (esz * (1 + (p is not None) + (pd is not None)) + (keep is not None)) + B * K * 4  # noqa: E731
    with _span("softmax_fwd", "hbm", work):
        _lib.call("dfx_softmax_fwd", dfx_dtype(scores), B, NH, Q, K, scores.data_ptr(), float(inv_divisor),
                  _ptr(add_mask), _ptr(_u8(keep, scores.numel(), "keep")), float(keep_scale), _ptr(p),
                  _ptr(pd), _stream())
    return p, pd


def softmax_bwd(dpd, p, keep, keep_scale, inv_divisor, out=None):
    _contig(dpd, "dpd")
    _contig(p, "p")
    K = dpd.shape[-1]
    out = torch.empty_like(dpd) if out is None else out
    work = lambda: dpd.numel() * (3 * dpd.element_size() + (keep is not None))  # noqa: E731
    with _span("softmax_bwd", "hbm", work):
        _lib.call("dfx_softmax_bwd", dfx_dtype(dpd), dpd.numel() // K, K, dpd.data_ptr(), p.data_ptr(),
                  _ptr(_u8(keep, dpd.numel(), "keep")), float(keep_scale), float(inv_divisor),
                  out.data_ptr(), _stream())
    return out


# ---------------------------------------------------------------------------
# fused attention (QKᵀ -> scale + mask -> softmax -> dropout -> PV)


def pack_keep_bits(keep):
    """u8/bool keep flags [..., S] -> int32 [..., S/32], bit i of word w = keep[32w + i]
    (the packed layout dfx_attn_fwd / dfx_attn_bwd read)."""
    *lead, S = keep.shape
    if S % 32:
        raise ShapeError("pack_keep_bits: last dim must be a multiple of 32")
    k = keep.reshape(*lead, S // 32, 32).to(torch.int64)
    w = (k << torch.arange(32, device=keep.device, dtype=torch.int64)).sum(-1)
    return torch.where(w >= 2 ** 31, w - 2 ** 32, w).to(torch.int32)


def attn_fwd(qkv, B, S, heads, add_mask, keep, keep_scale, inv_divisor, ctx, lse, kbits_row=None,
             kbits_col=None):
    """qkv bf16 [B*S, >=3H] (Q|K|V blocks); ctx bf16 [B*S, >=H]; lse f32 [B, NH, S];
    keep u8 [B, NH, S, S] or None; kbits_* int32 [B, NH, S, S/32] (packed keep flags).
    keep None with kbits_row given: the flags arrive packed in kbits_row (input)."""
    if qkv.dtype != torch.bfloat16 or ctx.dtype != torch.bfloat16:
        raise ShapeError("attn_fwd: qkv and ctx must be bfloat16")
    if qkv.stride(1) != 1 or ctx.stride(1) != 1:
        raise ShapeError("attn_fwd: qkv/ctx rows must be contiguous")
    if add_mask is not None and (add_mask.dtype != torch.float32 or add_mask.numel() != B * S):
        raise ShapeError("attn_fwd: add_mask must be f32 with B*S elements")
    flops = 4.0 * B * heads * S * S * 64
    with _span("attn_fwd", "tensor", lambda: flops):
        _lib.call("dfx_attn_fwd", B, heads, S, 64, qkv.data_ptr(), qkv.stride(0), _ptr(add_mask),
                  _ptr(None if keep is None else _u8(keep, B * heads * S * S, "keep")), float(keep_scale),
                  float(inv_divisor), ctx.data_ptr(), ctx.stride(0), lse.data_ptr(), _ptr(kbits_row),
                  _ptr(kbits_col), _stream())
    return ctx


def attn_bwd_workspace(B, S, heads):
    """A dedicated workspace for attn_bwd whose qkv-bias partial sums
    attn_bwd_bias_grad reduces later (possibly on another stream)."""
    return torch.empty(_lib.load().dfx_attn_bwd_workspace(B, heads, S), dtype=torch.uint8, device="cuda")


def attn_bwd(qkv, ctx, dctx, B, S, heads, add_mask, lse, kbits_row, kbits_col, keep_scale, inv_divisor, dqkv,
             ws=None):
    """Writes dQ | dK | dV into dqkv (bf16 [B*S, >=3H]); ``ws`` (attn_bwd_workspace)
    keeps the per-strip qkv-bias column sums for attn_bwd_bias_grad."""
    for t, nm in ((qkv, "qkv"), (ctx, "ctx"), (dctx, "dctx"), (dqkv, "dqkv")):
        if t.dtype != torch.bfloat16 or t.stride(1) != 1:
            raise ShapeError(f"attn_bwd: {nm} must be bfloat16 with contiguous rows")
    if ctx.stride(0) != dctx.stride(0):
        raise ShapeError("attn_bwd: ctx and dctx must share a row stride")
    need = _lib.load().dfx_attn_bwd_workspace(B, heads, S)
    if ws is None:
        ws = WORKSPACE.get(need)
    elif ws.numel() < need:
        raise ShapeError("attn_bwd: workspace too small")
    flops = 8.0 * B * heads * S * S * 64  # algorithmic: dPd, dV, dQ, dK (the S recomputes are extra)
    with _span("attn_bwd", "tensor", lambda: flops):
        _lib.call("dfx_attn_bwd", B, heads, S, 64, qkv.data_ptr(), qkv.stride(0), ctx.data_ptr(), dctx.data_ptr(),
                  ctx.stride(0), _ptr(add_mask), lse.data_ptr(), _ptr(kbits_row), _ptr(kbits_col),
                  float(keep_scale), float(inv_divisor), dqkv.data_ptr(), dqkv.stride(0), ws.data_ptr(),
                  ws.numel(), _stream())
    return dqkv


def attn_bwd_bias_grad(B, S, heads, ws, dbias, accumulate=False):
    """dbias [3*heads*64] (+)= column sums of the dQ | dK | dV an attn_bwd(..., ws=ws) produced."""
    _vec(dbias, 3 * heads * 64, "dbias")
    with _span("attn_bwd_bias_grad", "hbm", lambda: B * (S // 128) * 3 * heads * 64 * 4):
        _lib.call("dfx_attn_bwd_bias_grad", B, heads, S, ws.data_ptr(), ws.numel(), dbias.data_ptr(),
                  int(bool(accumulate)), _stream())
    return dbias


# ---------------------------------------------------------------------------
# bias + GELU, column sums


def bias_gelu_fwd(f, bias, pre=None, y=None):
    _contig(f, "f")
    cols = f.shape[-1]
    y = torch.empty_like(f) if y is None else y
    work = lambda: f.numel() * f.element_size() * (2 + (pre is not None))  # noqa: E731
    with _span("bias_gelu_fwd", "hbm", work):
        _lib.call("dfx_bias_gelu_fwd", dfx_dtype(f), f.numel() // cols, cols, f.data_ptr(),
                  _ptr(_vec(bias, cols, "bias")), _ptr(pre), y.data_ptr(), _stream())
    return y


def bias_gelu_bwd(dy, pre, dpre=None, dbias=None):
    _contig(dy, "dy")
    cols = dy.shape[-1]
    rows = dy.numel() // cols
    dpre = torch.empty_like(dy) if dpre is None else dpre
    ws = WORKSPACE.get(_lib.load().dfx_colsum_workspace(rows, cols))
    work = lambda: dy.numel() * dy.element_size() * (3 + (dbias is not None))  # noqa: E731
    with _span("bias_gelu_bwd", "hbm", work):
        _lib.call("dfx_bias_gelu_bwd", dfx_dtype(dy), rows, cols, dy.data_ptr(), _contig(pre, "pre").data_ptr(),
                  dpre.data_ptr(), _ptr(dbias), ws.data_ptr(), ws.numel(), _stream())
    return dpre


def colsum(x2d, out, accumulate=False):
    """out[c] (+)= sum_r x2d[r, c]; x2d may have a row stride."""
    if x2d.dim() != 2 or x2d.stride(1) != 1:
        raise ShapeError("colsum: x must be a 2-D row-major view")
    rows, cols = x2d.shape
    ws = WORKSPACE.get(_lib.load().dfx_colsum_workspace(rows, cols))
    with _span("colsum", "hbm", lambda: rows * cols * x2d.element_size() + cols * 4):
        _lib.call("dfx_colsum", dfx_dtype(x2d), rows, cols, x2d.data_ptr(), x2d.stride(0), out.data_ptr(),
                  int(accumulate), ws.data_ptr(), ws.numel(), _stream())
    return out


# ---------------------------------------------------------------------------
# contractions


def _bstr(t, nb):
    """(count1, stride1, count2, stride2) of up to two leading batch dims."""
    lead = t.shape[:-2]
    if len(lead) > 2:
        raise ShapeError("gemm: at most two batch dimensions")
    shp = list(lead) + [1] * (2 - len(lead))
    st = list(t.stride()[:-2]) + [0] * (2 - len(lead))
    return shp[0], st[0], shp[1], st[1]


def gemm_args(a, b, d, epilogue=_lib.EPI_NONE, alpha=1.0, beta=1.0, bias=None, aux=None,
              aux_out=None, force_simt=False) -> GemmArgs:
    """D[..., m, n] = epi(alpha * A[..., m, k] @ B[..., n, k]^T) on tensor VIEWS.

    Any view works as long as each of A and B has a unit stride along one of
    its two trailing dims (transposed operands need no copy)."""
    if a.dim() != b.dim() or a.dim() != d.dim() or a.dim() < 2:
        raise ShapeError("gemm: A, B, D must have the same rank >= 2")
    m, k = a.shape[-2:]
    n, k2 = b.shape[-2:]
    if k != k2 or tuple(d.shape[-2:]) != (m, n):
        raise ShapeError(f"gemm: shapes {tuple(a.shape)} x {tuple(b.shape)} -> {tuple(d.shape)}")
    if a.shape[:-2] != b.shape[:-2] or a.shape[:-2] != d.shape[:-2]:
        raise ShapeError("gemm: batch dims differ")
    if d.stride(-1) != 1:
        raise ShapeError("gemm: D must be contiguous along n")
    if a.dtype != b.dtype:
        raise ShapeError("gemm: A and B dtypes differ")
    g = GemmArgs()
    g.in_dtype, g.out_dtype, g.epilogue, g.force_simt = dfx_dtype(a), dfx_dtype(d), int(epilogue), int(force_simt)
    g.m, g.n, g.k = m, n, k
    b1, sa1, b2, sa2 = _bstr(a, 0)
    _, sb1, _, sb2 = _bstr(b, 0)
    _, sd1, _, sd2 = _bstr(d, 0)
    g.batch1, g.batch2 = b1, b2
    g.a, g.a_stride_m, g.a_stride_k, g.a_stride_b1, g.a_stride_b2 = a.data_ptr(), a.stride(-2), a.stride(-1), sa1, sa2
    g.b, g.b_stride_n, g.b_stride_k, g.b_stride_b1, g.b_stride_b2 = b.data_ptr(), b.stride(-2), b.stride(-1), sb1, sb2
    g.d, g.d_stride_m, g.d_stride_b1, g.d_stride_b2 = d.data_ptr(), d.stride(-2), sd1, sd2
    g.alpha, g.beta = float(alpha), float(beta)
    if bias is not None:
        g.bias = _vec(bias, n, "bias").data_ptr()
    for name, t in (("aux", aux), ("aux_out", aux_out)):
        if t is None:
            continue
        if tuple(t.shape) != tuple(d.shape) or t.dtype != d.dtype or t.stride(-1) != 1:
            raise ShapeError(f"gemm: {name} must match D")
        _, s1, _, s2 = _bstr(t, 0)
        setattr(g, name, t.data_ptr())
        setattr(g, name + "_stride_m", t.stride(-2))
        setattr(g, name + "_stride_b1", s1)
        setattr(g, name + "_stride_b2", s2)
    return g


def gemm(a, b, d, epilogue=_lib.EPI_NONE, alpha=1.0, beta=1.0, bias=None, aux=None, aux_out=None,
         force_simt=False):
    g = gemm_args(a, b, d, epilogue, alpha, beta, bias, aux, aux_out, force_simt)
    lib = _lib.load()
    need = lib.dfx_gemm_workspace(g)
    if need:
        ws = WORKSPACE.get(need)
        g.workspace, g.workspace_bytes = ws.data_ptr(), ws.numel()
    if _TIMER is None:
        _lib.check(lib.dfx_gemm(g, _stream()), "dfx_gemm")
        return d
    kind = "tensor" if lib.dfx_gemm_uses_tensor_cores(g) else "simt"

    def nbytes():  # A, B read once, D written once (+ the aux operand read)
        z = g.batch1 * g.batch2
        return z * (g.m * g.k * a.element_size() + g.n * g.k * b.element_size()
                    + g.m * g.n * d.element_size() * (1 + (aux is not None) + (aux_out is not None)))

    with _span("gemm", kind, lambda: 2.0 * g.m * g.n * g.k * g.batch1 * g.batch2, nbytes):
        _lib.check(lib.dfx_gemm(g, _stream()), "dfx_gemm")
    return d


def gemm_excite(z, hw, mean, rstd, gamma, beta, gate, w, d, y_out=None):
    """d [M, N] = y · wᵀ with y = swish(BN(z)) * gate[row // hw] formed inside
    the tcgen05 GEMM from z [M, K] (the MBConv SE excite folded into the
    project 1x1 conv, dfx_gemm_excite); y_out [M, K] receives y when given."""
    for t, nm in ((z, "z"), (w, "w"), (d, "d")):
        if t.dtype != torch.bfloat16 or t.dim() != 2 or not t.is_contiguous():
            raise ShapeError(f"gemm_excite: {nm} must be a contiguous 2-D bfloat16 tensor")
    M, Kc = z.shape
    N = w.shape[0]
    if w.shape[1] != Kc or d.shape != (M, N):
        raise ShapeError("gemm_excite: shape mismatch")
    if y_out is not None and (y_out.shape != z.shape or y_out.dtype != torch.bfloat16 or not y_out.is_contiguous()):
        raise ShapeError("gemm_excite: y_out must match z")
    for t, nm in ((mean, "mean"), (rstd, "rstd"), (gamma, "gamma"), (beta, "beta")):
        _vec(t, Kc, nm)
    if gate.dtype != torch.float32 or gate.dim() != 2 or gate.shape[1] != Kc or gate.shape[0] * hw < M:
        raise ShapeError("gemm_excite: gate must be f32 [images, K] covering every row")
    esz = 2

    def nbytes():  # z and w read once, d written once (+ y written)
        return M * Kc * esz + N * Kc * esz + M * N * esz + (M * Kc * esz if y_out is not None else 0)

    with _span("gemm_excite", "tensor", lambda: 2.0 * M * N * Kc, nbytes):
        _lib.call("dfx_gemm_excite", M, Kc, N, z.data_ptr(), hw, mean.data_ptr(), rstd.data_ptr(), gamma.data_ptr(),
                  beta.data_ptr(), _contig(gate, "gate").data_ptr(), w.data_ptr(), d.data_ptr(), _ptr(y_out),
                  _stream())
    return d


def gemm_uses_tensor_cores(a, b, d, **kw) -> bool:
    return bool(_lib.load().dfx_gemm_uses_tensor_cores(gemm_args(a, b, d, **kw)))


# ---------------------------------------------------------------------------
# optimizer


def sgd_update(master, grad, lr, bf16_copy=None):
    if master.dtype != torch.float32 or grad.dtype != torch.float32 or master.numel() != grad.numel():
        raise ShapeError("sgd_update: master and grad must be f32 of equal size")
    work = lambda: master.numel() * (12 + (2 if bf16_copy is not None else 0))  # noqa: E731
    with _span("sgd_update", "hbm", work):
        _lib.call("dfx_sgd_update", master.numel(), master.data_ptr(), grad.data_ptr(), float(lr),
                  _ptr(bf16_copy), _stream())


def scale_(x, s):
    _lib.call("dfx_scale_f32", x.numel(), x.data_ptr(), float(s), _stream())


def cast(src, dst):
    if src.numel() != dst.numel():
        raise ShapeError("cast: size mismatch")
    _lib.call("dfx_cast", src.numel(), dfx_dtype(src), src.data_ptr(), dfx_dtype(dst), dst.data_ptr(), _stream())
    return dst


def cast2(src0, dst0, src1, dst1):
    """dst0 = src0 and dst1 = src1 (equal sizes, dtype-converting) in one launch."""
    n = src0.numel()
    if src1.numel() != n or dst0.numel() != n or dst1.numel() != n:
        raise ShapeError("cast2: size mismatch")
    if src0.dtype != src1.dtype or dst0.dtype != dst1.dtype:
        raise ShapeError("cast2: both pairs must share dtypes")
    _lib.call("dfx_cast2", n, dfx_dtype(src0), src0.data_ptr(), src1.data_ptr(), dfx_dtype(dst0), dst0.data_ptr(),
              dst1.data_ptr(), _stream())


def launch_count() -> int:
    return int(_lib.load().dfx_launch_count())


def reset_launch_count() -> None:
    _lib.load().dfx_reset_launch_count()
