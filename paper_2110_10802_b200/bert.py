"""BERT encoder layer training step on the B200 hot path.

The layer is the one the reference expresses with registry operators
(golden graph in oracle/make_golden.py):

    QKV   = x @ Wqkvᵀ + bqkv                           Gemm (frontend.py:369-405)
    S     = Q Kᵀ (per batch, head)                     Einsum bsnd,btnd->bnst (408-481)
    P, Pd = softmax(S / sqrt(dh) + mask), P * drop     Div/Add/Softmax/Mul (294, 175-188, 493-501)
    ctx   = Pd V                                       Einsum bnst,btnd->bsnd
    ln1   = LN((ctx Woᵀ + bo) * drop1 + x)             Gemm/Add/Mul/Add/LayerNormalization (519-529)
    g     = gelu_tanh(ln1 W1ᵀ + b1)                    Gemm + Pow/Mul/Add/Tanh chain (223-295)
    out   = LN((g W2ᵀ + b2) * drop2 + ln1)

and its reverse pass follows the manual VJPs of autodiff.py (Gemm/Einsum
1363-1459, Softmax 1465-1484, LayerNormalization 1490-1545) and the symexpr
derivative of the GELU chain.  Every operation is one call into the sm_100a
library: 9 launches forward (5 tcgen05 GEMMs carrying bias / bias+GELU
epilogues, the fused softmax, two fused bias+dropout+residual+LN kernels) and
the mirrored backward.  Weights live in one flat f32 master arena (plus a bf16
copy of it for the tensor cores) and gradients in one flat f32 arena, so the
data-parallel allreduce and the SGD step each touch a single buffer.
"""

from __future__ import annotations

import contextlib
from dataclasses import dataclass

import torch

from . import _lib
from . import kernels as K
from ._lib import EPI_ADD, EPI_BIAS, EPI_BIAS_GELU, EPI_GELU_BWD
from .errors import ShapeError


@dataclass(frozen=True)
class BertLayerConfig:
    hidden: int = 768
    heads: int = 12
    ffn: int = 3072
    eps: float = 1e-12
    p_drop: float = 0.1
    dtype: torch.dtype = torch.bfloat16
    # bf16: QKᵀ -> softmax -> dropout -> PV as one tcgen05 kernel per direction
    # (csrc/attn.cu); False keeps the unfused GEMM + softmax-kernel chain
    fused_attention: bool = True

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads


def _model_specs(c: BertLayerConfig):
    H, F = c.hidden, c.ffn
    return [("wqkv", (3 * H, H)), ("wo", (H, H)), ("w1", (F, H)), ("w2", (H, F)),
            ("bqkv", (3 * H,)), ("bo", (H,)), ("g1", (H,)), ("be1", (H,)), ("b1", (F,)),
            ("b2", (H,)), ("g2", (H,)), ("be2", (H,))]


# Arena order = the order backward() finishes the gradients (LN2 / FFN2 group
# first, the QKV group last), so a bucketed data-parallel allreduce
# (dp.GradAllReducer) can reduce the front of the arena while the backward is
# still producing the rest.  GRAD_GROUP_ENDS close each group.
PRODUCTION_ORDER = ("g2", "be2", "b2", "w2", "b1", "w1", "g1", "be1", "bo", "wo", "wqkv", "bqkv")
GRAD_GROUP_ENDS = ("w2", "w1", "wo", "bqkv")


def _param_specs(c: BertLayerConfig):
    shapes = dict(_model_specs(c))
    return [(n, shapes[n]) for n in PRODUCTION_ORDER]


MATRICES = ("wqkv", "wo", "w1", "w2")


class FlatArena:
    """Named views into one contiguous buffer (parameters or gradients)."""

    def __init__(self, specs, dtype, device):
        self.offsets = {}
        off = 0
        for name, shape in specs:
            n = 1
            for d in shape:
                n *= d
            # keep every view 16-byte aligned for 128-bit / TMA access
            self.offsets[name] = (off, shape)
            off += (n + 7) // 8 * 8
        self.flat = torch.zeros(off, dtype=dtype, device=device)
        self.views = {name: self.flat[o:o + _numel(s)].view(s) for name, (o, s) in self.offsets.items()}

    def __getitem__(self, name):
        return self.views[name]


def _check_host(dev: dict, host: dict):
    """Host input buffers must already be in the device buffers' form: a u8
    mask copied into a packed int32 buffer would be converted, not packed."""
    for k, d in dev.items():
        h = host[k]
        if h.dtype != d.dtype or h.shape != d.shape:
            hint = " (pack keep flags with kernels.pack_keep_bits)" if d.dtype == torch.int32 else ""
            raise ShapeError(f"host input {k}: expected {d.dtype} {tuple(d.shape)}, got {h.dtype} {tuple(h.shape)}{hint}")


def _numel(shape):
    n = 1
    for d in shape:
        n *= d
    return n


class BertEncoderLayer:
    def __init__(self, cfg: BertLayerConfig = BertLayerConfig(), device="cuda", seed: int = 0):
        if cfg.dtype not in (torch.float32, torch.bfloat16):
            raise ShapeError("BertEncoderLayer: dtype must be float32 or bfloat16")
        if cfg.hidden % cfg.heads:
            raise ShapeError("hidden must be divisible by heads")
        _lib.load(check_device=True)
        self.cfg = cfg
        self.device = torch.device(device)
        specs = _param_specs(cfg)
        self.master = FlatArena(specs, torch.float32, self.device)
        self.grad = FlatArena(specs, torch.float32, self.device)
        self.wlow = FlatArena(specs, torch.bfloat16, self.device) if cfg.dtype == torch.bfloat16 else None
        self._bufs = {}
        self.slot = 0  # activation / input buffer set (see train_step_host_async)
        # three sets: step i+3's H2D may start once step i's dx has left
        # (D2H), i.e. with two compute periods of slack (two sets stalled
        # every step on H2D(i+2) waiting for D2H(i): tools/e2e_probe.py)
        self.nslots = 3
        self.concurrent = True  # weight gradients on a forked stream (backward)
        self.reducer = None  # dp.GradAllReducer once attach_process_group() is called
        self.world = 1
        self._init_params(seed)

    def attach_process_group(self, group=None, bucket_bytes: int = 8 << 20):
        """Data-parallel replica: the backward all-reduces (SUM) the gradient
        arena bucket by bucket as each parameter group completes, and
        ``train_step`` / the captured step fold the 1/world average into the
        SGD learning rate.  Under NCCL the buckets are captured into the step's
        CUDA graph with everything else."""
        import torch.distributed as dist

        from .dp import GradAllReducer

        ends = [self.grad.offsets[n][0] + _numel(self.grad.offsets[n][1]) for n in GRAD_GROUP_ENDS]
        self.reducer = GradAllReducer(self.grad.flat, group, bucket_bytes, boundaries=ends)
        self.world = dist.get_world_size(group)
        return self.reducer

    # ------------------------------------------------------------ parameters
    def _init_params(self, seed):
        g = torch.Generator(device="cpu").manual_seed(seed)
        H = self.cfg.hidden
        vals = {}
        for name, shape in _model_specs(self.cfg):  # draw order fixed (independent of the arena order)
            if name.startswith("w"):
                vals[name] = 0.02 * torch.randn(shape, generator=g)
            elif name.startswith("g"):
                vals[name] = 1.0 + 0.1 * torch.randn(shape, generator=g)
            else:
                vals[name] = 0.1 * torch.randn(shape, generator=g)
        del H
        self.load_params(vals)

    def load_params(self, vals: dict):
        """Load weights given either fused ``wqkv``/``bqkv`` or the separate
        ``wq, wk, wv`` / ``bq, bk, bv`` of the reference graph."""
        v = {k: torch.as_tensor(x, dtype=torch.float32) for k, x in vals.items()}
        if "wq" in v:
            v["wqkv"] = torch.cat([v.pop("wq"), v.pop("wk"), v.pop("wv")], 0)
            v["bqkv"] = torch.cat([v.pop("bq"), v.pop("bk"), v.pop("bv")], 0)
        for name, _ in _param_specs(self.cfg):
            self.master[name].copy_(v[name].to(self.device))
        self.refresh_low_precision()

    def refresh_low_precision(self):
        if self.wlow is not None:
            K.cast(self.master.flat, self.wlow.flat)

    def weight(self, name):
        """Matrix operand as consumed by the GEMMs (bf16 copy or f32 master)."""
        return self.wlow[name] if self.wlow is not None else self.master[name]

    def params_numpy(self, split_qkv=True):
        out = {k: v.detach().cpu().numpy().astype("float64") for k, v in self.master.views.items()}
        if self.wlow is not None:  # the GEMMs see bf16-rounded matrices
            for k in MATRICES:
                out[k] = self.wlow[k].float().cpu().numpy().astype("float64")
        if split_qkv:
            H = self.cfg.hidden
            w, b = out.pop("wqkv"), out.pop("bqkv")
            for i, t in enumerate("qkv"):
                out["w" + t] = w[i * H:(i + 1) * H]
                out["b" + t] = b[i * H:(i + 1) * H]
        return out

    def grads_numpy(self, split_qkv=True):
        out = {k: v.detach().cpu().numpy().astype("float64") for k, v in self.grad.views.items()}
        if split_qkv:
            H = self.cfg.hidden
            w, b = out.pop("wqkv"), out.pop("bqkv")
            for i, t in enumerate("qkv"):
                out["w" + t] = w[i * H:(i + 1) * H]
                out["b" + t] = b[i * H:(i + 1) * H]
        return out

    @property
    def num_params(self) -> int:
        return sum(_numel(s) for _, s in _param_specs(self.cfg))

    # ------------------------------------------------------------ activations
    def buffers(self, B: int, S: int):
        # one activation set per pipeline slot (train_step_host_async rotates them)
        key = (B, S, self.slot)
        if key not in self._bufs:
            c = self.cfg
            T, H, F, NH = B * S, c.hidden, c.ffn, c.heads
            dt, dev = c.dtype, self.device
            e = lambda *s: torch.empty(s, dtype=dt, device=dev)  # noqa: E731
            self._bufs[key] = dict(
                qkv=e(T, 3 * H), scores=e(B, NH, S, S), p=e(B, NH, S, S), pd=e(B, NH, S, S),
                ctx=e(T, H), a1=e(T, H), s1=e(T, H), ln1=e(T, H), pre=e(T, F), g=e(T, F),
                a2=e(T, H), s2=e(T, H), out=e(T, H),
                ds2=e(T, H), da2=e(T, H), dpre=e(T, F), dln1=e(T, H), ds1=e(T, H), da1=e(T, H),
                dctx=e(T, H), dpd=e(B, NH, S, S), dsc=e(B, NH, S, S), dqkv=e(T, 3 * H), dx=e(T, H),
            )
            if self._fused(S):
                for nm in ("scores", "p", "pd", "dpd", "dsc"):
                    del self._bufs[key][nm]
                i32 = dict(dtype=torch.int32, device=dev)
                self._bufs[key].update(lse=torch.empty(B, NH, S, dtype=torch.float32, device=dev),
                                       kbits_row=torch.empty(B, NH, S, S // 32, **i32),
                                       kbits_col=torch.empty(B, NH, S, S // 32, **i32))
        return self._bufs[key]

    def _fused(self, S) -> bool:
        c = self.cfg
        return (c.fused_attention and c.dtype == torch.bfloat16 and c.head_dim == 64
                and S % 128 == 0 and S <= 512)

    def _heads(self, t, B, S, which):
        """[B, NH, S, dh] view of the Q/K/V (which=0/1/2) block of a [T, 3H] tensor."""
        c = self.cfg
        H, NH, dh = c.hidden, c.heads, c.head_dim
        return t.as_strided((B, NH, S, dh), (S * 3 * H, dh, 3 * H, 1), t.storage_offset() + which * H)

    def _ctx_heads(self, t, B, S):
        c = self.cfg
        return t.as_strided((B, c.heads, S, c.head_dim), (S * c.hidden, c.head_dim, c.hidden, 1),
                            t.storage_offset())

    # ------------------------------------------------------------ forward
    def forward(self, x, add_mask, keep_attn, keep1, keep2):
        """x [T, H] (T = B*S); add_mask f32 [B, S]; keep_* u8 dropout keep flags
        ([B, NH, S, S], [T, H], [T, H]); keep_attn may instead be the packed
        int32 [B, NH, S, S/32] form (kernels.pack_keep_bits, fused path only),
        keep1 / keep2 the packed int32 [T, H/32] form (any path).
        Returns the layer output [T, H]."""
        c = self.cfg
        B, S = add_mask.shape
        T = B * S
        if x.shape != (T, c.hidden) or x.dtype != c.dtype:
            raise ShapeError(f"x must be [{T}, {c.hidden}] {c.dtype}")
        ks = 1.0 / (1.0 - c.p_drop)
        b = self.buffers(B, S)
        P = self.master
        self._saved = (x, add_mask, keep_attn, keep1, keep2, B, S)
        packed = keep_attn.dtype == torch.int32
        if packed and not self._fused(S):
            raise ShapeError("packed keep_attn needs the fused (bf16) attention path")
        # the backward reads the row-major packed flags: the input itself when packed
        self._kb_row = keep_attn if packed else b.get("kbits_row")
        L = K.label
        with L("fwd.qkv_gemm+bias"):
            K.gemm(x, self.weight("wqkv"), b["qkv"], EPI_BIAS, bias=P["bqkv"])
        if self._fused(S):
            with L("fwd.attention"):
                K.attn_fwd(b["qkv"], B, S, c.heads, add_mask, None if packed else keep_attn, ks,
                           1.0 / (c.head_dim ** 0.5), b["ctx"], b["lse"], self._kb_row, b["kbits_col"])
        else:
            q, k, v = (self._heads(b["qkv"], B, S, i) for i in range(3))
            with L("fwd.scores_gemm"):
                K.gemm(q, k, b["scores"])
            with L("fwd.softmax"):
                K.softmax_fwd(b["scores"], 1.0 / (c.head_dim ** 0.5), add_mask, keep_attn, ks, b["p"], b["pd"])
            with L("fwd.ctx_gemm"):
                K.gemm(b["pd"], v.transpose(-1, -2), self._ctx_heads(b["ctx"], B, S))
        with L("fwd.out_gemm"):
            K.gemm(b["ctx"], self.weight("wo"), b["a1"])
        with L("fwd.bdrln1"):
            K.bdrln_fwd(b["a1"], P["bo"], keep1, ks, x, P["g1"], P["be1"], c.eps, y=b["ln1"], s=b["s1"])
        with L("fwd.ffn1_gemm+bias+gelu"):
            K.gemm(b["ln1"], self.weight("w1"), b["g"], EPI_BIAS_GELU, bias=P["b1"], aux_out=b["pre"])
        with L("fwd.ffn2_gemm"):
            K.gemm(b["g"], self.weight("w2"), b["a2"])
        with L("fwd.bdrln2"):
            K.bdrln_fwd(b["a2"], P["b2"], keep2, ks, b["ln1"], P["g2"], P["be2"], c.eps, y=b["out"], s=b["s2"])
        return b["out"]

    # ------------------------------------------------------------ backward
    def backward(self, dout):
        """Gradients of <dout, out> w.r.t. x (returned) and every parameter
        (written into ``self.grad``)."""
        c = self.cfg
        x, add_mask, keep_attn, keep1, keep2, B, S = self._saved
        ks = 1.0 / (1.0 - c.p_drop)
        b = self.buffers(B, S)
        P, G = self.master, self.grad
        L = K.label
        # Weight-gradient GEMMs and bias column sums do not feed the dgrad
        # chain: they run on a second stream (forked after their inputs exist,
        # joined before returning), so their CTAs fill the wave-quantisation
        # tails of the dgrad GEMMs and the attention kernels.  The CUDA graph
        # captures the fork/join as parallel branches.
        main = torch.cuda.current_stream(self.device)
        if not hasattr(self, "_side"):
            self._side = torch.cuda.Stream(device=self.device)
        side = self._side

        def fork():
            if not self.concurrent:  # the per-kernel attribution twin runs one stream
                return contextlib.nullcontext()
            ev = torch.cuda.Event()
            ev.record(main)
            side.wait_event(ev)
            return torch.cuda.stream(side)

        def ready(name):  # gradient group complete: its allreduce bucket may start
            if self.reducer is not None:
                off, shape = G.offsets[name]
                self.reducer.mark_ready(off + _numel(shape), (main, side) if self.concurrent else (main,))

        # BDRLN backward: the dx half stays on the critical path; the
        # parameter-gradient finalize (partials in a per-site workspace) forks
        wsb = self._bdrln_ws(B, S)
        with L("bwd.bdrln2"):
            K.bdrln_bwd(dout, b["s2"], P["g2"], keep2, ks, c.eps, ds=b["ds2"], dh=b["da2"], ws=wsb[0])
        with fork():
            K.bdrln_bwd_finalize(dout, wsb[0], G["g2"], G["be2"], G["b2"])
            with L("bwd.ffn2_wgrad"):
                K.gemm(b["da2"].t(), b["g"].t(), G["w2"])
        ready("w2")
        # FFN2: dgrad with the GELU-backward epilogue, wgrad straight into f32 grads
        with L("bwd.ffn2_dgrad+gelu_bwd"):
            K.gemm(b["da2"], self.weight("w2").t(), b["dpre"], EPI_GELU_BWD, aux=b["pre"])
        with fork():
            with L("bwd.ffn1_bias_grad"):
                K.colsum(b["dpre"], G["b1"])
            with L("bwd.ffn1_wgrad"):
                K.gemm(b["dpre"].t(), b["ln1"].t(), G["w1"])
        ready("w1")
        # FFN1: dgrad + residual gradient from LN2
        with L("bwd.ffn1_dgrad+residual"):
            K.gemm(b["dpre"], self.weight("w1").t(), b["dln1"], EPI_ADD, aux=b["ds2"])
        with L("bwd.bdrln1"):
            K.bdrln_bwd(b["dln1"], b["s1"], P["g1"], keep1, ks, c.eps, ds=b["ds1"], dh=b["da1"], ws=wsb[1])
        with fork():
            K.bdrln_bwd_finalize(b["dln1"], wsb[1], G["g1"], G["be1"], G["bo"])
            with L("bwd.out_wgrad"):
                K.gemm(b["da1"].t(), b["ctx"].t(), G["wo"])
        ready("wo")
        with L("bwd.out_dgrad"):
            K.gemm(b["da1"], self.weight("wo").t(), b["dctx"])
        # attention
        if self._fused(S):
            with L("bwd.attention"):
                K.attn_bwd(b["qkv"], b["ctx"], b["dctx"], B, S, c.heads, add_mask, b["lse"], self._kb_row,
                           b["kbits_col"], ks, 1.0 / (c.head_dim ** 0.5), b["dqkv"], ws=self._attn_ws(B, S))
        else:
            self._attn_bwd_unfused(b, B, S, keep_attn, ks)
        with fork():
            if not self._fused(S):
                with L("bwd.qkv_bias_grad"):
                    K.colsum(b["dqkv"], G["bqkv"])
            with L("bwd.qkv_wgrad"):
                K.gemm(b["dqkv"].t(), x.t(), G["wqkv"])
        with L("bwd.qkv_dgrad+residual"):
            K.gemm(b["dqkv"], self.weight("wqkv").t(), b["dx"], EPI_ADD, aux=b["ds1"])
        if self._fused(S):
            # the attention backward left per-strip column sums: the tiny reduce
            # rides the main stream after the dgrad (shorter than the forked
            # weight-gradient GEMM), keeping it off the step's tail
            with L("bwd.qkv_bias_grad"):
                K.attn_bwd_bias_grad(B, S, c.heads, self._attn_ws(B, S), G["bqkv"])
        if self.concurrent:
            main.wait_stream(side)  # join: every gradient is complete on the caller's stream
        return b["dx"]

    def _attn_ws(self, B, S):
        """Persistent attention-backward workspace (delta and the qkv-bias
        partial sums the side stream reduces)."""
        key = ("attn_ws", B, S)
        if key not in self._bufs:
            self._bufs[key] = K.attn_bwd_workspace(B, S, self.cfg.heads)
        return self._bufs[key]

    def _bdrln_ws(self, B, S):
        """Two persistent BDRLN-backward workspaces (one per call site): their
        partial sums are reduced on the side stream while the main stream runs on."""
        key = ("bdrln_ws", B, S, self.slot)
        if key not in self._bufs:
            n = _lib.load().dfx_bdrln_bwd_workspace(B * S, self.cfg.hidden)
            self._bufs[key] = [torch.empty(n, dtype=torch.uint8, device=self.device) for _ in range(2)]
        return self._bufs[key]

    def _attn_bwd_unfused(self, b, B, S, keep_attn, ks):
        c, L = self.cfg, K.label
        q, k, v = (self._heads(b["qkv"], B, S, i) for i in range(3))
        dq, dk, dv = (self._heads(b["dqkv"], B, S, i) for i in range(3))
        dctx = self._ctx_heads(b["dctx"], B, S)
        with L("bwd.dprobs_gemm"):
            K.gemm(dctx, v, b["dpd"])
        with L("bwd.dv_gemm"):
            K.gemm(b["pd"].transpose(-1, -2), dctx.transpose(-1, -2), dv)
        with L("bwd.softmax"):
            K.softmax_bwd(b["dpd"], b["p"], keep_attn, ks, 1.0 / (c.head_dim ** 0.5), out=b["dsc"])
        with L("bwd.dq_gemm"):
            K.gemm(b["dsc"], k.transpose(-1, -2), dq)
        with L("bwd.dk_gemm"):
            K.gemm(b["dsc"].transpose(-1, -2), q.transpose(-1, -2), dk)

    def sgd_step(self, lr: float):
        with K.label("sgd_update"):
            K.sgd_update(self.master.flat, self.grad.flat, lr,
                         None if self.wlow is None else self.wlow.flat)

    def reduce_gradients(self):
        """Data parallel: finish the bucketed allreduce the backward started
        (no-op for a single replica).  Returns the world size."""
        return self.reducer.finish() if self.reducer is not None else 1

    def train_step(self, x, add_mask, keep_attn, keep1, keep2, dout, lr=None):
        """fwd + bwd (+ gradient allreduce over the attached process group)
        (+ SGD with the gradient averaged over the replicas)."""
        out = self.forward(x, add_mask, keep_attn, keep1, keep2)
        dx = self.backward(dout)
        world = self.reduce_gradients()
        if lr is not None:
            self.sgd_step(lr / world)
        return out, dx

    # ------------------------------------------------------------ host-buffer API
    def step_bytes(self, B: int, S: int) -> int:
        """Compulsory HBM bytes of one fused training step (fused attention,
        SGD included): every kernel's tensor arguments read once and written
        once — the schedule's own data movement, compared in bench.py with the
        reference's ``ir.movement_volume`` of the unfused graph."""
        return fused_step_bytes(self.cfg, B, S)

    def step_flops(self, B: int, S: int) -> int:
        return fused_step_flops(self.cfg, B, S)

    def host_inputs_bytes(self, B: int, S: int) -> tuple[int, int]:
        """(H2D, D2H) bytes per train_step_host call."""
        c = self.cfg
        T, H = B * S, c.hidden
        esz = torch.tensor([], dtype=c.dtype).element_size()
        # counted from the device input buffers every step copies into
        h2d = sum(t.numel() * t.element_size() for t in self._dev_inputs(B, S).values())
        return h2d, T * H * esz

    def train_step_host(self, host: dict, lr=None, dx_host=None, graph=True):
        """One training step from HOST buffers: copies x, dout, the additive
        mask and the dropout keep masks to the device (pinned memory,
        stream-ordered), runs forward + backward (+ SGD when ``lr`` is given)
        as one CUDA-graph replay and copies dx back into ``dx_host``.  This
        is the call the e2e benchmark times: the reference's
        ``interp.execute`` likewise takes host arrays (interp.py:1301-1317)."""
        B, S = host["add_mask"].shape
        dev = self._dev_inputs(B, S)
        _check_host(dev, host)
        for k in ("x", "add_mask", "keep_attn", "keep1", "keep2", "dout"):
            dev[k].copy_(host[k], non_blocking=True)
        if graph:
            key = ("graph", B, S, lr, self.slot)
            if key not in self._bufs:
                self._bufs[key] = self.capture_step(B, S, lr)
            self._bufs[key].replay()
            dx = self.buffers(B, S)["dx"]
        else:
            _, dx = self.train_step(dev["x"], dev["add_mask"], dev["keep_attn"], dev["keep1"], dev["keep2"],
                                    dev["dout"], lr)
        if dx_host is not None:
            dx_host.copy_(dx, non_blocking=True)
        return dx_host

    def _dev_inputs(self, B, S):
        key = ("in", B, S, self.slot)
        if key not in self._bufs:
            c = self.cfg
            T, H, NH, dev = B * S, c.hidden, c.heads, self.device
            u8 = torch.uint8
            packed = self._fused(S) and H % 32 == 0
            self._bufs[key] = dict(
                x=torch.empty(T, H, dtype=c.dtype, device=dev),
                dout=torch.empty(T, H, dtype=c.dtype, device=dev),
                add_mask=torch.empty(B, S, dtype=torch.float32, device=dev),
                # fused path: the attention keep flags travel packed (1 bit each)
                keep_attn=(torch.empty(B, NH, S, S // 32, dtype=torch.int32, device=dev) if self._fused(S)
                           else torch.empty(B, NH, S, S, dtype=u8, device=dev)),
                # the BDRLN keep flags travel packed as well (0.4 MB instead of 3.1 MB each)
                keep1=(torch.empty(T, H // 32, dtype=torch.int32, device=dev) if packed
                       else torch.empty(T, H, dtype=u8, device=dev)),
                keep2=(torch.empty(T, H // 32, dtype=torch.int32, device=dev) if packed
                       else torch.empty(T, H, dtype=u8, device=dev)))
        return self._bufs[key]

    # ------------------------------------------------------------ CUDA graphs
    def train_step_host_async(self, host: dict, lr=None, dx_host=None):
        """Pipelined form of ``train_step_host``: ``nslots`` device input /
        activation sets rotate, so step i+1's H2D copy (its own stream) and step
        i's D2H of dx (another stream) overlap step i's CUDA-graph replay — the
        prefetching a data loader does.  Every step still copies its own inputs
        from pinned host memory and reads its own dx back; ``finish_host()``
        joins the copy streams into the compute stream."""
        B, S = host["add_mask"].shape
        if not hasattr(self, "_pipe"):
            self._pipe = {"h2d": torch.cuda.Stream(device=self.device), "d2h": torch.cuda.Stream(device=self.device),
                          "free": [None] * self.nslots}
        pp = self._pipe
        slot = self.slot
        comp = torch.cuda.current_stream(self.device)
        dev = self._dev_inputs(B, S)
        key = ("graph", B, S, lr, slot)
        if key not in self._bufs:
            torch.cuda.synchronize(self.device)
            self._bufs[key] = self.capture_step(B, S, lr)
        with torch.cuda.stream(pp["h2d"]):
            _check_host(dev, host)
            if pp["free"][slot] is not None:
                pp["h2d"].wait_event(pp["free"][slot])  # slot's previous step fully drained
            for k in ("x", "add_mask", "keep_attn", "keep1", "keep2", "dout"):
                dev[k].copy_(host[k], non_blocking=True)
            ev_in = torch.cuda.Event()
            ev_in.record(pp["h2d"])
        comp.wait_event(ev_in)
        self._bufs[key].replay()
        ev_done = torch.cuda.Event()
        ev_done.record(comp)
        with torch.cuda.stream(pp["d2h"]):
            pp["d2h"].wait_event(ev_done)
            if dx_host is not None:
                dx_host.copy_(self.buffers(B, S)["dx"], non_blocking=True)
            ev_free = torch.cuda.Event()
            ev_free.record(pp["d2h"])
        pp["free"][slot] = ev_free
        self.slot = (self.slot + 1) % self.nslots
        return dx_host

    def finish_host(self):
        """Make the current stream wait for every pipelined copy."""
        if hasattr(self, "_pipe"):
            comp = torch.cuda.current_stream(self.device)
            comp.wait_stream(self._pipe["h2d"])
            comp.wait_stream(self._pipe["d2h"])

    def capture_step(self, B: int, S: int, lr=None, timer=None):
        """Capture forward + backward (+ SGD) on the static device input
        buffers (``device_inputs``) into a CUDA graph; returns a
        ``CapturedStep`` whose ``replay()`` runs one training step."""
        from .graphs import CapturedStep

        dev = self._dev_inputs(B, S)

        def fn():  # fwd + bwd (+ bucketed NCCL allreduce when data parallel) (+ SGD)
            self.train_step(dev["x"], dev["add_mask"], dev["keep_attn"], dev["keep1"], dev["keep2"], dev["dout"], lr)

        keep = self.training_state()
        if timer is None:
            return CapturedStep(fn, preserve=keep)
        cs = CapturedStep(fn, preserve=keep)  # warm-up/capture without events, then an instrumented twin
        # the twin is single-stream: each kernel's events then time that kernel
        # alone, not its contention with the forked weight-gradient branch
        timer.reset_records()
        self.concurrent = False
        try:
            with timer:
                inst = CapturedStep(fn, warmup=0)
        finally:
            self.concurrent = True
        return cs, inst

    def training_state(self) -> list:
        """Tensors a step mutates beyond its activations (restored around a
        capture's warm-up, graphs.CapturedStep)."""
        return [t.flat for t in (self.master, self.grad, self.wlow) if t is not None]

    def device_inputs(self, B: int, S: int) -> dict:
        """Static device buffers a captured step reads (fill before replay)."""
        return self._dev_inputs(B, S)



def fused_step_bytes(c: BertLayerConfig, B: int, S: int) -> int:
    """Compulsory HBM bytes of one fused training step (bf16 fused attention
    path, SGD included): every kernel's tensor arguments read once and written
    once, as scheduled by BertEncoderLayer.forward / backward / sgd_step."""
    T, H, F, NH = B * S, c.hidden, c.ffn, c.heads
    e = torch.tensor([], dtype=c.dtype).element_size()
    th, tf, t3 = T * H * e, T * F * e, T * 3 * H * e
    fused = c.fused_attention and c.dtype == torch.bfloat16 and c.head_dim == 64 and S % 128 == 0 and S <= 512
    bits = B * NH * S * S // 8
    lse = B * NH * S * 4
    kb = T * H // 8 if fused and H % 32 == 0 else T * H  # BDRLN keep flags (packed or u8)
    w = lambda n, k: n * k * e  # noqa: E731  (bf16 weight operand)
    g32 = lambda n, k: n * k * 4  # noqa: E731  (f32 weight gradient)
    # D pre-pass: O, dO -> D; key-strip kernel: Q, K, V, dO, lse, D, column keep bits -> dK, dV, dSᵀ;
    # dQ GEMM: dSᵀ, K -> dQ
    ds = B * NH * S * S * e
    attn_bwd = (2 * th + lse) + (t3 + th + 2 * lse + bits + 2 * t3 // 3 + ds) + (ds + t3 // 3 + t3 // 3)
    fwd = (th + w(3 * H, H) + t3) + (t3 + bits + th + bits + lse) + (th + w(H, H) + th) \
        + (2 * th + kb + 2 * th) + (th + w(F, H) + 2 * tf) + (tf + w(H, F) + th) + (2 * th + kb + 2 * th)
    bwd = (2 * th + kb + 2 * th) + (th + w(H, F) + tf + tf) + (th + tf + g32(H, F)) + tf \
        + (tf + w(F, H) + th + th) + (tf + th + g32(F, H)) + (2 * th + kb + 2 * th) + (th + w(H, H) + th) \
        + (2 * th + g32(H, H)) + attn_bwd \
        + (t3 + w(3 * H, H) + th + th) + (t3 + th + g32(3 * H, H))
    nparam = sum(_numel(sh) for _, sh in _param_specs(c))
    sgd = nparam * (4 + 4 + 4 + (2 if c.dtype == torch.bfloat16 else 0))
    return int(fwd + bwd + sgd)


def fused_step_flops(c: BertLayerConfig, B: int, S: int) -> int:
    """Algorithmic contraction FLOPs of one fwd+bwd step (SURVEY.md §8a row
    a8): QKV, QKᵀ, PV, out-proj, FFN1, FFN2 forward, x3 for the backward."""
    T = B * S
    fwd = 2 * T * c.hidden * (3 * c.hidden) + 2 * 2 * B * c.heads * S * S * c.head_dim \
        + 2 * T * c.hidden * c.hidden + 2 * 2 * T * c.hidden * c.ffn
    return 3 * fwd
