"""EfficientNet-B0 training step on the B200 path (BASELINE.json configs[4], C5).

The network is torchvision's ``efficientnet_b0`` topology (width 1.0, depth
1.0): stem conv 3x3/2 -> 16 MBConv blocks -> 1x1 head conv -> global average
pool -> classifier, NHWC bf16 activations.  Every operation of the step runs
in the sm_100a library:

* the depthwise conv + BatchNorm(train) + swish + squeeze-excite of each block
  is the fused MBConv path (mbconv.py -> csrc/mbconv.cu + csrc/dwconv.cu), the
  reference's Conv(group=C) / BatchNormalization / Sigmoid+Mul /
  GlobalAveragePool+Gemm chain (frontend.py:544-706);
* every 1x1 convolution (expand, project, head), the stem (im2col + GEMM) and
  the classifier are tcgen05 GEMMs (csrc/gemm_tc.cu; the reference's Conv with
  1x1 kernels / Gemm, frontend.py:369-405, 598-678), weight and input
  gradients included;
* the GEMM-side BatchNorms (+ swish) are the channels-last BN kernels of the
  normalisation sweep (norms.py -> csrc/norm.cu);
* pooling, the softmax cross-entropy and the residual adds are the small
  kernels of csrc/effnet.cu.

Deliberate simplifications (no effect on the data movement being measured):
no dropout before the classifier and no stochastic depth (both are identity
at p = 0); BatchNorm follows the reference's running-statistics convention
(frontend.py:565-571, momentum m: ``run = m*run + (1-m)*batch``, biased var).

Parameters live in ONE flat f32 master arena (+ a bf16 copy for the tensor
cores) and gradients in ONE flat f32 arena — the SGD step and the
data-parallel gradient allreduce are one pass / one bucketed collective each.
With a process group every BatchNorm is SyncBN (dp.py).
"""

from __future__ import annotations

import contextlib
import ctypes
import os
from dataclasses import dataclass

import torch

from . import _lib
from . import kernels as K
from ._lib import EPI_BIAS
from .bert import FlatArena
from .errors import ShapeError
from .mbconv import MBConvBlock, MBConvConfig
from .norms import BatchNormAct

# (expand ratio, kernel, stride, in, out, layers) — torchvision efficientnet_b0
B0_STAGES = ((1, 3, 1, 32, 16, 1), (6, 3, 2, 16, 24, 2), (6, 5, 2, 24, 40, 2), (6, 3, 2, 40, 80, 3),
             (6, 5, 1, 80, 112, 3), (6, 5, 2, 112, 192, 4), (6, 3, 1, 192, 320, 1))


def _divisible(v: float, d: int = 8) -> int:
    """torchvision's _make_divisible: round to a multiple of 8, never below 90%."""
    n = max(d, int(v + d / 2) // d * d)
    if n < 0.9 * v:
        n += d
    return n


@dataclass(frozen=True)
class EffNetConfig:
    image: int = 224
    classes: int = 1000
    width: float = 1.0
    eps: float = 1e-5
    momentum: float = 0.9
    dtype: torch.dtype = torch.bfloat16
    # bf16: the SE excite is folded into the project 1x1 GEMM (kernels.gemm_excite:
    # y = swish(BN(z)) * s formed from z inside the tcgen05 GEMM)
    fold_excite: bool = os.environ.get("DFX_EXCITE_FOLD", "1") != "0"

    def blocks(self):
        """[(expand, k, stride, cin, cexp, cout, se)] for the 16 blocks."""
        out = []
        for e, k, s, cin, cout, n in B0_STAGES:
            cin, cout = _divisible(cin * self.width), _divisible(cout * self.width)
            for i in range(n):
                ci = cin if i == 0 else cout
                out.append((e, k, s if i == 0 else 1, ci, _divisible(ci * e), cout, max(1, ci // 4)))
        return out

    @property
    def stem(self) -> int:
        return _divisible(32 * self.width)

    @property
    def head(self) -> int:
        return 4 * self.blocks()[-1][5]  # torchvision: last_channel = 4 x lastconv input (1280 at width 1)


STEM_K = 32  # 3x3x3 = 27 im2col taps, padded to a 16-byte multiple


def param_specs(c: EffNetConfig):
    """Arena order = the order ``EfficientNetB0.backward`` finishes the
    gradients (classifier and head first, then the blocks from last to first,
    the stem last; inside a block: project BN, project weight, the MBConv
    parameters, expand BN, expand weight), so the bucketed data-parallel
    allreduce (dp.GradAllReducer) reduces the front of the arena while the
    backward is still producing the rest."""
    model = dict(model_specs(c))
    order = ["fc.w", "fc.b", "head.g", "head.b", "head.w"]
    for i in reversed(range(len(c.blocks()))):
        p = f"b{i}."
        order += [p + n for n in ("g3", "b3", "wp", "wdw", "g", "b", "wr", "br", "wse", "bse", "g1", "b1", "we")
                  if p + n in model]
    order += ["stem.g", "stem.b", "stem.w"]
    assert sorted(order) == sorted(model)
    return [(n, model[n]) for n in order]


def grad_group_ends(c: EffNetConfig):
    """Last arena entry of each gradient group (head, every block, stem)."""
    ends = ["head.w"]
    for i in reversed(range(len(c.blocks()))):
        ends.append(f"b{i}." + ("we" if c.blocks()[i][0] != 1 else "bse"))
    return ends + ["stem.w"]


def model_specs(c: EffNetConfig):
    """Parameters in model order (initialisation draws in this order)."""
    specs = [("stem.w", (c.stem, STEM_K)), ("stem.g", (c.stem,)), ("stem.b", (c.stem,))]
    for i, (e, k, s, ci, cx, co, se) in enumerate(c.blocks()):
        p = f"b{i}."
        if e != 1:
            specs += [(p + "we", (cx, ci)), (p + "g1", (cx,)), (p + "b1", (cx,))]
        specs += [(p + "wdw", (k, k, cx)), (p + "g", (cx,)), (p + "b", (cx,)), (p + "wr", (se, cx)),
                  (p + "br", (se,)), (p + "wse", (cx, se)), (p + "bse", (cx,)),
                  (p + "wp", (co, cx)), (p + "g3", (co,)), (p + "b3", (co,))]
    last = c.blocks()[-1][5]
    specs += [("head.w", (c.head, last)), ("head.g", (c.head,)), ("head.b", (c.head,)),
              ("fc.w", (c.classes, c.head)), ("fc.b", (c.classes,))]
    return specs


class _Names:
    """A block-local name -> arena view map (what MBConvBlock indexes)."""

    def __init__(self, arena, mapping):
        self.views = {local: arena[glob] for local, glob in mapping.items()}

    def __getitem__(self, name):
        return self.views[name]


def _gemm(a, w, out, **kw):
    return K.gemm(a, w, out, **kw)


class _Block:
    """expand 1x1 (GEMM) + BN + swish -> fused dw/BN/swish/SE -> project 1x1 + BN (+ residual)."""

    def __init__(self, net, i, spec, pg):
        e, k, s, ci, cx, co, se = spec
        self.e, self.k, self.s, self.ci, self.cx, self.co = e, k, s, ci, cx, co
        self.residual = s == 1 and ci == co
        c, dev, P, G, Wl = net.cfg, net.device, net.master, net.grad, net.wlow
        p = f"b{i}."
        self.p = p
        self.net = net
        if e != 1:
            self.bn1 = BatchNormAct(cx, c.eps, c.momentum, "swish", dev, pg)
            _bind_bn(self.bn1, P, G, p + "g1", p + "b1")
        self.bn3 = BatchNormAct(co, c.eps, c.momentum, "none", dev, pg)
        _bind_bn(self.bn3, P, G, p + "g3", p + "b3")
        mb = MBConvBlock(MBConvConfig(channels=cx, se=se, stride=s, pads=(k // 2,) * 4, ksize=k, eps=c.eps,
                                      momentum=c.momentum, dtype=c.dtype), device=dev, process_group=pg)
        names = {"wdw": p + "wdw", "g": p + "g", "b": p + "b", "wr": p + "wr", "br": p + "br", "we": p + "wse",
                 "be": p + "bse"}
        mb.master, mb.grad = _Names(P, names), _Names(G, names)
        self.mb = mb
        self.Wl = Wl

    def w(self, name):
        return self.Wl[self.p + name] if self.Wl is not None else self.net.master[self.p + name]

    def _out_hw(self, x):
        """Output pixels per image of the depthwise conv (the fold needs >= 32)."""
        _, H, W, _ = x.shape
        p = self.k // 2
        return ((H + 2 * p - self.k) // self.s + 1) * ((W + 2 * p - self.k) // self.s + 1)

    def forward(self, x):
        N, H, W, _ = x.shape
        self.x = x
        if self.e != 1:
            h = torch.empty(N, H, W, self.cx, dtype=x.dtype, device=x.device)
            with K.label("block.expand_gemm"):
                _gemm(x.view(-1, self.ci), self.w("we"), h.view(-1, self.cx))
            a = self.bn1.forward(h)
        else:
            a = x
        self.a = a
        if self.net.cfg.fold_excite and x.dtype == torch.bfloat16 and self._out_hw(x) >= 32:
            # excite + project as one GEMM over z; y is still written for the weight gradient
            self.mb.forward(a, excite=False)
            mbb = self.mb.buffers(a.shape)
            y = mbb["y"]
            No, Ho, Wo, _ = y.shape
            pr = torch.empty(No, Ho, Wo, self.co, dtype=x.dtype, device=x.device)
            with K.label("block.excite_project_gemm"):
                K.gemm_excite(mbb["z"].view(-1, self.cx), Ho * Wo, mbb["mean"], mbb["rstd"], self.mb.master["g"],
                              self.mb.master["b"], mbb["s"], self.w("wp"), pr.view(-1, self.co),
                              y_out=y.view(-1, self.cx))
        else:
            y = self.mb.forward(a)
            No, Ho, Wo, _ = y.shape
            pr = torch.empty(No, Ho, Wo, self.co, dtype=x.dtype, device=x.device)
            with K.label("block.project_gemm"):
                _gemm(y.view(-1, self.cx), self.w("wp"), pr.view(-1, self.co))
        self.y = y
        o = self.bn3.forward(pr)
        if self.residual:
            _lib.call("dfx_add", K.dfx_dtype(o), o.numel(), o.data_ptr(), x.data_ptr(), o.data_ptr(), K._stream())
        return o

    def backward(self, do):
        G = self.net.grad
        dp = self.bn3.backward(do)
        y2 = self.y.view(-1, self.cx)
        dy = torch.empty_like(self.y)
        with K.label("block.project_dgrad"):
            _gemm(dp.view(-1, self.co), self.w("wp").t(), dy.view(-1, self.cx))
        with self.net.fork(dp):
            with K.label("block.project_wgrad"):
                _gemm(dp.view(-1, self.co).t(), y2.t(), G[self.p + "wp"])
        da = self.mb.backward(dy)
        if self.e != 1:
            dh = self.bn1.backward(da)
            dx = torch.empty_like(self.x)
            with K.label("block.expand_dgrad"):
                _gemm(dh.view(-1, self.cx), self.w("we").t(), dx.view(-1, self.ci))
            with self.net.fork(dh):
                with K.label("block.expand_wgrad"):
                    _gemm(dh.view(-1, self.cx).t(), self.x.view(-1, self.ci).t(), G[self.p + "we"])
        else:
            dx = da  # the MBConv block's own dx buffer (no residual on expand-ratio-1 blocks)
        if self.residual:
            _lib.call("dfx_add", K.dfx_dtype(dx), dx.numel(), dx.data_ptr(), do.data_ptr(), dx.data_ptr(),
                      K._stream())
        return dx


def _bind_bn(bn, P, G, gname, bname):
    bn.gamma, bn.beta = P[gname], P[bname]
    bn.dgamma, bn.dbeta = G[gname], G[bname]


class EfficientNetB0:
    """One data-parallel replica of the EfficientNet-B0 training step."""

    def __init__(self, cfg: EffNetConfig = EffNetConfig(), device="cuda", seed: int = 0, process_group=None):
        if cfg.dtype not in (torch.float32, torch.bfloat16):
            raise ShapeError("EfficientNetB0: dtype must be float32 or bfloat16")
        _lib.load(check_device=True)
        self.cfg = cfg
        self.device = torch.device(device)
        self.pg = process_group
        self.world = 1 if process_group is None else torch.distributed.get_world_size(process_group)
        specs = param_specs(cfg)
        self.master = FlatArena(specs, torch.float32, self.device)
        self.grad = FlatArena(specs, torch.float32, self.device)
        self.wlow = FlatArena(specs, torch.bfloat16, self.device) if cfg.dtype == torch.bfloat16 else None
        self._init(seed)
        self.stem_bn = BatchNormAct(cfg.stem, cfg.eps, cfg.momentum, "swish", self.device, process_group)
        _bind_bn(self.stem_bn, self.master, self.grad, "stem.g", "stem.b")
        self.blocks = [_Block(self, i, b, process_group) for i, b in enumerate(cfg.blocks())]
        self.head_bn = BatchNormAct(cfg.head, cfg.eps, cfg.momentum, "swish", self.device, process_group)
        _bind_bn(self.head_bn, self.master, self.grad, "head.g", "head.b")
        self.loss = torch.zeros(1, device=self.device)
        self._pads = (ctypes.c_int * 4)(1, 1, 1, 1)
        self.concurrent = True  # weight gradients on a forked stream (backward)
        self._bufs = {}
        self.reducer = None
        if process_group is not None and self.world > 1:
            self.attach_process_group(process_group)

    def attach_process_group(self, group=None, bucket_bytes: int = 4 << 20):
        """Data parallel: the backward all-reduces (SUM) the gradient arena
        bucket by bucket as the head, each block and the stem finish their
        gradients; ``train_step`` folds the 1/world average into the SGD
        learning rate."""
        from .dp import GradAllReducer

        G = self.grad
        ends = [G.offsets[n][0] + G[n].numel() for n in grad_group_ends(self.cfg)]
        self.reducer = GradAllReducer(G.flat, group, bucket_bytes, boundaries=ends)
        return self.reducer

    def _ready(self, name):
        if self.reducer is not None:
            off, _ = self.grad.offsets[name]
            main = torch.cuda.current_stream(self.device)
            streams = (main, self._side) if self.concurrent and hasattr(self, "_side") else (main,)
            self.reducer.mark_ready(off + self.grad[name].numel(), streams)

    # ------------------------------------------------------------ parameters
    def _init(self, seed):
        g = torch.Generator(device="cpu").manual_seed(seed)
        for name, shape in model_specs(self.cfg):  # draw order independent of the arena order
            v = self.master[name]
            leaf = name.split(".")[-1]
            if leaf in ("g", "g1", "g3"):
                t = torch.ones(shape)
            elif leaf in ("b", "b1", "b3", "br", "bse"):
                t = torch.zeros(shape)
            elif leaf == "wdw":
                t = torch.randn(shape, generator=g) / shape[0]
            elif name == "stem.w":
                t = torch.randn(shape, generator=g) / 27 ** 0.5
                t[:, 27:] = 0
            elif name == "fc.b":
                t = torch.zeros(shape)
            else:  # GEMM / SE weights [out, in]
                t = torch.randn(shape, generator=g) / shape[-1] ** 0.5
            v.copy_(t)
        self.refresh_low()

    def refresh_low(self):
        if self.wlow is not None:
            K.cast(self.master.flat, self.wlow.flat)

    def w(self, name):
        return self.wlow[name] if self.wlow is not None else self.master[name]

    @property
    def num_params(self) -> int:
        return sum(v.numel() for v in self.master.views.values()) - self.cfg.stem * (STEM_K - 27)

    # ------------------------------------------------------------ step
    def forward(self, x, labels):
        """x [N, H, W, 3] NHWC, labels int32 [N] -> loss (device scalar)."""
        c = self.cfg
        if x.dtype != c.dtype or x.dim() != 4 or x.shape[-1] != 3 or not x.is_contiguous():
            raise ShapeError(f"EfficientNetB0: x must be a contiguous NHWC [N, H, W, 3] {c.dtype} tensor")
        if labels.dtype != torch.int32 or labels.shape != (x.shape[0],):
            raise ShapeError("EfficientNetB0: labels must be int32 [N]")
        N, H, W, _ = x.shape
        Ho, Wo = (H - 1) // 2 + 1, (W - 1) // 2 + 1
        dt, st = K.dfx_dtype(x), K._stream()
        cols = torch.empty(N * Ho * Wo, STEM_K, dtype=x.dtype, device=x.device)
        with K._span("stem.im2col", "hbm", lambda: cols.numel() * cols.element_size()):
            _lib.call("dfx_im2col3x3", dt, N, H, W, 3, 2, self._pads, STEM_K, x.data_ptr(), cols.data_ptr(), st)
        self.cols = cols
        h = torch.empty(N, Ho, Wo, c.stem, dtype=x.dtype, device=x.device)
        with K.label("stem.gemm"):
            _gemm(cols, self.w("stem.w"), h.view(-1, c.stem))
        cur = self.stem_bn.forward(h)
        for b in self.blocks:
            cur = b.forward(cur)
        self.last = cur
        Nb, Hh, Wh, Cl = cur.shape
        hh = torch.empty(Nb, Hh, Wh, c.head, dtype=x.dtype, device=x.device)
        with K.label("head.gemm"):
            _gemm(cur.view(-1, Cl), self.w("head.w"), hh.view(-1, c.head))
        ah = self.head_bn.forward(hh)
        self.ah = ah
        pooled = torch.empty(N, c.head, dtype=x.dtype, device=x.device)
        with K._span("head.avgpool", "hbm", lambda: ah.numel() * ah.element_size()):
            _lib.call("dfx_avgpool_fwd", dt, N, Hh * Wh, c.head, ah.data_ptr(), pooled.data_ptr(), st)
        self.pooled = pooled
        logits = torch.empty(N, c.classes, dtype=torch.float32, device=x.device)
        with K.label("fc.gemm"):
            _gemm(pooled, self.w("fc.w"), logits, epilogue=EPI_BIAS, bias=self.master["fc.b"])
        self.logits = logits
        rows = torch.empty(N, dtype=torch.float32, device=x.device)
        dlogits = torch.empty(N, c.classes, dtype=x.dtype, device=x.device)
        with K._span("loss.xent", "hbm", lambda: logits.numel() * 4):
            _lib.call("dfx_softmax_xent", N, c.classes, logits.data_ptr(), labels.data_ptr(), self.loss.data_ptr(),
                      rows.data_ptr(), dt, dlogits.data_ptr(), st)
        self.dlogits = dlogits
        return self.loss

    def fork(self, *uses):
        """Run the enclosed launches on the side stream after everything queued
        so far on the main stream (weight gradients: off the dgrad chain).
        ``uses``: freshly allocated tensors the side stream reads — recorded on
        it so the caching allocator cannot hand their memory to a later
        main-stream allocation while the side stream still reads them."""
        main = torch.cuda.current_stream(self.device)
        if not hasattr(self, "_side"):
            self._side = torch.cuda.Stream(device=self.device)
        if not self.concurrent:  # per-kernel attribution: one stream
            return contextlib.nullcontext()
        ev = torch.cuda.Event()
        ev.record(main)
        self._side.wait_event(ev)
        for t in uses:
            t.record_stream(self._side)
        return torch.cuda.stream(self._side)

    def backward(self):
        """Gradients of the mean loss w.r.t. every parameter (this rank's
        batch; the data-parallel sum is the caller's allreduce).  Weight
        gradients run on a forked stream joined at the end."""
        c, G = self.cfg, self.grad
        N = self.pooled.shape[0]
        dt, st = K.dfx_dtype(self.pooled), K._stream()
        dl = self.dlogits
        with self.fork():
            with K.label("fc.wgrad"):
                _gemm(dl.t(), self.pooled.t(), G["fc.w"])
            K.colsum(dl, G["fc.b"])
        dpooled = torch.empty_like(self.pooled)
        with K.label("fc.dgrad"):
            _gemm(dl, self.w("fc.w").t(), dpooled)
        dah = torch.empty_like(self.ah)
        Nb, Hh, Wh, _ = dah.shape
        with K._span("head.avgpool_bwd", "hbm", lambda: dah.numel() * dah.element_size()):
            _lib.call("dfx_avgpool_bwd", dt, N, Hh * Wh, c.head, dpooled.data_ptr(), dah.data_ptr(), st)
        dhh = self.head_bn.backward(dah)
        Cl = self.last.shape[-1]
        dcur = torch.empty_like(self.last)
        with K.label("head.dgrad"):
            _gemm(dhh.view(-1, c.head), self.w("head.w").t(), dcur.view(-1, Cl))
        with self.fork(dhh):
            with K.label("head.wgrad"):
                _gemm(dhh.view(-1, c.head).t(), self.last.view(-1, Cl).t(), G["head.w"])
        self._ready("head.w")
        for i in reversed(range(len(self.blocks))):
            b = self.blocks[i]
            dcur = b.backward(dcur)
            self._ready(b.p + ("we" if b.e != 1 else "bse"))
        dh = self.stem_bn.backward(dcur)
        with self.fork(dh):
            with K.label("stem.wgrad"):
                _gemm(dh.view(-1, c.stem).t(), self.cols.t(), G["stem.w"])
        if self.concurrent:
            torch.cuda.current_stream(self.device).wait_stream(self._side)  # join

    def sgd_step(self, lr: float):
        with K.label("sgd_update"):
            K.sgd_update(self.master.flat, self.grad.flat, lr, None if self.wlow is None else self.wlow.flat)

    def reduce_gradients(self):
        """Finish the bucketed gradient allreduce the backward started (data
        parallel; no-op for one replica).  Returns the world size."""
        return self.reducer.finish() if self.reducer is not None else 1

    def train_step(self, x, labels, lr=None):
        """fwd + bwd (+ bucketed gradient allreduce) (+ SGD on the replica-averaged gradient)."""
        loss = self.forward(x, labels)
        self.backward()
        world = self.reduce_gradients()
        if lr is not None:
            self.sgd_step(lr / world)
        return loss

    # ------------------------------------------------------------ graph / host API
    def device_inputs(self, N: int):
        key = ("in", N, getattr(self, "slot", 0))
        if key not in self._bufs:
            s = self.cfg.image
            self._bufs[key] = {"x": torch.zeros(N, s, s, 3, dtype=self.cfg.dtype, device=self.device),
                               "labels": torch.zeros(N, dtype=torch.int32, device=self.device),
                               "loss": torch.zeros(1, device=self.device)}
        return self._bufs[key]

    def training_state(self) -> list:
        """Tensors a step mutates beyond its activations: parameter / gradient
        arenas, the bf16 shadow and every BatchNorm's running statistics
        (restored around a capture's warm-up, graphs.CapturedStep)."""
        out = [t.flat for t in (self.master, self.grad, self.wlow) if t is not None]
        bns = [self.stem_bn, self.head_bn]
        for b in self.blocks:
            bns += [getattr(b, "bn1", None), b.bn3, b.mb]
        for bn in bns:
            if bn is not None:
                out += [bn.running_mean, bn.running_var]
        return out

    def capture_step(self, N: int, lr=None, timer=None):
        """Forward + backward (+ SGD) on the static ``device_inputs(N)`` as one
        CUDA graph.  Data parallel, the SyncBN statistics collectives and the
        gradient buckets are captured with it (NCCL; gloo cannot be captured)."""
        from .graphs import CapturedStep

        dev = self.device_inputs(N)
        self.loss = dev["loss"]  # per input slot: the graph bakes this buffer in

        def fn():
            self.train_step(dev["x"], dev["labels"], lr)

        keep = self.training_state()
        if timer is None:
            return CapturedStep(fn, preserve=keep)
        cs = CapturedStep(fn, preserve=keep)
        timer.reset_records()
        with timer:
            inst = CapturedStep(fn, warmup=0)
        return cs, inst

    def train_step_host_async(self, x_host, labels_host, lr=None, loss_host=None):
        """Pipelined host-buffer step (single process): two input sets and two
        captured graphs alternate, so step i+1's H2D and step i's loss D2H
        overlap step i's compute.  ``finish_host()`` joins the copy streams."""
        N = x_host.shape[0]
        if not hasattr(self, "_pipe"):
            self._pipe = {"h2d": torch.cuda.Stream(device=self.device), "d2h": torch.cuda.Stream(device=self.device),
                          "free": [None, None], "graphs": {}}
        pp = self._pipe
        slot = getattr(self, "slot", 0)
        comp = torch.cuda.current_stream(self.device)
        key = (N, lr, slot)
        if key not in pp["graphs"]:
            torch.cuda.synchronize(self.device)
            pp["graphs"][key] = self.capture_step(N, lr)
        dev = self.device_inputs(N)
        loss = dev["loss"]
        with torch.cuda.stream(pp["h2d"]):
            if pp["free"][slot] is not None:
                pp["h2d"].wait_event(pp["free"][slot])
            dev["x"].copy_(x_host, non_blocking=True)
            dev["labels"].copy_(labels_host, non_blocking=True)
            ev_in = torch.cuda.Event()
            ev_in.record(pp["h2d"])
        comp.wait_event(ev_in)
        pp["graphs"][key].replay()
        ev_done = torch.cuda.Event()
        ev_done.record(comp)
        with torch.cuda.stream(pp["d2h"]):
            pp["d2h"].wait_event(ev_done)
            if loss_host is not None:
                loss_host.copy_(loss, non_blocking=True)  # this slot's own loss buffer
            ev_free = torch.cuda.Event()
            ev_free.record(pp["d2h"])
        pp["free"][slot] = ev_free
        self.slot = slot ^ 1
        return loss_host

    def finish_host(self):
        if hasattr(self, "_pipe"):
            comp = torch.cuda.current_stream(self.device)
            comp.wait_stream(self._pipe["h2d"])
            comp.wait_stream(self._pipe["d2h"])

    def host_inputs_bytes(self, N: int):
        s = self.cfg.image
        esz = torch.tensor([], dtype=self.cfg.dtype).element_size()
        return N * s * s * 3 * esz + N * 4, 4

    def train_step_host(self, x_host, labels_host, lr=None, loss_host=None, graph=None):
        """One step from HOST (pinned) images/labels: H2D copies, the step
        (CUDA-graph replay when ``graph`` is given), D2H of the loss."""
        N = x_host.shape[0]
        dev = self.device_inputs(N)
        dev["x"].copy_(x_host, non_blocking=True)
        dev["labels"].copy_(labels_host, non_blocking=True)
        if graph is not None:
            graph.replay()  # captured by capture_step(N): writes this slot's dev["loss"]
            loss = dev["loss"]
        else:
            loss = self.train_step(dev["x"], dev["labels"], lr)
        if loss_host is not None:
            loss_host.copy_(loss, non_blocking=True)
        return loss_host
