"""EfficientNet-B0 MBConv block (depthwise 3x3 + BatchNorm(train) + swish +
squeeze-excite) training step on the B200 hot path, NHWC.

Reference graph (SURVEY.md:512-514; golden in oracle/make_golden.py):

    z  = Conv(x, w_dw, group=C, pads, strides)          frontend.py:598-678
    u, run_mean', run_var' = BatchNormalization(z, ...)  frontend.py:544-591 (training)
    a  = u * Sigmoid(u)                                  frontend.py:229, 293
    p  = GlobalAveragePool(a) -> [N, C]                  frontend.py:681-706
    s  = Sigmoid(Gemm(swish(Gemm(p, Wr, br, transB)), We, be, transB))
    y  = a * s[:, :, None, None]

The reference is NCHW; this path is NHWC (channels contiguous, 128-bit
vectors across channels).  ``forward``/``backward`` take NHWC tensors; the
weight views accept/produce the reference layouts.

Data parallel: pass a ``torch.distributed`` process group to get SyncBN —
each rank's per-channel (count, mean, M2) is all-gathered and merged in
rank order (no E[x^2]-E[x]^2 cancellation), and the backward BN sums are
all-reduced before the input gradient is formed.  Parity contract: the result
equals single-GPU BatchNorm over the concatenated batch
(frontend.py:558-573).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from . import kernels as K
from .bert import FlatArena
from .dp import allreduce_sum, bn_slot, exchange_bn_sets
from .errors import ShapeError


@dataclass(frozen=True)
class MBConvConfig:
    channels: int = 96
    se: int = 4
    stride: int = 1
    pads: tuple = (1, 1, 1, 1)
    ksize: int = 3
    eps: float = 1e-3
    momentum: float = 0.99
    dtype: torch.dtype = torch.float32


def _specs(c: MBConvConfig):
    C, SE = c.channels, c.se
    return [("wdw", (c.ksize, c.ksize, C)), ("g", (C,)), ("b", (C,)), ("wr", (SE, C)), ("br", (SE,)),
            ("we", (C, SE)), ("be", (C,))]


class MBConvBlock:
    def __init__(self, cfg: MBConvConfig = MBConvConfig(), device="cuda", seed: int = 0,
                 process_group=None):
        if cfg.dtype not in (torch.float32, torch.bfloat16):
            raise ShapeError("MBConvBlock: dtype must be float32 or bfloat16")
        _lib.load(check_device=True)
        self.cfg = cfg
        self.device = torch.device(device)
        self.pg = process_group
        self.world = 1 if process_group is None else torch.distributed.get_world_size(process_group)
        self.master = FlatArena(_specs(cfg), torch.float32, self.device)
        self.grad = FlatArena(_specs(cfg), torch.float32, self.device)
        C = cfg.channels
        self.running_mean = torch.zeros(C, device=self.device)
        self.running_var = torch.ones(C, device=self.device)
        self._bufs = {}
        g = torch.Generator(device="cpu").manual_seed(seed)
        self.load_params({
            "wdw": 0.3 * torch.randn(C, 1, cfg.ksize, cfg.ksize, generator=g),
            "g": 1 + 0.1 * torch.randn(C, generator=g), "b": 0.1 * torch.randn(C, generator=g),
            "wr": 0.3 * torch.randn(cfg.se, C, generator=g), "br": 0.1 * torch.randn(cfg.se, generator=g),
            "we": 0.3 * torch.randn(C, cfg.se, generator=g), "be": 0.1 * torch.randn(C, generator=g)})

    # ------------------------------------------------------------ parameters
    def load_params(self, vals: dict):
        """``wdw`` in the reference layout (C, 1, 3, 3); ``rm``/``rv`` load
        the running statistics."""
        for name, _ in _specs(self.cfg):
            v = torch.as_tensor(vals[name], dtype=torch.float32)
            if name == "wdw":
                k = self.cfg.ksize
                v = v.reshape(self.cfg.channels, k, k).permute(1, 2, 0)
            self.master[name].copy_(v.to(self.device))
        if "rm" in vals:
            self.running_mean.copy_(torch.as_tensor(vals["rm"], dtype=torch.float32))
        if "rv" in vals:
            self.running_var.copy_(torch.as_tensor(vals["rv"], dtype=torch.float32))

    def grads_numpy(self):
        out = {k: v.detach().cpu().double().numpy() for k, v in self.grad.views.items()}
        k = self.cfg.ksize
        out["wdw"] = out["wdw"].transpose(2, 0, 1).reshape(self.cfg.channels, 1, k, k)
        return out

    # ------------------------------------------------------------ buffers
    def _geo(self, x_shape):
        N, H, W, C = x_shape
        if C != self.cfg.channels:
            raise ShapeError(f"MBConvBlock: expected {self.cfg.channels} channels, got {C}")
        p = self.cfg.pads
        k = self.cfg.ksize
        Ho = (H + p[0] + p[2] - k) // self.cfg.stride + 1
        Wo = (W + p[1] + p[3] - k) // self.cfg.stride + 1
        return N, H, W, C, Ho, Wo

    def buffers(self, x_shape):
        key = tuple(x_shape)
        if key not in self._bufs:
            c = self.cfg
            N, H, W, C, Ho, Wo = self._geo(x_shape)
            dev, dt = self.device, c.dtype
            f = lambda *s: torch.empty(s, dtype=torch.float32, device=dev)  # noqa: E731
            ws = _lib.load().dfx_mbconv_workspace(N, H, W, C, c.stride, c.ksize, self._pads(), c.se)
            self._bufs[key] = dict(
                z=torch.empty(N, Ho, Wo, C, dtype=dt, device=dev),
                y=torch.empty(N, Ho, Wo, C, dtype=dt, device=dev),
                dx=torch.empty(N, H, W, C, dtype=dt, device=dev),
                bn_local=f(3, C), bn_sets=f(self.world, 3, C), mean=f(C), var=f(C), rstd=f(C),
                pooled=f(N, C), r=f(N, c.se), s=f(N, C), dpool=f(N, C), bnsum=f(3, C),
                ws=torch.empty(ws, dtype=torch.uint8, device=dev))
        return self._bufs[key]

    def _pads(self):
        import ctypes

        self._pads_c = (ctypes.c_int * 4)(*self.cfg.pads)
        return self._pads_c

    # ------------------------------------------------------------ forward
    def forward(self, x, excite: bool = True):
        """x [N, H, W, C] (NHWC) -> y [N, Ho, Wo, C]; updates running stats.
        ``excite=False`` stops after the SE gate ``s`` (buffers()["s"]): the
        caller folds y = swish(BN(z)) * s into its consumer
        (kernels.gemm_excite) and None is returned."""
        c = self.cfg
        if x.dtype != c.dtype or x.dim() != 4 or not x.is_contiguous():
            raise ShapeError(f"MBConvBlock: x must be a contiguous NHWC {c.dtype} tensor")
        N, H, W, C, Ho, Wo = self._geo(x.shape)
        b = self.buffers(x.shape)
        P = self.master
        dt = K.dfx_dtype(x)
        st = K._stream()
        pads = self._pads()
        ws = b["ws"]
        self._saved = x
        esz = x.element_size()
        # SyncBN: the statistics land directly in this rank's slot of the exchange buffer
        stats = bn_slot(b["bn_sets"], self.pg) if self.world > 1 else b["bn_local"]
        with K._span("mbconv.dwconv_stats", "hbm", lambda: (N * H * W + N * Ho * Wo) * C * esz):
            _lib.call("dfx_mbconv_fwd_stats", dt, N, H, W, C, c.stride, c.ksize, pads, x.data_ptr(),
                      P["wdw"].data_ptr(), b["z"].data_ptr(), stats.data_ptr(), ws.data_ptr(),
                      ws.numel(), st)
        sets = exchange_bn_sets(b["bn_sets"], group=self.pg) if self.world > 1 else b["bn_local"]
        with K._span("mbconv.bn_finalize", "hbm", lambda: 8 * C * 4):
            _lib.call("dfx_bn_finalize", C, self.world, sets.data_ptr(), float(c.eps), float(c.momentum),
                      b["mean"].data_ptr(), b["var"].data_ptr(), b["rstd"].data_ptr(),
                      self.running_mean.data_ptr(), self.running_var.data_ptr(), st)
        with K._span("mbconv.bn_swish_se_excite" if excite else "mbconv.bn_swish_se", "hbm",
                     lambda: (3 if excite else 1) * N * Ho * Wo * C * esz):
            _lib.call("dfx_mbconv_fwd_se", dt, N, H, W, C, c.stride, c.ksize, pads, c.se, b["z"].data_ptr(),
                      b["mean"].data_ptr(), b["rstd"].data_ptr(), P["g"].data_ptr(), P["b"].data_ptr(),
                      P["wr"].data_ptr(), P["br"].data_ptr(), P["we"].data_ptr(), P["be"].data_ptr(),
                      b["pooled"].data_ptr(), b["r"].data_ptr(), b["s"].data_ptr(),
                      b["y"].data_ptr() if excite else None, ws.data_ptr(), ws.numel(), st)
        return b["y"] if excite else None

    # ------------------------------------------------------------ backward
    def backward(self, dy):
        c = self.cfg
        x = self._saved
        N, H, W, C, Ho, Wo = self._geo(x.shape)
        if tuple(dy.shape) != (N, Ho, Wo, C) or dy.dtype != c.dtype or not dy.is_contiguous():
            raise ShapeError("MBConvBlock.backward: dy must match the forward output")
        b = self.buffers(x.shape)
        P, G = self.master, self.grad
        dt = K.dfx_dtype(x)
        st = K._stream()
        pads = self._pads()
        ws = b["ws"]
        esz = x.element_size()
        with K._span("mbconv.bwd_reduce", "hbm", lambda: 2 * N * Ho * Wo * C * esz):
            _lib.call("dfx_mbconv_bwd_reduce", dt, N, H, W, C, c.stride, c.ksize, pads, c.se, dy.data_ptr(),
                      b["z"].data_ptr(), b["mean"].data_ptr(), b["rstd"].data_ptr(), P["g"].data_ptr(),
                      P["b"].data_ptr(), b["s"].data_ptr(), b["r"].data_ptr(), b["pooled"].data_ptr(),
                      P["wr"].data_ptr(), P["we"].data_ptr(), G["we"].data_ptr(), G["be"].data_ptr(),
                      G["wr"].data_ptr(), G["br"].data_ptr(), b["dpool"].data_ptr(), b["bnsum"].data_ptr(),
                      ws.data_ptr(), ws.numel(), st)
        # local BN parameter gradients (dbeta = sum du, dgamma = sum du*xhat)
        K.cast2(b["bnsum"][0], G["b"], b["bnsum"][1], G["g"])
        count = float(N * Ho * Wo)
        if self.world > 1:
            # SyncBN: global (sum du, sum du*xhat, count) for the input gradient;
            # each rank adds its OWN count, so unequal per-rank batches normalise
            # like the forward's merged statistics (count 0 = read bnsum[2])
            b["bnsum"][2].fill_(count)
            allreduce_sum(b["bnsum"], group=self.pg)
            count = 0.0
        with K._span("mbconv.dwconv_bwd", "hbm", lambda: (2 * N * Ho * Wo + 2 * N * H * W) * C * esz):
            _lib.call("dfx_mbconv_bwd_dx", dt, N, H, W, C, c.stride, c.ksize, pads, dy.data_ptr(), b["z"].data_ptr(),
                      x.data_ptr(), P["wdw"].data_ptr(), b["mean"].data_ptr(), b["rstd"].data_ptr(),
                      P["g"].data_ptr(), P["b"].data_ptr(), b["s"].data_ptr(), b["dpool"].data_ptr(),
                      b["bnsum"].data_ptr(), count, b["dx"].data_ptr(), G["wdw"].data_ptr(), ws.data_ptr(),
                      ws.numel(), st)
        return b["dx"]

    def sgd_step(self, lr: float):
        K.sgd_update(self.master.flat, self.grad.flat, lr)
