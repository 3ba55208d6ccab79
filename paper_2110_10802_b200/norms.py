"""Normalisation sweep (config C4): LayerNorm vs BatchNorm fused with an
activation, forward + backward, on 4D/5D activations.

* ``LayerNormAct``: LayerNormalization over the last axis (frontend.py:519-529)
  followed by swish (or identity); one row kernel each way.
* ``BatchNormAct``: training-mode BatchNormalization over the channel axis
  (frontend.py:544-591) followed by swish; the tensor is channels-last
  ([N, *spatial, C]) so the channel vector is contiguous.  With a process
  group the statistics are SyncBN (same protocol as mbconv.py).
"""

from __future__ import annotations

import torch

from . import _lib
from . import kernels as K
from .dp import allreduce_sum, bn_slot, exchange_bn_sets
from .errors import ShapeError

ACTS = {"none": 0, "swish": 1}


def _act(name):
    try:
        return ACTS[name]
    except KeyError:
        raise ShapeError(f"activation {name!r} not supported (none, swish)") from None


class LayerNormAct:
    def __init__(self, dim: int, eps: float = 1e-5, act: str = "swish", device="cuda"):
        _lib.load(check_device=True)
        self.dim, self.eps, self.act = dim, eps, _act(act)
        self.gamma = torch.ones(dim, device=device)
        self.beta = torch.zeros(dim, device=device)
        self.dgamma = torch.zeros(dim, device=device)
        self.dbeta = torch.zeros(dim, device=device)

    def forward(self, x, y=None):
        if x.shape[-1] != self.dim or not x.is_contiguous():
            raise ShapeError("LayerNormAct: x must be contiguous with last dim == dim")
        self._x = x
        y = torch.empty_like(x) if y is None else y
        rows = x.numel() // self.dim
        with K._span("ln_act_fwd", "hbm", lambda: 2 * x.numel() * x.element_size()):
            _lib.call("dfx_layernorm_act_fwd", K.dfx_dtype(x), rows, self.dim, x.data_ptr(),
                      self.gamma.data_ptr(), self.beta.data_ptr(), float(self.eps), self.act, y.data_ptr(),
                      K._stream())
        return y

    def backward(self, dy, dx=None):
        x = self._x
        dx = torch.empty_like(x) if dx is None else dx
        rows = x.numel() // self.dim
        ws = K.WORKSPACE.get(_lib.load().dfx_bdrln_bwd_workspace(rows, self.dim))
        with K._span("ln_act_bwd", "hbm", lambda: 3 * x.numel() * x.element_size()):
            _lib.call("dfx_layernorm_act_bwd", K.dfx_dtype(x), rows, self.dim, dy.data_ptr(), x.data_ptr(),
                      self.gamma.data_ptr(), self.beta.data_ptr(), float(self.eps), self.act, dx.data_ptr(),
                      self.dgamma.data_ptr(), self.dbeta.data_ptr(), ws.data_ptr(), ws.numel(), K._stream())
        return dx


class BatchNormAct:
    def __init__(self, channels: int, eps: float = 1e-5, momentum: float = 0.9, act: str = "swish",
                 device="cuda", process_group=None):
        _lib.load(check_device=True)
        self.C, self.eps, self.momentum, self.act = channels, eps, momentum, _act(act)
        self.pg = process_group
        self.world = 1 if process_group is None else torch.distributed.get_world_size(process_group)
        f = lambda *s: torch.zeros(s, device=device)  # noqa: E731
        self.gamma, self.beta = torch.ones(channels, device=device), f(channels)
        self.running_mean, self.running_var = f(channels), torch.ones(channels, device=device)
        self.dgamma, self.dbeta = f(channels), f(channels)
        self.local, self.sets = f(3, channels), f(self.world, 3, channels)
        self.mean, self.var, self.rstd, self.bnsum = f(channels), f(channels), f(channels), f(3, channels)

    def forward(self, x, y=None):
        """x channels-last [..., C]; returns act(BN(x))."""
        if x.shape[-1] != self.C or not x.is_contiguous():
            raise ShapeError("BatchNormAct: x must be contiguous channels-last [..., C]")
        self._x = x
        rows = x.numel() // self.C
        dt, st = K.dfx_dtype(x), K._stream()
        ws = K.WORKSPACE.get(_lib.load().dfx_batchnorm_workspace(rows, self.C))
        y = torch.empty_like(x) if y is None else y
        # SyncBN: the statistics land directly in this rank's slot of the exchange buffer
        stats = bn_slot(self.sets, self.pg) if self.world > 1 else self.local
        if self.world == 1:  # statistics and their finalize in one pass over the block partials
            with K._span("bn_stats", "hbm", lambda: x.numel() * x.element_size()):
                _lib.call("dfx_batchnorm_stats_finalize", dt, rows, self.C, x.data_ptr(), stats.data_ptr(),
                          float(self.eps), float(self.momentum), self.mean.data_ptr(), self.var.data_ptr(),
                          self.rstd.data_ptr(), self.running_mean.data_ptr(), self.running_var.data_ptr(),
                          ws.data_ptr(), ws.numel(), st)
        else:
            with K._span("bn_stats", "hbm", lambda: x.numel() * x.element_size()):
                _lib.call("dfx_batchnorm_stats", dt, rows, self.C, x.data_ptr(), stats.data_ptr(), ws.data_ptr(),
                          ws.numel(), st)
            sets = exchange_bn_sets(self.sets, group=self.pg)
            _lib.call("dfx_bn_finalize", self.C, self.world, sets.data_ptr(), float(self.eps), float(self.momentum),
                      self.mean.data_ptr(), self.var.data_ptr(), self.rstd.data_ptr(), self.running_mean.data_ptr(),
                      self.running_var.data_ptr(), st)
        with K._span("bn_act_apply", "hbm", lambda: 2 * x.numel() * x.element_size()):
            _lib.call("dfx_batchnorm_act_apply", dt, rows, self.C, x.data_ptr(), self.mean.data_ptr(),
                      self.rstd.data_ptr(), self.gamma.data_ptr(), self.beta.data_ptr(), self.act, y.data_ptr(), st)
        return y

    def backward(self, dy, dx=None):
        x = self._x
        rows = x.numel() // self.C
        dt, st = K.dfx_dtype(x), K._stream()
        ws = K.WORKSPACE.get(_lib.load().dfx_batchnorm_workspace(rows, self.C))
        dx = torch.empty_like(x) if dx is None else dx
        with K._span("bn_act_bwd_reduce", "hbm", lambda: 2 * x.numel() * x.element_size()):
            # bnsum, and the local parameter gradients dbeta / dgamma straight from the same sums
            _lib.call("dfx_batchnorm_act_bwd_reduce_grads", dt, rows, self.C, dy.data_ptr(), x.data_ptr(),
                      self.mean.data_ptr(), self.rstd.data_ptr(), self.gamma.data_ptr(), self.beta.data_ptr(),
                      self.act, self.bnsum.data_ptr(), self.dbeta.data_ptr(), self.dgamma.data_ptr(),
                      ws.data_ptr(), ws.numel(), st)
        count = float(rows)
        if self.world > 1:  # SyncBN: (sum du, sum du*xhat, count) over ranks; count 0 = read bnsum[2]
            self.bnsum[2].fill_(count)
            allreduce_sum(self.bnsum, group=self.pg)
            count = 0.0
        with K._span("bn_act_bwd_dx", "hbm", lambda: 3 * x.numel() * x.element_size()):
            _lib.call("dfx_batchnorm_act_bwd_dx", dt, rows, self.C, dy.data_ptr(), x.data_ptr(), self.mean.data_ptr(),
                      self.rstd.data_ptr(), self.gamma.data_ptr(), self.beta.data_ptr(), self.act,
                      self.bnsum.data_ptr(), count, dx.data_ptr(), st)
        return dx
