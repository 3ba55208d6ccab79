"""The dfir plugin contract for the B200 fused operators.

``install()`` puts every fused operator of ``registry.FUSED_OPS`` into a live
``dfir`` (the reference package) the way the reference's own operators are
wired, so its interpreter, passes and AD treat them as ordinary operators:

* ``frontend.register_op(OpSpec(...))`` (frontend.py:73-98) with a shape
  ``infer`` and a numpy ``reference``.  The forward references compose the
  reference's own ``reference_apply`` (frontend.py:146-150); the ``...Grad``
  references restate the reference's manual VJP formulas (autodiff.py:1465-1617)
  in float64 and cast back like ``reference_apply`` does (frontend.py:216-218).
* ``lowering.register_lowering(op, program)`` (lowering.py:59-66).  Each program
  replaces the fused node by the chain of registry operators it stands for and
  expands those in place (``lowering.expand``, lowering.py:1045-1074), so only
  native maps and rank-1 Einsum/Reduce nodes remain — ``lower_all``'s
  strictly-decreasing operator-rank rule (lowering.py:1110-1126) holds without
  touching the reference's private rank table.  ``MBConvBlockGrad`` has no
  lowering (the reference itself reverses a depthwise conv only by lowering its
  forward, autodiff.py:1623-1629); ``lower_all`` leaves it as a library node.
* ``autodiff._register_manual(op, build, decline)`` (autodiff.py:1344-1346): the
  VJP of a fused forward op is ONE fused ``...Grad`` library node plus the
  reference's adjoint accumulation (``_Ctx.accumulate``, autodiff.py:681-695).
  A VJP declines (and AD lowers the op instead, autodiff.py:1701-1745) when an
  auxiliary output (the stashed pre-LN sum, the running statistics, ...) carries
  an adjoint.
* ``transforms.register_transformation("fuse_to_b200", ...)``
  (transforms.py:117-120), modelled on ``lift_layernorm`` (transforms.py:792-956):
  it recognises the registry-operator chains of SURVEY.md Appendix B (the BERT
  layer's bias+dropout+residual+LayerNorm, scaled-masked softmax + dropout,
  bias + tanh-GELU; the MBConv dw-conv + BN + swish + SE block; LN/BN + swish)
  and rewrites each into its fused operator.  ``fuse_to_b200(g)`` applies it to
  a fixpoint through ``find_matches``/``apply`` (transforms.py:135-208).

After ``fuse_to_b200`` + ``autodiff.differentiate_graph`` every library node of
a BERT-layer / MBConv training graph is one ``library_eval`` executes on the
GPU (library_eval.py); the interpreter keeps running its own glue maps (adjoint
zero-fill / accumulation, Reshape copies).
"""

from __future__ import annotations

import numpy as np

from .registry import FUSED_OPS

GELU_C0 = 0.044715
GELU_C1 = 0.7978845608028654

_STATE: dict = {}


def _dfir():
    from dfir import autodiff, frontend, ir, lowering, transforms  # noqa: F401

    return frontend, lowering, autodiff, transforms, ir


# ---------------------------------------------------------------------------
# numpy references (float64, cast back to the first input's dtype)


def _f64(*xs):
    return [np.asarray(x, dtype=np.float64) for x in xs]


def _cast(like, *outs):
    dt = np.asarray(like).dtype
    return [np.asarray(o).astype(dt, copy=False) for o in outs]


def _ln_parts(s, eps, axes):
    mu = s.mean(axis=axes, keepdims=True)
    xc = s - mu
    var = (xc * xc).mean(axis=axes, keepdims=True)
    rstd = 1.0 / np.sqrt(var + eps)
    return xc * rstd, rstd


def _ln_vjp(gy, g, xhat, rstd, axes, lead):
    """autodiff.py:1511-1542 (LayerNormalization manual VJP)."""
    dyg = gy * g
    m1 = dyg.mean(axis=axes, keepdims=True)
    m2 = (dyg * xhat).mean(axis=axes, keepdims=True)
    dx = rstd * (dyg - m1 - xhat * m2)
    return dx, (gy * xhat).sum(axis=lead), gy.sum(axis=lead)


def _bn_vjp(gy, g, xhat, rstd, axes, C):
    """autodiff.py:1569-1611 (BatchNormalization manual VJP, channel axis 1)."""
    shp = [1] * gy.ndim
    shp[1] = C
    m1 = gy.mean(axis=axes, keepdims=True)
    m2 = (gy * xhat).mean(axis=axes, keepdims=True)
    dx = g.reshape(shp) * rstd * (gy - m1 - xhat * m2)
    return dx, (gy * xhat).sum(axis=axes), gy.sum(axis=axes)


def _swish_vjp(gy, u):
    """d/du u*sigmoid(u) = sg + u*sg*(1-sg) (symexpr.differentiate of the
    Mul(u, Sigmoid(u)) chain, symexpr.py:672-738)."""
    sg = 1.0 / (1.0 + np.exp(-u))
    return gy * (sg + u * sg * (1.0 - sg))


def _gelu_grad(x):
    u = GELU_C1 * (x + GELU_C0 * x ** 3)
    t = np.tanh(u)
    return 0.5 * (1.0 + t) + 0.5 * x * (1.0 - t * t) * GELU_C1 * (1.0 + 3.0 * GELU_C0 * x * x)


def _references(frontend):
    ra = frontend.reference_apply

    def bdrln(attrs, ins):
        h, b, m, r, g, be = ins
        (s,) = ra("Add", {}, [ra("Mul", {}, [ra("Add", {}, [h, b])[0], m])[0], r])
        (y,) = ra("LayerNormalization", {"epsilon": attrs["epsilon"], "axis": -1}, [s, g, be])
        return [y, s]

    def bdrln_grad(attrs, ins):
        dy, s, g, m = _f64(*ins)
        axes, lead = (s.ndim - 1,), tuple(range(s.ndim - 1))
        xhat, rstd = _ln_parts(s, float(attrs["epsilon"]), axes)
        ds, dg, dbe = _ln_vjp(dy, g, xhat, rstd, axes, lead)
        dh = ds * m
        return _cast(ins[0], ds, dh, dh.sum(axis=lead), dg, dbe)

    def sms(attrs, ins):
        sc, am, dm = ins
        (z,) = ra("Div", {"divisor": attrs["divisor"]}, [sc])
        (p,) = ra("Softmax", {"axis": -1}, [ra("Add", {}, [z, am])[0]])
        return [ra("Mul", {}, [p, dm])[0], p]

    def sms_grad(attrs, ins):
        dpd, p, dm = _f64(*ins)
        gp = dpd * dm  # Mul VJP
        dz = (gp - (gp * p).sum(axis=-1, keepdims=True)) * p  # autodiff.py:1465-1484
        return _cast(ins[0], dz / float(attrs["divisor"]))  # Div VJP

    def bias_gelu(attrs, ins):
        f, b = ins
        (x,) = ra("Add", {}, [f, b])
        c = lambda v: np.asarray(v, dtype=x.dtype)  # noqa: E731
        (x3,) = ra("Pow", {"exponent": 3.0}, [x])
        (t,) = ra("Tanh", {}, [ra("Mul", {}, [ra("Add", {}, [x, ra("Mul", {}, [x3, c(GELU_C0)])[0]])[0],
                                             c(GELU_C1)])[0]])
        (y,) = ra("Mul", {}, [ra("Mul", {}, [x, ra("Add", {}, [t, c(1.0)])[0]])[0], c(0.5)])
        return [y, x]

    def bias_gelu_grad(attrs, ins):
        dy, pre = _f64(*ins)
        dpre = dy * _gelu_grad(pre)
        return _cast(ins[0], dpre, dpre.sum(axis=tuple(range(dpre.ndim - 1))))

    def mbconv(attrs, ins):
        x, wdw, g, b, rm, rv, wr, br, we, be = ins
        N, C = x.shape[:2]
        (z,) = ra("Conv", {"group": C, "strides": attrs["strides"], "pads": attrs["pads"]}, [x, wdw])
        bn, nrm, nrv = ra("BatchNormalization", {"epsilon": attrs["epsilon"], "momentum": attrs["momentum"]},
                          [z, g, b, rm, rv])
        (a,) = ra("Mul", {}, [bn, ra("Sigmoid", {}, [bn])[0]])
        (p,) = ra("Reshape", {"shape": [N, C]}, [ra("GlobalAveragePool", {}, [a])[0]])
        (r,) = ra("Gemm", {"transB": 1}, [p, wr, br])
        (r2,) = ra("Mul", {}, [r, ra("Sigmoid", {}, [r])[0]])
        (e,) = ra("Gemm", {"transB": 1}, [r2, we, be])
        (es,) = ra("Reshape", {"shape": [N, C, 1, 1]}, [ra("Sigmoid", {}, [e])[0]])
        return [ra("Mul", {}, [a, es])[0], nrm, nrv]

    def mbconv_grad(attrs, ins):
        dy, x, wdw, g, b, rm, rv, wr, br, we, be = _f64(*ins)
        N, C, H, W = x.shape
        k = wdw.shape[-1]
        (z,) = ra("Conv", {"group": C, "strides": attrs["strides"], "pads": attrs["pads"]}, [x, wdw])
        axes = (0, 2, 3)
        xhat, rstd = _ln_parts(z, float(attrs["epsilon"]), axes)
        u = xhat * g.reshape(1, C, 1, 1) + b.reshape(1, C, 1, 1)
        sg = 1.0 / (1.0 + np.exp(-u))
        a = u * sg
        pooled = a.mean(axis=(2, 3))
        r = pooled @ wr.T + br
        sr = 1.0 / (1.0 + np.exp(-r))
        r2 = r * sr
        e = r2 @ we.T + be
        s = 1.0 / (1.0 + np.exp(-e))
        # y = a * s[n, c]
        da = dy * s[:, :, None, None]
        ds = (dy * a).sum(axis=(2, 3))
        de = ds * s * (1.0 - s)
        dwe, dbe = de.T @ r2, de.sum(axis=0)
        dr2 = de @ we
        dr = dr2 * (sr + r * sr * (1.0 - sr))
        dwr, dbr = dr.T @ pooled, dr.sum(axis=0)
        da = da + (dr @ wr)[:, :, None, None] / (z.shape[2] * z.shape[3])
        du = _swish_vjp(da, u)
        dz, dg, db = _bn_vjp(du, g, xhat, rstd, axes, C)
        # depthwise conv VJP (the reference differentiates the lowered Conv
        # loop nest, lowering.py:930-1004): scatter-add of dz over the taps
        st = int((attrs["strides"] or [1, 1])[0])
        pt, pl = (attrs["pads"] or [0, 0, 0, 0])[:2]
        xp = np.pad(x, ((0, 0), (0, 0), (pt, pt + k), (pl, pl + k)))
        dxp = np.zeros_like(xp)
        dw = np.zeros_like(wdw)
        Ho, Wo = dz.shape[2:]
        for ky in range(k):
            for kx in range(k):
                win = (slice(None), slice(None), slice(ky, ky + st * Ho, st), slice(kx, kx + st * Wo, st))
                dw[:, 0, ky, kx] = (dz * xp[win]).sum(axis=(0, 2, 3))
                dxp[win] += dz * wdw[None, :, 0, ky, kx, None, None]
        dx = dxp[:, :, pt:pt + H, pl:pl + W]
        return _cast(ins[0], dx, dw, dg, db, dwr, dbr, dwe, dbe)

    def ln_act(attrs, ins):
        x, g, b = ins
        (y,) = ra("LayerNormalization", {"epsilon": attrs["epsilon"], "axis": -1}, [x, g, b])
        if attrs["activation"] == "swish":
            (y,) = ra("Mul", {}, [y, ra("Sigmoid", {}, [y])[0]])
        return [y]

    def ln_act_grad(attrs, ins):
        dy, x, g, b = _f64(*ins)
        axes, lead = (x.ndim - 1,), tuple(range(x.ndim - 1))
        xhat, rstd = _ln_parts(x, float(attrs["epsilon"]), axes)
        du = _swish_vjp(dy, xhat * g + b) if attrs["activation"] == "swish" else dy
        return _cast(ins[0], *_ln_vjp(du, g, xhat, rstd, axes, lead))

    def bn_act(attrs, ins):
        y, nrm, nrv = ra("BatchNormalization", {"epsilon": attrs["epsilon"], "momentum": attrs["momentum"]},
                         list(ins))
        if attrs["activation"] == "swish":
            (y,) = ra("Mul", {}, [y, ra("Sigmoid", {}, [y])[0]])
        return [y, nrm, nrv]

    def bn_act_grad(attrs, ins):
        dy, x, g, b = _f64(*ins)
        C = x.shape[1]
        axes = tuple(a for a in range(x.ndim) if a != 1)
        shp = [1] * x.ndim
        shp[1] = C
        xhat, rstd = _ln_parts(x, float(attrs["epsilon"]), axes)
        du = _swish_vjp(dy, xhat * g.reshape(shp) + b.reshape(shp)) if attrs["activation"] == "swish" else dy
        return _cast(ins[0], *_bn_vjp(du, g, xhat, rstd, axes, C))

    return {
        "BiasDropoutResidualLayerNorm": bdrln, "BiasDropoutResidualLayerNormGrad": bdrln_grad,
        "ScaledMaskedSoftmax": sms, "ScaledMaskedSoftmaxGrad": sms_grad,
        "BiasGelu": bias_gelu, "BiasGeluGrad": bias_gelu_grad,
        "MBConvBlock": mbconv, "MBConvBlockGrad": mbconv_grad,
        "LayerNormAct": ln_act, "LayerNormActGrad": ln_act_grad,
        "BatchNormAct": bn_act, "BatchNormActGrad": bn_act_grad,
    }


# ---------------------------------------------------------------------------
# shape inference  (InferFn = (attrs, in_shapes, in_dtypes) -> [(shape, dtype)])


def _infers(frontend):
    def same(k_out):
        return lambda a, s, d: [(s[0], d[0])] * k_out

    def mbconv(a, s, d):
        conv = frontend.get_op("Conv")
        attrs = frontend.normalize_attrs(conv, {"group": _int(s[0][1]), "strides": a["strides"], "pads": a["pads"]})
        (zs, _), = conv.infer(attrs, [s[0], s[1]], d[:2])
        return [(zs, d[0]), (s[4], d[0]), (s[5], d[0])]

    return {
        "BiasDropoutResidualLayerNorm": same(2),
        "BiasDropoutResidualLayerNormGrad": lambda a, s, d: [(s[1], d[0]), (s[1], d[0]), (s[2], d[0]),
                                                             (s[2], d[0]), (s[2], d[0])],
        "ScaledMaskedSoftmax": same(2),
        "ScaledMaskedSoftmaxGrad": same(1),
        "BiasGelu": same(2),
        "BiasGeluGrad": lambda a, s, d: [(s[1], d[0]), ((s[1][-1],), d[0])],
        "MBConvBlock": mbconv,
        "MBConvBlockGrad": lambda a, s, d: [(s[k], d[0]) for k in (1, 2, 3, 4, 7, 8, 9, 10)],
        "LayerNormAct": same(1),
        "LayerNormActGrad": lambda a, s, d: [(s[1], d[0]), (s[2], d[0]), (s[3], d[0])],
        "BatchNormAct": lambda a, s, d: [(s[0], d[0]), (s[3], d[0]), (s[4], d[0])],
        "BatchNormActGrad": lambda a, s, d: [(s[1], d[0]), (s[2], d[0]), (s[3], d[0])],
    }


# ---------------------------------------------------------------------------
# lowerings: compose registry operators, expand them in place


class _Chain:
    """Builds a chain of registry library nodes inside a lowering program.

    Refs: ``("in", k)`` / ``("out", k)`` are the fused node's connectors,
    ``("c", value)`` a scalar constant container, a plain string a fresh
    transient produced earlier in the chain."""

    def __init__(self, g, state, node, ins, outs):
        self.frontend, self.lowering, _, _, self.ir = _dfir()
        self.g, self.st, self.node = g, state, node
        self.env = {("in", k): (acc, name) for k, (_, acc, name) in enumerate(ins)}
        self.env.update({("out", k): (acc, name) for k, (_, acc, name) in enumerate(outs)})
        self.dtype = g.container(ins[0][2]).dtype
        self.created = []

    def _ref(self, r):
        if isinstance(r, tuple) and r[0] == "c":
            name = self.g.fresh_name(f"{self.node.name}_c")
            self.g.add_container(name, (), self.dtype, "Global", constant=True)
            self.g.constants[name] = np.array(r[1], dtype=self.ir.NUMPY_DTYPES[self.dtype])
            return self.st.add_access(name), name
        return self.env[r]

    def op(self, op, attrs, inputs, outputs):
        fe, ir = self.frontend, self.ir
        attrs = fe.normalize_attrs(op, attrs)
        srcs = [self._ref(r) for r in inputs]
        shapes = [tuple(self.g.container(n).shape) for _, n in srcs]
        dtypes = [self.g.container(n).dtype for _, n in srcs]
        inferred = fe.infer_shapes(op, attrs, shapes, dtypes)
        dsts = []
        for r, (shape, dtype) in zip(outputs, inferred):
            if r not in self.env:
                name = self.g.fresh_name(f"{self.node.name}_{r}")
                self.g.add_container(name, shape, dtype, "Transient")
                self.env[r] = (self.st.add_access(name), name)
            dsts.append(self.env[r])
        nid = self.st.add_node(ir.LibraryNode(op, f"{self.node.name}_{len(self.created)}_{op.lower()}", attrs,
                                              tuple(f"in_{k}" for k in range(len(srcs))),
                                              tuple(f"out_{k}" for k in range(len(dsts)))))
        for k, (acc, name) in enumerate(srcs):
            self.st.add_edge(acc, None, nid, f"in_{k}", ir.Memlet(name, ir.Subset.full(self.g.container(name).shape)))
        for k, (acc, name) in enumerate(dsts):
            self.st.add_edge(nid, f"out_{k}", acc, None, ir.Memlet(name, ir.Subset.full(self.g.container(name).shape)))
        self.created.append(nid)
        return outputs[0]

    def expand(self):
        for nid in self.created:
            node = self.st.nodes.get(nid)
            if node is not None and self.lowering.has_lowering(node.op):
                self.lowering.expand(self.g, self.st, nid, validate=False)
        return True


def _int(e):
    """Concrete value of a shape expression (symexpr.Const)."""
    return int(getattr(e, "value", e))


def _lower_bdrln(ch, attrs, rank):
    ch.op("Add", {}, [("in", 0), ("in", 1)], ["hb"])
    ch.op("Mul", {}, ["hb", ("in", 2)], ["hd"])
    ch.op("Add", {}, ["hd", ("in", 3)], [("out", 1)])
    ch.op("LayerNormalization", {"axis": -1, "epsilon": attrs["epsilon"]}, [("out", 1), ("in", 4), ("in", 5)],
          [("out", 0)])


def _ln_backward_chain(ch, gy, x, g, eps, axes, lead, outs, scale_shape=None):
    """Manual LayerNorm/BatchNorm VJP formulas (autodiff.py:1500-1611) as
    registry operators; outs = (dx, dgamma, dbeta) refs (None = skip)."""
    mean = {"axes": list(axes), "keepdims": 1}
    ch.op("ReduceMean", mean, [x], ["mu"])
    ch.op("Sub", {}, [x, "mu"], ["xc"])
    ch.op("Mul", {}, ["xc", "xc"], ["sq"])
    ch.op("ReduceMean", mean, ["sq"], ["var"])
    ch.op("Add", {}, ["var", ("c", eps)], ["ve"])
    ch.op("Sqrt", {}, ["ve"], ["sd"])
    ch.op("Div", {}, ["xc", "sd"], ["xhat"])
    gs = g
    if scale_shape is not None:
        ch.op("Reshape", {"shape": scale_shape}, [g], ["g_b"])
        gs = "g_b"
    ch.op("Mul", {}, [gy, gs], ["dyg"])
    ch.op("ReduceMean", mean, ["dyg"], ["m1"])
    ch.op("Mul", {}, ["dyg", "xhat"], ["dygx"])
    ch.op("ReduceMean", mean, ["dygx"], ["m2"])
    ch.op("Sub", {}, ["dyg", "m1"], ["t1"])
    ch.op("Mul", {}, ["xhat", "m2"], ["t2"])
    ch.op("Sub", {}, ["t1", "t2"], ["t3"])
    ch.op("Div", {}, ["t3", "sd"], [outs[0]])
    red = {"axes": list(lead), "keepdims": 0}
    if outs[1] is not None:
        ch.op("Mul", {}, [gy, "xhat"], ["gx"])
        ch.op("ReduceSum", red, ["gx"], [outs[1]])
    if outs[2] is not None:
        ch.op("ReduceSum", red, [gy], [outs[2]])


def _lower_bdrln_grad(ch, attrs, rank):
    lead = list(range(rank - 1))
    _ln_backward_chain(ch, ("in", 0), ("in", 1), ("in", 2), float(attrs["epsilon"]), [rank - 1], lead,
                       (("out", 0), ("out", 3), ("out", 4)))
    ch.op("Mul", {}, [("out", 0), ("in", 3)], [("out", 1)])
    ch.op("ReduceSum", {"axes": lead, "keepdims": 0}, [("out", 1)], [("out", 2)])


def _lower_sms(ch, attrs, rank):
    ch.op("Div", {"divisor": attrs["divisor"]}, [("in", 0)], ["z"])
    ch.op("Add", {}, ["z", ("in", 1)], ["za"])
    ch.op("Softmax", {"axis": -1}, ["za"], [("out", 1)])
    ch.op("Mul", {}, [("out", 1), ("in", 2)], [("out", 0)])


def _lower_sms_grad(ch, attrs, rank):
    ch.op("Mul", {}, [("in", 0), ("in", 2)], ["gp"])
    ch.op("Mul", {}, ["gp", ("in", 1)], ["gpp"])
    ch.op("ReduceSum", {"axes": [rank - 1], "keepdims": 1}, ["gpp"], ["tot"])
    ch.op("Sub", {}, ["gp", "tot"], ["cen"])
    ch.op("Mul", {}, ["cen", ("in", 1)], ["dz"])
    ch.op("Div", {"divisor": attrs["divisor"]}, ["dz"], [("out", 0)])


def _lower_bias_gelu(ch, attrs, rank):
    x = ("out", 1)
    ch.op("Add", {}, [("in", 0), ("in", 1)], [x])
    ch.op("Pow", {"exponent": 3.0}, [x], ["x3"])
    ch.op("Mul", {}, ["x3", ("c", GELU_C0)], ["t1"])
    ch.op("Add", {}, [x, "t1"], ["t2"])
    ch.op("Mul", {}, ["t2", ("c", GELU_C1)], ["t3"])
    ch.op("Tanh", {}, ["t3"], ["t4"])
    ch.op("Add", {}, ["t4", ("c", 1.0)], ["t5"])
    ch.op("Mul", {}, [x, "t5"], ["t6"])
    ch.op("Mul", {}, ["t6", ("c", 0.5)], [("out", 0)])


def _lower_bias_gelu_grad(ch, attrs, rank):
    x = ("in", 1)
    ch.op("Mul", {}, [x, x], ["x2"])
    ch.op("Mul", {}, ["x2", x], ["x3"])
    ch.op("Mul", {}, ["x3", ("c", GELU_C0)], ["u0"])
    ch.op("Add", {}, [x, "u0"], ["u1"])
    ch.op("Mul", {}, ["u1", ("c", GELU_C1)], ["u"])
    ch.op("Tanh", {}, ["u"], ["t"])
    ch.op("Add", {}, ["t", ("c", 1.0)], ["a0"])
    ch.op("Mul", {}, ["a0", ("c", 0.5)], ["a"])
    ch.op("Mul", {}, ["t", "t"], ["tt"])
    ch.op("Sub", {}, [("c", 1.0), "tt"], ["sech2"])
    ch.op("Mul", {}, ["x2", ("c", 3.0 * GELU_C0)], ["d0"])
    ch.op("Add", {}, ["d0", ("c", 1.0)], ["d1"])
    ch.op("Mul", {}, ["d1", ("c", 0.5 * GELU_C1)], ["du"])
    ch.op("Mul", {}, [x, "sech2"], ["b0"])
    ch.op("Mul", {}, ["b0", "du"], ["b"])
    ch.op("Add", {}, ["a", "b"], ["dg"])
    ch.op("Mul", {}, [("in", 0), "dg"], [("out", 0)])
    ch.op("ReduceSum", {"axes": list(range(rank - 1)), "keepdims": 0}, [("out", 0)], [("out", 1)])


def _swish_chain(ch, u, out):
    ch.op("Sigmoid", {}, [u], [f"{u}_sg" if isinstance(u, str) else "u_sg"])
    ch.op("Mul", {}, [u, f"{u}_sg" if isinstance(u, str) else "u_sg"], [out])


def _swish_grad_chain(ch, gy, u, out):
    """gy * (sg + u*sg*(1-sg))."""
    ch.op("Sigmoid", {}, [u], ["sw_sg"])
    ch.op("Sub", {}, [("c", 1.0), "sw_sg"], ["sw_1m"])
    ch.op("Mul", {}, [u, "sw_sg"], ["sw_us"])
    ch.op("Mul", {}, ["sw_us", "sw_1m"], ["sw_t"])
    ch.op("Add", {}, ["sw_sg", "sw_t"], ["sw_d"])
    ch.op("Mul", {}, [gy, "sw_d"], [out])


def _lower_mbconv(ch, attrs, rank):
    x = ("in", 0)
    N, C = (_int(d) for d in ch.g.container(ch.env[x][1]).shape[:2])
    ch.op("Conv", {"group": C, "strides": attrs["strides"], "pads": attrs["pads"]}, [x, ("in", 1)], ["z"])
    ch.op("BatchNormalization", {"epsilon": attrs["epsilon"], "momentum": attrs["momentum"]},
          ["z", ("in", 2), ("in", 3), ("in", 4), ("in", 5)], ["bn", ("out", 1), ("out", 2)])
    _swish_chain(ch, "bn", "a")
    ch.op("GlobalAveragePool", {}, ["a"], ["pool"])
    ch.op("Reshape", {"shape": [N, C]}, ["pool"], ["p2"])
    ch.op("Gemm", {"transB": 1}, ["p2", ("in", 6), ("in", 7)], ["r"])
    _swish_chain(ch, "r", "r2")
    ch.op("Gemm", {"transB": 1}, ["r2", ("in", 8), ("in", 9)], ["e"])
    ch.op("Sigmoid", {}, ["e"], ["es"])
    ch.op("Reshape", {"shape": [N, C, 1, 1]}, ["es"], ["es4"])
    ch.op("Mul", {}, ["a", "es4"], [("out", 0)])


def _lower_ln_act(ch, attrs, rank):
    if attrs["activation"] == "swish":
        ch.op("LayerNormalization", {"axis": -1, "epsilon": attrs["epsilon"]}, [("in", 0), ("in", 1), ("in", 2)],
              ["ln"])
        _swish_chain(ch, "ln", ("out", 0))
    else:
        ch.op("LayerNormalization", {"axis": -1, "epsilon": attrs["epsilon"]}, [("in", 0), ("in", 1), ("in", 2)],
              [("out", 0)])


def _lower_ln_act_grad(ch, attrs, rank):
    gy = ("in", 0)
    if attrs["activation"] == "swish":
        ch.op("LayerNormalization", {"axis": -1, "epsilon": attrs["epsilon"]}, [("in", 1), ("in", 2), ("in", 3)],
              ["u"])
        _swish_grad_chain(ch, gy, "u", "du")
        gy = "du"
    _ln_backward_chain(ch, gy, ("in", 1), ("in", 2), float(attrs["epsilon"]), [rank - 1], list(range(rank - 1)),
                       (("out", 0), ("out", 1), ("out", 2)))


def _lower_bn_act(ch, attrs, rank):
    bn_out = "bn" if attrs["activation"] == "swish" else ("out", 0)
    ch.op("BatchNormalization", {"epsilon": attrs["epsilon"], "momentum": attrs["momentum"]},
          [("in", k) for k in range(5)], [bn_out, ("out", 1), ("out", 2)])
    if attrs["activation"] == "swish":
        _swish_chain(ch, "bn", ("out", 0))


def _lower_bn_act_grad(ch, attrs, rank):
    axes = [a for a in range(rank) if a != 1]
    C = _int(ch.g.container(ch.env[("in", 1)][1]).shape[1])
    bshape = [C] + [1] * (rank - 2)
    gy = ("in", 0)
    if attrs["activation"] == "swish":
        # u = BN(x) with batch statistics, recomputed as the reference's VJP does
        mean = {"axes": axes, "keepdims": 1}
        ch.op("ReduceMean", mean, [("in", 1)], ["fmu"])
        ch.op("Sub", {}, [("in", 1), "fmu"], ["fxc"])
        ch.op("Mul", {}, ["fxc", "fxc"], ["fsq"])
        ch.op("ReduceMean", mean, ["fsq"], ["fvar"])
        ch.op("Add", {}, ["fvar", ("c", float(attrs["epsilon"]))], ["fve"])
        ch.op("Sqrt", {}, ["fve"], ["fsd"])
        ch.op("Div", {}, ["fxc", "fsd"], ["fxh"])
        ch.op("Reshape", {"shape": bshape}, [("in", 2)], ["fg"])
        ch.op("Reshape", {"shape": bshape}, [("in", 3)], ["fb"])
        ch.op("Mul", {}, ["fxh", "fg"], ["fu0"])
        ch.op("Add", {}, ["fu0", "fb"], ["u"])
        _swish_grad_chain(ch, gy, "u", "du")
        gy = "du"
    _ln_backward_chain(ch, gy, ("in", 1), ("in", 2), float(attrs["epsilon"]), axes, axes,
                       (("out", 0), ("out", 1), ("out", 2)), scale_shape=bshape)


_LOWERINGS = {
    "BiasDropoutResidualLayerNorm": _lower_bdrln,
    "BiasDropoutResidualLayerNormGrad": _lower_bdrln_grad,
    "ScaledMaskedSoftmax": _lower_sms,
    "ScaledMaskedSoftmaxGrad": _lower_sms_grad,
    "BiasGelu": _lower_bias_gelu,
    "BiasGeluGrad": _lower_bias_gelu_grad,
    "MBConvBlock": _lower_mbconv,
    "LayerNormAct": _lower_ln_act,
    "LayerNormActGrad": _lower_ln_act_grad,
    "BatchNormAct": _lower_bn_act,
    "BatchNormActGrad": _lower_bn_act_grad,
}


def _program(builder):
    """A lowering program (lowering.py:1045-1074 calling convention)."""

    def program(g, state, nid, node, ins, outs):
        for e in list(state.in_edges(nid)) + list(state.out_edges(nid)):
            state.remove_edge(e)
        state.remove_node(nid)
        ch = _Chain(g, state, node, ins, outs)
        builder(ch, node.attrs, len(g.container(ins[0][2]).shape))
        return ch.expand()

    return program


# ---------------------------------------------------------------------------
# manual VJPs: one fused ...Grad node + the reference's adjoint accumulation


def _acc(ctx, pairs):
    for src, target, wanted in pairs:
        if wanted:
            ctx.accumulate(src, target)


def _bwd_bdrln(ctx, node, ins, outs, wanted):
    gy = ctx.adj.get(outs[0])
    if gy is None:
        return
    h, b, m, r, gm, be = ins
    for n in (outs[1], gm, m):
        ctx.ensure_value(n)
    ds, dh, db, dg, dbe = ctx.lib("BiasDropoutResidualLayerNormGrad", {"epsilon": node.attrs["epsilon"]},
                                  [gy, outs[1], gm, m], "bdrln")
    _acc(ctx, [(ds, r, wanted[3]), (dh, h, wanted[0]), (db, b, wanted[1]), (dg, gm, wanted[4]),
               (dbe, be, wanted[5])])
    if wanted[2]:  # d mask = ds * (h + bias)
        ctx.ensure_value(h)
        ctx.ensure_value(b)
        hb = ctx.lib("Add", {}, [h, b], "bdrln_hb")[0]
        ctx.accumulate(ctx.lib("Mul", {}, [ds, hb], "bdrln_dm")[0], m)


def _decline_bdrln(g, node, ins, outs, outs_adjointed):
    if outs_adjointed[1]:
        return "the pre-LayerNorm sum output carries an adjoint"
    s = tuple(g.container(ins[0]).shape)
    if tuple(g.container(ins[3]).shape) != s or tuple(g.container(ins[2]).shape) != s:
        return "broadcast residual / mask operands are reversed by lowering"
    return None


def _bwd_sms(ctx, node, ins, outs, wanted):
    gpd = ctx.adj.get(outs[0])
    if gpd is None:
        return
    sc, am, dm = ins
    ctx.ensure_value(outs[1])
    ctx.ensure_value(dm)
    (dsc,) = ctx.lib("ScaledMaskedSoftmaxGrad", {"divisor": node.attrs["divisor"]}, [gpd, outs[1], dm], "sms")
    _acc(ctx, [(dsc, sc, wanted[0])])
    if wanted[1]:  # d add_mask = unbroadcast(dscores * divisor)
        ctx.accumulate(ctx.unbroadcast(ctx.scale(dsc, float(node.attrs["divisor"]), "sms_dam"),
                                       ctx.g.container(am).shape), am)
    if wanted[2]:  # d drop_mask = gpd * p
        ctx.accumulate(ctx.lib("Mul", {}, [gpd, outs[1]], "sms_ddm")[0], dm)


def _decline_sms(g, node, ins, outs, outs_adjointed):
    if outs_adjointed[1]:
        return "the un-dropped probabilities carry an adjoint"
    if tuple(g.container(ins[2]).shape) != tuple(g.container(ins[0]).shape):
        return "a broadcast dropout mask is reversed by lowering"
    return None


def _bwd_bias_gelu(ctx, node, ins, outs, wanted):
    gy = ctx.adj.get(outs[0])
    if gy is None:
        return
    ctx.ensure_value(outs[1])
    dpre, db = ctx.lib("BiasGeluGrad", {}, [gy, outs[1]], "bgelu")
    _acc(ctx, [(dpre, ins[0], wanted[0]), (db, ins[1], wanted[1])])


def _decline_bias_gelu(g, node, ins, outs, outs_adjointed):
    if outs_adjointed[1]:
        return "the pre-activation output carries an adjoint"
    return None


def _bwd_mbconv(ctx, node, ins, outs, wanted):
    gy = ctx.adj.get(outs[0])
    if gy is None:
        return
    for n in ins:
        ctx.ensure_value(n)
    attrs = {k: node.attrs[k] for k in ("strides", "pads", "epsilon", "momentum")}
    grads = ctx.lib("MBConvBlockGrad", attrs, [gy] + list(ins), "mbconv")
    targets = [0, 1, 2, 3, 6, 7, 8, 9]  # x, w_dw, gamma, beta, w_r, b_r, w_e, b_e
    _acc(ctx, [(gd, ins[k], wanted[k]) for gd, k in zip(grads, targets)])


def _decline_running_stats(g, node, ins, outs, outs_adjointed):
    if any(outs_adjointed[1:]):
        return "adjoints of the running-statistic outputs require lowering"
    return None


def _bwd_ln_act(ctx, node, ins, outs, wanted):
    gy = ctx.adj.get(outs[0])
    if gy is None:
        return
    for n in ins:
        ctx.ensure_value(n)
    dx, dg, db = ctx.lib("LayerNormActGrad", dict(node.attrs), [gy] + list(ins), "lnact")
    _acc(ctx, [(dx, ins[0], wanted[0]), (dg, ins[1], wanted[1]), (db, ins[2], wanted[2])])


def _bwd_bn_act(ctx, node, ins, outs, wanted):
    gy = ctx.adj.get(outs[0])
    if gy is None:
        return
    for n in ins[:3]:
        ctx.ensure_value(n)
    attrs = {"epsilon": node.attrs["epsilon"], "activation": node.attrs["activation"]}
    dx, dg, db = ctx.lib("BatchNormActGrad", attrs, [gy] + list(ins[:3]), "bnact")
    _acc(ctx, [(dx, ins[0], wanted[0]), (dg, ins[1], wanted[1]), (db, ins[2], wanted[2])])


_VJPS = {
    "BiasDropoutResidualLayerNorm": (_bwd_bdrln, _decline_bdrln),
    "ScaledMaskedSoftmax": (_bwd_sms, _decline_sms),
    "BiasGelu": (_bwd_bias_gelu, _decline_bias_gelu),
    "MBConvBlock": (_bwd_mbconv, _decline_running_stats),
    "LayerNormAct": (_bwd_ln_act, None),
    "BatchNormAct": (_bwd_bn_act, _decline_running_stats),
}


# ---------------------------------------------------------------------------
# fuse_to_b200: pattern finder + applier (transforms.py:117-208 contract)


class _View:
    """Read-only dataflow view of one state (one access node per container,
    as ``frontend.build_graph`` produces, frontend.py:1006-1011)."""

    def __init__(self, g, st):
        _, _, _, _, ir = _dfir()
        self.g, self.st, self.ir = g, st, ir
        self.producer, self.consumers = {}, {}
        self.ins, self.outs = {}, {}
        for nid, n in st.nodes.items():
            if isinstance(n, ir.LibraryNode):
                ins = {e.dst_conn: st.nodes[e.src].data for e in st.in_edges(nid)}
                outs = {e.src_conn: st.nodes[e.dst].data for e in st.out_edges(nid)}
                self.ins[nid] = [ins.get(c) for c in n.in_conns]
                self.outs[nid] = [outs.get(c) for c in n.out_conns]
                for name in self.ins[nid]:
                    self.consumers.setdefault(name, []).append(nid)
                for name in self.outs[nid]:
                    self.producer[name] = nid

    def node(self, nid):
        return self.st.nodes[nid]

    def prod(self, name, op):
        nid = self.producer.get(name)
        if nid is None or self.node(nid).op != op:
            return None
        return nid

    def only_consumer(self, name, op=None):
        cs = self.consumers.get(name, [])
        if len(cs) != 1 or self.g.container(name).storage == "Global":
            return None
        if op is not None and self.node(cs[0]).op != op:
            return None
        return cs[0]

    def shape(self, name):
        return tuple(self.g.container(name).shape)

    def const(self, name):
        arr = self.g.constants.get(name)
        if arr is None or arr.size != 1:
            return None
        return float(arr.reshape(-1)[0])

    def other(self, nid, name):
        ins = self.ins[nid]
        if len(ins) != 2 or name not in ins:
            return None
        return ins[1] if ins[0] == name else ins[0]


def _eq(a, b):
    from dfir.ir import as_expr
    from dfir.symexpr import expr_equal

    return len(a) == len(b) and all(expr_equal(as_expr(x), as_expr(y)) for x, y in zip(a, b))


def _match_bdrln(v, ln):
    """Add(h, bias) -> Mul(., mask) -> Add(., residual) -> LayerNormalization(last axis)."""
    node = v.node(ln)
    x, gamma = v.ins[ln][0], v.ins[ln][1]
    beta = v.ins[ln][2] if len(v.ins[ln]) == 3 else None
    rank = len(v.shape(x))
    if beta is None or int(node.attrs.get("axis", -1)) % rank != rank - 1:
        return None
    add2 = v.prod(x, "Add")
    if add2 is None:
        return None
    for t2 in v.ins[add2]:
        mul = v.prod(t2, "Mul")
        if mul is None or v.only_consumer(t2) != add2:
            continue
        res = v.other(add2, t2)
        for t1 in v.ins[mul]:
            add1 = v.prod(t1, "Add")
            if add1 is None or v.only_consumer(t1) != mul:
                continue
            mask = v.other(mul, t1)
            for h in v.ins[add1]:
                bias = v.other(add1, h)
                if bias is None or not _eq(v.shape(h), v.shape(x)) or len(v.shape(bias)) != 1 \
                        or not _eq(v.shape(bias), v.shape(x)[-1:]) or not _eq(v.shape(mask), v.shape(x)) \
                        or not _eq(v.shape(res), v.shape(x)):
                    continue
                return {"kind": "bdrln", "remove": [add1, mul, add2, ln], "tmp": [t1, t2],
                        "op": "BiasDropoutResidualLayerNorm", "attrs": {"epsilon": float(node.attrs["epsilon"])},
                        "ins": [h, bias, mask, res, gamma, beta], "outs": [v.outs[ln][0], x]}
    return None


def _match_sms(v, sm):
    """Div(scores; divisor) -> Add(., add_mask) -> Softmax(last axis) -> Mul(., drop_mask)."""
    node = v.node(sm)
    za = v.ins[sm][0]
    rank = len(v.shape(za))
    if int(node.attrs.get("axis", -1)) % rank != rank - 1:
        return None
    p = v.outs[sm][0]
    add = v.prod(za, "Add")
    if add is None or v.only_consumer(za) != sm:
        return None
    for z in v.ins[add]:
        div = v.prod(z, "Div")
        if div is None or v.only_consumer(z) != add or len(v.ins[div]) != 1:
            continue
        am = v.other(add, z)
        muls = [c for c in v.consumers.get(p, []) if v.node(c).op == "Mul"]
        for mul in muls:
            dm = v.other(mul, p)
            if dm is None or not _eq(v.shape(dm), v.shape(za)):
                continue
            return {"kind": "sms", "remove": [div, add, sm, mul], "tmp": [z, za], "op": "ScaledMaskedSoftmax",
                    "attrs": {"divisor": float(v.node(div).attrs["divisor"])},
                    "ins": [v.ins[div][0], am, dm], "outs": [v.outs[mul][0], p]}
    return None


def _match_gelu(v, x):
    """The tanh-GELU chain of SURVEY.md Appendix B on container x:
    Pow(x,3) -> Mul(c0) -> Add(x,.) -> Mul(c1) -> Tanh -> Add(1) -> Mul(x,.) -> Mul(0.5),
    with x = Add(f, bias) or x = Gemm(A, W, bias)."""
    cs = v.consumers.get(x, [])
    if len(cs) != 3:
        return None
    pw = next((c for c in cs if v.node(c).op == "Pow"), None)
    if pw is None or v.node(pw).attrs.get("exponent") != 3.0 or len(v.ins[pw]) != 1:
        return None
    chain = [pw]

    def step(name, op, const=None, other=None):
        nid = v.only_consumer(name, op)
        if nid is None:
            return None
        o = v.other(nid, name)
        if const is not None and (o is None or v.const(o) is None or abs(v.const(o) - const) > 1e-6 * max(1.0, abs(const))):
            return None
        if other is not None and o != other:
            return None
        chain.append(nid)
        return v.outs[nid][0]

    t = step(v.outs[pw][0], "Mul", const=GELU_C0)
    t = t and step(t, "Add", other=x)
    t = t and step(t, "Mul", const=GELU_C1)
    if t:
        nid = v.only_consumer(t, "Tanh")
        t = None if nid is None else v.outs[nid][0]
        if t:
            chain.append(nid)
    t = t and step(t, "Add", const=1.0)
    t = t and step(t, "Mul", other=x)
    y = t and step(t, "Mul", const=0.5)
    if not y or set(cs) != {chain[0], chain[2], chain[6]}:
        return None
    tmp = [v.outs[n][0] for n in chain[:-1]]
    consts = [v.other(chain[k], tmp[k - 1]) for k in (1, 3, 5, 7)]
    rank = len(v.shape(x))
    add = v.prod(x, "Add")
    if add is not None:
        for f in v.ins[add]:
            b = v.other(add, f)
            if b is not None and _eq(v.shape(f), v.shape(x)) and _eq(v.shape(b), v.shape(x)[rank - 1:]):
                return {"kind": "gelu", "remove": [add] + chain, "tmp": tmp, "consts": consts, "op": "BiasGelu",
                        "attrs": {}, "ins": [f, b], "outs": [y, x]}
    gemm = v.prod(x, "Gemm")
    if gemm is not None and len(v.ins[gemm]) == 3 and float(v.node(gemm).attrs.get("beta", 1.0)) == 1.0 \
            and rank == 2 and _eq(v.shape(v.ins[gemm][2]), v.shape(x)[1:]):
        return {"kind": "gelu_gemm", "remove": chain, "tmp": tmp, "consts": consts, "op": "BiasGelu",
                "attrs": {}, "gemm": gemm, "ins": [None, v.ins[gemm][2]], "outs": [y, x]}
    return None


def _match_swish(v, u):
    """Mul(u, Sigmoid(u)) with u consumed only by that pair; returns (sig, mul, out)."""
    cs = v.consumers.get(u, [])
    if len(cs) != 2 or v.g.container(u).storage == "Global":
        return None
    sig = next((c for c in cs if v.node(c).op == "Sigmoid"), None)
    mul = next((c for c in cs if v.node(c).op == "Mul"), None)
    if sig is None or mul is None:
        return None
    s = v.outs[sig][0]
    if v.only_consumer(s) != mul or sorted(v.ins[mul]) != sorted([u, s]):
        return None
    return sig, mul, v.outs[mul][0]


def _match_mbconv(v, conv):
    """Conv(group=C, 3x3) -> BatchNormalization -> swish -> GlobalAveragePool -> Reshape
    -> Gemm -> swish -> Gemm -> Sigmoid -> Reshape -> Mul (SURVEY.md:512-514)."""
    node = v.node(conv)
    if len(v.ins[conv]) != 2:
        return None
    x, wdw = v.ins[conv]
    xs, ws = v.shape(x), v.shape(wdw)
    if len(xs) != 4 or len(ws) != 4 or int(node.attrs.get("group", 1)) != _int(xs[1]) or _int(ws[1]) != 1:
        return None
    N, C = xs[0], xs[1]
    z = v.outs[conv][0]
    bn = v.only_consumer(z, "BatchNormalization")
    if bn is None or len(v.outs[bn]) != 3:
        return None
    u = v.outs[bn][0]
    sw = _match_swish(v, u)
    if sw is None:
        return None
    a = sw[2]
    ca = v.consumers.get(a, [])
    if len(ca) != 2 or v.g.container(a).storage == "Global":
        return None
    gap = next((c for c in ca if v.node(c).op == "GlobalAveragePool"), None)
    fin = next((c for c in ca if v.node(c).op == "Mul"), None)
    if gap is None or fin is None:
        return None
    rs1 = v.only_consumer(v.outs[gap][0], "Reshape")
    if rs1 is None:
        return None
    g1 = v.only_consumer(v.outs[rs1][0], "Gemm")
    if g1 is None or len(v.ins[g1]) != 3 or v.ins[g1][0] != v.outs[rs1][0] or not v.node(g1).attrs.get("transB") \
            or v.node(g1).attrs.get("transA") or float(v.node(g1).attrs.get("alpha", 1)) != 1 \
            or float(v.node(g1).attrs.get("beta", 1)) != 1:
        return None
    sw2 = _match_swish(v, v.outs[g1][0])
    if sw2 is None:
        return None
    g2 = v.only_consumer(sw2[2], "Gemm")
    if g2 is None or len(v.ins[g2]) != 3 or v.ins[g2][0] != sw2[2] or not v.node(g2).attrs.get("transB") \
            or v.node(g2).attrs.get("transA") or float(v.node(g2).attrs.get("alpha", 1)) != 1 \
            or float(v.node(g2).attrs.get("beta", 1)) != 1:
        return None
    sg = v.only_consumer(v.outs[g2][0], "Sigmoid")
    rs2 = sg is not None and v.only_consumer(v.outs[sg][0], "Reshape")
    if not rs2 or v.only_consumer(v.outs[rs2][0]) != fin or v.other(fin, v.outs[rs2][0]) != a:
        return None
    if not _eq(v.shape(v.outs[rs1][0]), (N, C)) or not _eq(v.shape(v.outs[rs2][0]), (N, C, 1, 1)):
        return None
    bnn = v.node(bn)
    nodes = [conv, bn, sw[0], sw[1], gap, rs1, g1, sw2[0], sw2[1], g2, sg, rs2, fin]
    tmp = [z, u, v.outs[sw[0]][0], a, v.outs[gap][0], v.outs[rs1][0], v.outs[g1][0], v.outs[sw2[0]][0], sw2[2],
           v.outs[g2][0], v.outs[sg][0], v.outs[rs2][0]]
    return {"kind": "mbconv", "remove": nodes, "tmp": tmp, "op": "MBConvBlock",
            "attrs": {"strides": node.attrs.get("strides"), "pads": node.attrs.get("pads"),
                      "epsilon": float(bnn.attrs["epsilon"]), "momentum": float(bnn.attrs["momentum"])},
            "ins": [x, wdw] + v.ins[bn][1:5] + v.ins[g1][1:3] + v.ins[g2][1:3],
            "outs": [v.outs[fin][0], v.outs[bn][1], v.outs[bn][2]]}


def _match_norm_act(v, nid):
    node = v.node(nid)
    if node.op == "LayerNormalization":
        x = v.ins[nid][0]
        rank = len(v.shape(x))
        if len(v.ins[nid]) != 3 or int(node.attrs.get("axis", -1)) % rank != rank - 1:
            return None
        sw = _match_swish(v, v.outs[nid][0])
        if sw is None:
            return None
        return {"kind": "ln_act", "remove": [nid, sw[0], sw[1]], "tmp": [v.outs[nid][0], v.outs[sw[0]][0]],
                "op": "LayerNormAct", "attrs": {"epsilon": float(node.attrs["epsilon"]), "activation": "swish"},
                "ins": list(v.ins[nid]), "outs": [sw[2]]}
    if node.op == "BatchNormalization" and len(v.outs[nid]) == 3:
        sw = _match_swish(v, v.outs[nid][0])
        if sw is None:
            return None
        return {"kind": "bn_act", "remove": [nid, sw[0], sw[1]], "tmp": [v.outs[nid][0], v.outs[sw[0]][0]],
                "op": "BatchNormAct", "attrs": {"epsilon": float(node.attrs["epsilon"]),
                                                "momentum": float(node.attrs["momentum"]), "activation": "swish"},
                "ins": list(v.ins[nid]), "outs": [sw[2]] + v.outs[nid][1:]}
    return None


_PRIORITY = ["mbconv", "bdrln", "sms", "gelu", "gelu_gemm", "ln_act", "bn_act"]


def _find_fuse(g) -> list:
    _, _, _, _, ir = _dfir()
    found = []
    for st in g.states:
        v = _View(g, st)
        cands = []
        for nid in st.topological():
            n = st.nodes[nid]
            if isinstance(n, ir.AccessNode):
                m = _match_gelu(v, n.data)
                if m:
                    cands.append(m)
                continue
            if not isinstance(n, ir.LibraryNode):
                continue
            m = {"LayerNormalization": _match_bdrln, "Softmax": _match_sms, "Conv": _match_mbconv}.get(n.op)
            m = m(v, nid) if m else None
            if m:
                cands.append(m)
            m = _match_norm_act(v, nid)
            if m:
                cands.append(m)
        cands.sort(key=lambda m: _PRIORITY.index(m["kind"]))
        taken = set()
        for m in cands:
            touched = set(m["remove"]) | ({m["gemm"]} if "gemm" in m else set())
            if touched & taken:
                continue
            taken |= touched
            found.append({
                "nodes": [[st.name, int(n)] for n in m["remove"]],
                "certificate": f"the {len(m['remove'])}-node registry chain is exactly {m['op']} "
                               f"(registry.py FUSED_OPS 'replaces'); its intermediates have no other consumer",
                "description": f"replace the {m['kind']} chain producing {m['outs'][0]!r} with one {m['op']} node",
                "payload": {k: m[k] for k in ("kind", "op", "attrs", "ins", "outs", "tmp")}
                | ({"gemm": int(m["gemm"])} if "gemm" in m else {}) | ({"consts": m["consts"]} if "consts" in m else {}),
            })
    return found


def _apply_fuse(g, match):
    frontend, _, _, _, ir = _dfir()
    st = next(s for s in g.states if s.name == match.nodes[0][0])
    p = match.payload
    for _, nid in match.nodes:
        st.remove_node(nid)

    def access(name):
        for nid, n in sorted(st.nodes.items()):
            if isinstance(n, ir.AccessNode) and n.data == name:
                return nid
        return st.add_access(name)

    def memlet(name):
        return ir.Memlet(name, ir.Subset.full(g.container(name).shape))

    ins = list(p["ins"])
    if p["kind"] == "gelu_gemm":
        # Gemm(A, W, bias) -> Gemm(A, W) + BiasGelu(., bias): the bias moves
        # into the fused epilogue.
        gid = p["gemm"]
        gnode = st.nodes[gid]
        x = p["outs"][1]
        for e in list(st.in_edges(gid)):
            if e.dst_conn == gnode.in_conns[2]:
                st.remove_edge(e)
        for e in list(st.out_edges(gid)):
            st.remove_edge(e)
        gnode.in_conns = gnode.in_conns[:2]
        f = g.fresh_name(x + "_nobias")
        g.add_container(f, g.container(x).shape, g.container(x).dtype, "Transient")
        st.add_edge(gid, gnode.out_conns[0], st.add_access(f), None, memlet(f))
        ins[0] = f
    attrs = frontend.normalize_attrs(frontend.get_op(p["op"]), p["attrs"])
    nid = st.add_node(ir.LibraryNode(p["op"], g.fresh_name(p["op"].lower()), attrs,
                                     tuple(f"in_{k}" for k in range(len(ins))),
                                     tuple(f"out_{k}" for k in range(len(p["outs"])))))
    for k, name in enumerate(ins):
        st.add_edge(access(name), None, nid, f"in_{k}", memlet(name))
    for k, name in enumerate(p["outs"]):
        st.add_edge(nid, f"out_{k}", access(name), None, memlet(name))
    dead = [t for t in p["tmp"] if t not in p["outs"]] + list(p.get("consts", []))
    for aid in sorted(nid for nid, n in st.nodes.items()
                      if isinstance(n, ir.AccessNode) and n.data in dead and st.degree(nid) == 0):
        st.remove_node(aid)
    for name in sorted(set(dead)):
        desc = next((d for d in g.containers if d.name == name), None)
        if desc is None or (desc.storage == "Global" and not desc.constant):
            continue
        if not any(isinstance(n, ir.AccessNode) and n.data == name for s in g.states for n in s.nodes.values()):
            g.remove_container(name)


def fuse_to_b200(g, max_rounds: int = 1000):
    """Apply ``fuse_to_b200`` to a fixpoint; returns (new graph, applied count)."""
    _, _, _, transforms, _ = _dfir()
    install()
    applied = 0
    for _ in range(max_rounds):
        ms = transforms.find_matches(g, "fuse_to_b200")
        if not ms:
            return g, applied
        g, _ = transforms.apply(ms[0], g)
        applied += 1
    raise RuntimeError("fuse_to_b200 did not reach a fixpoint")


# ---------------------------------------------------------------------------


def install() -> dict:
    """Register every fused operator (spec, reference, lowering, manual VJP)
    and the ``fuse_to_b200`` transformation into the importable ``dfir``.
    Idempotent; returns {"ops": [...], "lowerings": [...], "vjps": [...]}"""
    frontend, lowering, autodiff, transforms, _ = _dfir()
    key = id(frontend)
    if key in _STATE:
        return _STATE[key]
    refs, infers = _references(frontend), _infers(frontend)
    ops = []
    specs = [(s.name, s.attr_schema, s.min_inputs, s.max_inputs, s.min_outputs, s.max_outputs) for s in FUSED_OPS]
    for name, schema, mi, ma, mo, mx in specs:
        if name in frontend.registered_ops():
            continue
        frontend.register_op(frontend.OpSpec(name, dict(schema), mi, ma, infers[name], refs[name],
                                             min_outputs=mo, max_outputs=mx))
        ops.append(name)
    for name, builder in _LOWERINGS.items():
        lowering.register_lowering(name, _program(builder))
    for name, (build, decline) in _VJPS.items():
        autodiff._register_manual(name, build, decline)
    if "fuse_to_b200" not in transforms.CATALOG:
        transforms.register_transformation(
            "fuse_to_b200", _find_fuse, _apply_fuse,
            "Rewrite the registry-operator chains the B200 kernels execute fused (bias+dropout+residual+"
            "LayerNorm, scaled-masked softmax+dropout, bias+tanh-GELU, depthwise-conv+BN+swish+SE, "
            "LN/BN+swish) into one fused operator each.")
    _STATE[key] = {"ops": ops, "lowerings": sorted(_LOWERINGS), "vjps": sorted(_VJPS)}
    return _STATE[key]
