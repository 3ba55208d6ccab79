"""Generate golden vectors for the hot path by running the REAL reference.

TEST INFRASTRUCTURE ONLY.  This script imports the reference ``dfir`` package
from ``/root/reference/pkg/src`` (read-only, present only in the build
container), builds ``dfm-0.1`` models made exclusively of registry operators
(the survey's Appendix B recipe, SURVEY.md:500-514), runs the forward pass with
``dfir.interp.execute`` (interp.py:1301-1317) and the backward pass with
``dfir.autodiff.differentiate_graph(..., seed="input")`` (autodiff.py:1760-1841)
followed by ``execute``, and stores inputs + outputs + gradients as DTNS
containers written by the reference's OWN encoder (``dfir.dtns.encode``,
dtns.py:52-70) — one ``tests/golden/<case>/<tensor>.dtns`` per array — next to
the case's ``dfm-0.1`` model documents: ``model.json`` (the registry-operator
graph the reference executed) and, where the B200 path has fused operators,
``model_fused.json`` (the same computation as fused operators; pinned to the
reference by tests/test_dfir_plugin.py and executed device-resident by
tests/test_gpu_dfm.py).

The fixtures pin ``oracle/oracle.py`` (tests/test_oracle_golden.py) so the
numpy restatement that travels to the GPU box is checked against the reference
itself.  Regenerate with::

    python oracle/make_golden.py            # writes tests/golden/<case>/*.dtns + model*.json

Every random draw uses ``numpy.random.default_rng(seed)`` with the seed stored
in the fixture.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")

GELU_C0 = 0.044715
GELU_C1 = 0.7978845608028654


def _import_dfir():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    from dfir import autodiff, frontend, interp  # noqa: WPS433

    return frontend, interp, autodiff


def _scalar(name, value, dtype):
    return {"name": name, "dtype": dtype, "dims": [], "data": [float(value)]}


class ModelBuilder:
    """Tiny helper producing ``dfm-0.1`` documents (frontend.py:886-964)."""

    def __init__(self, name, dtype):
        self.doc = {"version": "dfm-0.1", "name": name, "inputs": [], "outputs": [],
                    "initializers": [], "nodes": []}
        self.dtype = dtype
        self.k = 0

    def inp(self, name, shape):
        self.doc["inputs"].append({"name": name, "shape": list(shape), "dtype": self.dtype})
        return name

    def const(self, value):
        self.k += 1
        name = f"c{self.k}"
        self.doc["initializers"].append(_scalar(name, value, self.dtype))
        return name

    def node(self, op, inputs, n_out=1, **attrs):
        outs = []
        for _ in range(n_out):
            self.k += 1
            outs.append(f"t{self.k}_{op.lower()}")
        self.doc["nodes"].append({"op": op, "attrs": attrs, "inputs": list(inputs),
                                  "outputs": outs})
        return outs[0] if n_out == 1 else outs

    def output(self, name):
        self.doc["outputs"].append(name)


def _run(model, inputs, outputs, wrt):
    """Forward + reverse pass through the reference; returns (fwd, grads)."""
    frontend, interp, autodiff = _import_dfir()
    g = frontend.import_model(model)
    fwd, _ = interp.execute(g, inputs)
    req = autodiff.GradientRequest(outputs=tuple(outputs[:1]), wrt=tuple(wrt), seed="input")
    res = autodiff.differentiate_graph(g, req)
    rng = np.random.default_rng(4242)
    seed_name = res.adjoints.grads[outputs[0]]
    dy = rng.standard_normal(fwd[outputs[0]].shape).astype(fwd[outputs[0]].dtype)
    full_inputs = dict(inputs)
    full_inputs[seed_name] = dy
    mem, _ = interp.execute(res.graph, full_inputs)
    grads = {w: mem[res.adjoints.grads[w]] for w in wrt}
    return {o: fwd[o] for o in outputs}, dy, grads


def _drop_mask(rng, shape, p, dtype):
    keep = rng.random(shape) >= p
    return keep, (keep.astype(np.float64) * (1.0 / (1.0 - p))).astype(dtype)


def _save(name, model=None, fused=None, **arrays):
    """One DTNS container per array (reference encoder) + the model documents."""
    import json

    sys.path.insert(0, REF_SRC)
    from dfir import dtns  # noqa: WPS433

    d = os.path.join(OUT_DIR, name)
    os.makedirs(d, exist_ok=True)
    for key, val in arrays.items():
        arr = np.asarray(val)
        if arr.dtype == np.int32 or (arr.dtype.kind in "iu" and arr.dtype != np.int64):
            arr = arr.astype(np.int64)
        if isinstance(val, float):
            arr = np.float64(val)
        with open(os.path.join(d, key + ".dtns"), "wb") as fh:
            fh.write(dtns.encode(np.asarray(arr)))
    for fname, doc in (("model.json", model), ("model_fused.json", fused)):
        if doc is not None:
            with open(os.path.join(d, fname), "w") as fh:
                json.dump(doc, fh, indent=1)
    print(f"wrote {d} ({len(arrays)} tensors)")


# ---------------------------------------------------------------------------
# Hot-path subgraphs


def golden_bdrln(seed=11, T=24, H=40, p=0.1, eps=1e-12, dtype="f64"):
    npdt = np.float64 if dtype == "f64" else np.float32
    rng = np.random.default_rng(seed)
    mb = ModelBuilder("bdrln", dtype)
    h, b, m, r = mb.inp("h", (T, H)), mb.inp("b", (H,)), mb.inp("m", (T, H)), mb.inp("r", (T, H))
    g, be = mb.inp("g", (H,)), mb.inp("be", (H,))
    hb = mb.node("Add", [h, b])
    hd = mb.node("Mul", [hb, m])
    s = mb.node("Add", [hd, r])
    y = mb.node("LayerNormalization", [s, g, be], epsilon=eps, axis=-1)
    mb.output(y)
    keep, mask = _drop_mask(rng, (T, H), p, npdt)
    inputs = {"h": rng.standard_normal((T, H)).astype(npdt),
              "b": (0.1 * rng.standard_normal(H)).astype(npdt), "m": mask,
              "r": rng.standard_normal((T, H)).astype(npdt),
              "g": (1 + 0.1 * rng.standard_normal(H)).astype(npdt),
              "be": (0.1 * rng.standard_normal(H)).astype(npdt)}
    fwd, dy, grads = _run(mb.doc, inputs, [y], ["h", "b", "r", "g", "be"])
    fz = ModelBuilder("bdrln_fused", dtype)
    for k, v in inputs.items():
        fz.inp(k, v.shape)
    fz.doc["nodes"].append({"op": "BiasDropoutResidualLayerNorm", "attrs": {"epsilon": eps},
                            "inputs": ["h", "b", "m", "r", "g", "be"], "outputs": ["y", "s"]})
    fz.output("y")
    _save(f"bdrln_{dtype}", model=mb.doc, fused=fz.doc, seed=seed, p=p, eps=eps, keep=keep, **inputs, y=fwd[y],
          dy=dy, **{"d" + k: v for k, v in grads.items()})


def golden_softmax(seed=12, B=2, NH=3, S=16, p=0.1, divisor=8.0, dtype="f64"):
    npdt = np.float64 if dtype == "f64" else np.float32
    rng = np.random.default_rng(seed)
    mb = ModelBuilder("scaled_masked_softmax", dtype)
    sc, am, dm = mb.inp("sc", (B, NH, S, S)), mb.inp("am", (B, 1, 1, S)), mb.inp("dm", (B, NH, S, S))
    z = mb.node("Div", [sc], divisor=divisor)
    za = mb.node("Add", [z, am])
    pr = mb.node("Softmax", [za], axis=-1)
    pd = mb.node("Mul", [pr, dm])
    mb.output(pd)
    mb.output(pr)
    keep, dmask = _drop_mask(rng, (B, NH, S, S), p, npdt)
    amask = np.where(rng.random((B, 1, 1, S)) < 0.1, -10000.0, 0.0).astype(npdt)
    inputs = {"sc": (3.0 * rng.standard_normal((B, NH, S, S))).astype(npdt), "am": amask, "dm": dmask}
    fwd, dy, grads = _run(mb.doc, inputs, [pd, pr], ["sc"])
    fz = ModelBuilder("scaled_masked_softmax_fused", dtype)
    for k, v in inputs.items():
        fz.inp(k, v.shape)
    fz.doc["nodes"].append({"op": "ScaledMaskedSoftmax", "attrs": {"divisor": divisor},
                            "inputs": ["sc", "am", "dm"], "outputs": ["pd", "p_out"]})
    fz.output("pd")
    fz.output("p_out")
    _save(f"softmax_{dtype}", model=mb.doc, fused=fz.doc, seed=seed, p=p, divisor=divisor, keep=keep, **inputs,
          pd=fwd[pd], p_out=fwd[pr], dy=dy, dsc=grads["sc"])


def _gelu_chain(mb, x):
    x3 = mb.node("Pow", [x], exponent=3.0)
    t1 = mb.node("Mul", [x3, mb.const(GELU_C0)])
    t2 = mb.node("Add", [x, t1])
    t3 = mb.node("Mul", [t2, mb.const(GELU_C1)])
    t4 = mb.node("Tanh", [t3])
    t5 = mb.node("Add", [t4, mb.const(1.0)])
    t6 = mb.node("Mul", [x, t5])
    return mb.node("Mul", [t6, mb.const(0.5)])


def golden_bias_gelu(seed=13, T=20, F=48, dtype="f64"):
    npdt = np.float64 if dtype == "f64" else np.float32
    rng = np.random.default_rng(seed)
    mb = ModelBuilder("bias_gelu", dtype)
    f, b = mb.inp("f", (T, F)), mb.inp("b", (F,))
    x = mb.node("Add", [f, b])
    y = _gelu_chain(mb, x)
    mb.output(y)
    inputs = {"f": (2.0 * rng.standard_normal((T, F))).astype(npdt),
              "b": (0.1 * rng.standard_normal(F)).astype(npdt)}
    fwd, dy, grads = _run(mb.doc, inputs, [y], ["f", "b"])
    fz = ModelBuilder("bias_gelu_fused", dtype)
    for k, v in inputs.items():
        fz.inp(k, v.shape)
    fz.doc["nodes"].append({"op": "BiasGelu", "attrs": {}, "inputs": ["f", "b"], "outputs": ["y", "pre"]})
    fz.output("y")
    _save(f"bias_gelu_{dtype}", model=mb.doc, fused=fz.doc, seed=seed, **inputs, y=fwd[y], dy=dy, df=grads["f"],
          db=grads["b"])


def bert_layer_model(B, S, H, NH, FF, eps, dtype):
    """BERT encoder layer from registry ops only (SURVEY.md:500-511)."""
    dh = H // NH
    T = B * S
    mb = ModelBuilder("bert_layer", dtype)
    x = mb.inp("x", (T, H))
    am = mb.inp("am", (B, 1, 1, S))
    dm = mb.inp("dm", (B, NH, S, S))
    m1 = mb.inp("m1", (T, H))
    m2 = mb.inp("m2", (T, H))
    w = {}
    for nm, shp in [("wq", (H, H)), ("wk", (H, H)), ("wv", (H, H)), ("wo", (H, H)),
                    ("w1", (FF, H)), ("w2", (H, FF))]:
        w[nm] = mb.inp(nm, shp)
    for nm, n in [("bq", H), ("bk", H), ("bv", H), ("bo", H), ("b1", FF), ("b2", H),
                  ("g1", H), ("be1", H), ("g2", H), ("be2", H)]:
        w[nm] = mb.inp(nm, (n,))
    heads = {}
    for t in "qkv":
        lin = mb.node("Gemm", [x, w["w" + t], w["b" + t]], transB=1)
        heads[t] = mb.node("Reshape", [lin], shape=[B, S, NH, dh])
    sc = mb.node("Einsum", [heads["q"], heads["k"]], equation="bsnd,btnd->bnst")
    z = mb.node("Div", [sc], divisor=float(np.sqrt(dh)))
    za = mb.node("Add", [z, am])
    pr = mb.node("Softmax", [za], axis=-1)
    pd = mb.node("Mul", [pr, dm])
    c4 = mb.node("Einsum", [pd, heads["v"]], equation="bnst,btnd->bsnd")
    ctx = mb.node("Reshape", [c4], shape=[T, H])
    a1 = mb.node("Gemm", [ctx, w["wo"]], transB=1)
    s1 = mb.node("Add", [mb.node("Mul", [mb.node("Add", [a1, w["bo"]]), m1]), x])
    ln1 = mb.node("LayerNormalization", [s1, w["g1"], w["be1"]], epsilon=eps, axis=-1)
    f = mb.node("Gemm", [ln1, w["w1"], w["b1"]], transB=1)
    gl = _gelu_chain(mb, f)
    a2 = mb.node("Gemm", [gl, w["w2"]], transB=1)
    s2 = mb.node("Add", [mb.node("Mul", [mb.node("Add", [a2, w["b2"]]), m2]), ln1])
    out = mb.node("LayerNormalization", [s2, w["g2"], w["be2"]], epsilon=eps, axis=-1)
    mb.output(out)
    return mb.doc, out, list(w)


def bert_layer_model_fused(B, S, H, NH, FF, eps, dtype):
    """The same layer with the B200 path's fused operators (registry.py
    FUSED_OPS): what dfir_plugin.fuse_to_b200 makes of bert_layer_model."""
    dh = H // NH
    T = B * S
    mb = ModelBuilder("bert_layer_fused", dtype)
    x = mb.inp("x", (T, H))
    for nm, shp in [("am", (B, 1, 1, S)), ("dm", (B, NH, S, S)), ("m1", (T, H)), ("m2", (T, H)),
                    ("wq", (H, H)), ("wk", (H, H)), ("wv", (H, H)), ("wo", (H, H)), ("w1", (FF, H)),
                    ("w2", (H, FF))]:
        mb.inp(nm, shp)
    for nm, n in [("bq", H), ("bk", H), ("bv", H), ("bo", H), ("b1", FF), ("b2", H),
                  ("g1", H), ("be1", H), ("g2", H), ("be2", H)]:
        mb.inp(nm, (n,))
    heads = {}
    for t in "qkv":
        lin = mb.node("Gemm", [x, "w" + t, "b" + t], transB=1)
        heads[t] = mb.node("Reshape", [lin], shape=[B, S, NH, dh])
    sc = mb.node("Einsum", [heads["q"], heads["k"]], equation="bsnd,btnd->bnst")
    pd, _ = mb.node("ScaledMaskedSoftmax", [sc, "am", "dm"], n_out=2, divisor=float(np.sqrt(dh)))
    c4 = mb.node("Einsum", [pd, heads["v"]], equation="bnst,btnd->bsnd")
    ctx = mb.node("Reshape", [c4], shape=[T, H])
    a1 = mb.node("Gemm", [ctx, "wo"], transB=1)
    ln1, _ = mb.node("BiasDropoutResidualLayerNorm", [a1, "bo", "m1", x, "g1", "be1"], n_out=2, epsilon=eps)
    f = mb.node("Gemm", [ln1, "w1"], transB=1)
    gl, _ = mb.node("BiasGelu", [f, "b1"], n_out=2)
    a2 = mb.node("Gemm", [gl, "w2"], transB=1)
    mb.doc["nodes"].append({"op": "BiasDropoutResidualLayerNorm", "attrs": {"epsilon": eps},
                            "inputs": [a2, "b2", "m2", ln1, "g2", "be2"], "outputs": ["out", "s2"]})
    mb.output("out")
    return mb.doc


def bert_layer_inputs(rng, B, S, H, NH, FF, p, npdt):
    T = B * S
    inp = {"x": rng.standard_normal((T, H))}
    for nm, shp in [("wq", (H, H)), ("wk", (H, H)), ("wv", (H, H)), ("wo", (H, H)),
                    ("w1", (FF, H)), ("w2", (H, FF))]:
        inp[nm] = 0.02 * rng.standard_normal(shp)
    for nm, n in [("bq", H), ("bk", H), ("bv", H), ("bo", H), ("b1", FF), ("b2", H)]:
        inp[nm] = 0.1 * rng.standard_normal(n)
    for i in "12":
        inp["g" + i] = 1 + 0.1 * rng.standard_normal(H)
        inp["be" + i] = 0.1 * rng.standard_normal(H)
    inp["am"] = np.where(rng.random((B, 1, 1, S)) < 0.1, -10000.0, 0.0)
    keeps = {}
    for nm, shp in [("dm", (B, NH, S, S)), ("m1", (T, H)), ("m2", (T, H))]:
        keeps["keep_" + nm], inp[nm] = _drop_mask(rng, shp, p, np.float64)
    inp = {k: v.astype(npdt) for k, v in inp.items()}
    return inp, keeps


def golden_bert_layer(seed=14, B=2, S=8, H=32, NH=2, FF=64, p=0.1, eps=1e-12, dtype="f64"):
    npdt = np.float64 if dtype == "f64" else np.float32
    rng = np.random.default_rng(seed)
    doc, out, wnames = bert_layer_model(B, S, H, NH, FF, eps, dtype)
    inputs, keeps = bert_layer_inputs(rng, B, S, H, NH, FF, p, npdt)
    wrt = ["x"] + wnames
    fwd, dy, grads = _run(doc, inputs, [out], wrt)
    _save(f"bert_layer_{dtype}", model=doc, fused=bert_layer_model_fused(B, S, H, NH, FF, eps, dtype), seed=seed,
          B=B, S=S, H=H, NH=NH, FF=FF, p=p, eps=eps, **keeps, **inputs, out=fwd[out], dy=dy,
          **{"d_" + k: v for k, v in grads.items()})


def mbconv_model(N, C, Hh, Ww, SE, stride, eps, momentum, dtype):
    """dw3x3 + BN(train) + swish + SE, SURVEY.md:512-514."""
    mb = ModelBuilder("mbconv", dtype)
    x = mb.inp("x", (N, C, Hh, Ww))
    names = {"wdw": (C, 1, 3, 3), "g": (C,), "b": (C,), "rm": (C,), "rv": (C,),
             "wr": (SE, C), "br": (SE,), "we": (C, SE), "be": (C,)}
    for nm, shp in names.items():
        mb.inp(nm, shp)
    z = mb.node("Conv", [x, "wdw"], group=C, pads=[1, 1, 1, 1], strides=[stride, stride],
                kernel_shape=[3, 3])
    bn, nrm, nrv = mb.node("BatchNormalization", [z, "g", "b", "rm", "rv"], n_out=3,
                           epsilon=eps, momentum=momentum)
    a = mb.node("Mul", [bn, mb.node("Sigmoid", [bn])])
    pooled = mb.node("GlobalAveragePool", [a])
    p2 = mb.node("Reshape", [pooled], shape=[N, C])
    r = mb.node("Gemm", [p2, "wr", "br"], transB=1)
    r2 = mb.node("Mul", [r, mb.node("Sigmoid", [r])])
    e = mb.node("Gemm", [r2, "we", "be"], transB=1)
    es = mb.node("Reshape", [mb.node("Sigmoid", [e])], shape=[N, C, 1, 1])
    y = mb.node("Mul", [a, es])
    mb.output(y)
    mb.output(nrm)
    mb.output(nrv)
    return mb.doc, y, nrm, nrv, ["x", "wdw", "g", "b", "wr", "br", "we", "be"]


def golden_mbconv(seed=15, N=2, C=8, Hh=7, Ww=7, SE=2, stride=1, eps=1e-3, momentum=0.99,
                  dtype="f64"):
    npdt = np.float64 if dtype == "f64" else np.float32
    rng = np.random.default_rng(seed)
    doc, y, nrm, nrv, wrt = mbconv_model(N, C, Hh, Ww, SE, stride, eps, momentum, dtype)
    inputs = {"x": rng.standard_normal((N, C, Hh, Ww)),
              "wdw": 0.3 * rng.standard_normal((C, 1, 3, 3)),
              "g": rng.standard_normal(C), "b": rng.standard_normal(C),
              "rm": 0.1 * rng.standard_normal(C), "rv": 1.0 + 0.1 * rng.random(C),
              "wr": 0.3 * rng.standard_normal((SE, C)), "br": 0.1 * rng.standard_normal(SE),
              "we": 0.3 * rng.standard_normal((C, SE)), "be": 0.1 * rng.standard_normal(C)}
    inputs = {k: v.astype(npdt) for k, v in inputs.items()}
    fwd, dy, grads = _run(doc, inputs, [y, nrm, nrv], wrt)
    fz = ModelBuilder("mbconv_fused", dtype)
    for k, v in inputs.items():
        fz.inp(k, v.shape)
    fz.doc["nodes"].append({"op": "MBConvBlock", "attrs": {"strides": [stride, stride], "pads": [1, 1, 1, 1],
                                                            "epsilon": eps, "momentum": momentum},
                            "inputs": ["x", "wdw", "g", "b", "rm", "rv", "wr", "br", "we", "be"],
                            "outputs": ["y", "new_rm", "new_rv"]})
    for o in ("y", "new_rm", "new_rv"):
        fz.output(o)
    _save(f"mbconv_s{stride}_{dtype}", model=doc, fused=fz.doc, seed=seed, N=N, C=C, H=Hh, W=Ww, SE=SE,
          stride=stride, eps=eps, momentum=momentum, **inputs, y=fwd[y], new_rm=fwd[nrm], new_rv=fwd[nrv],
          dy=dy, **{"d_" + k: v for k, v in grads.items()})


def golden_norm_sweep(seed=16, dtype="f64"):
    """LN (last axis) vs BN (channel axis) on 4D/5D tensors, each fused with
    swish."""
    npdt = np.float64 if dtype == "f64" else np.float32
    rng = np.random.default_rng(seed)
    out = {"seed": seed}
    for shape in [(2, 3, 4, 5), (2, 3, 2, 4, 5)]:
        tag = f"{len(shape)}d"
        # LayerNorm over the last axis + bias add + swish
        mb = ModelBuilder("ln_swish", dtype)
        x = mb.inp("x", shape)
        g, b = mb.inp("g", (shape[-1],)), mb.inp("b", (shape[-1],))
        ln = mb.node("LayerNormalization", [x, g, b], epsilon=1e-5, axis=-1)
        y = mb.node("Mul", [ln, mb.node("Sigmoid", [ln])])
        mb.output(y)
        inputs = {"x": rng.standard_normal(shape).astype(npdt),
                  "g": (1 + 0.1 * rng.standard_normal(shape[-1])).astype(npdt),
                  "b": (0.1 * rng.standard_normal(shape[-1])).astype(npdt)}
        fwd, dy, grads = _run(mb.doc, inputs, [y], ["x", "g", "b"])
        for k, v in inputs.items():
            out[f"ln{tag}_{k}"] = v
        out[f"ln{tag}_y"], out[f"ln{tag}_dy"] = fwd[y], dy
        for k, v in grads.items():
            out[f"ln{tag}_d{k}"] = v
        # BatchNorm over channel axis 1 + swish
        c = shape[1]
        mb = ModelBuilder("bn_swish", dtype)
        x = mb.inp("x", shape)
        for nm in ("g", "b", "rm", "rv"):
            mb.inp(nm, (c,))
        bn, nrm, nrv = mb.node("BatchNormalization", [x, "g", "b", "rm", "rv"], n_out=3,
                               epsilon=1e-5, momentum=0.9)
        y = mb.node("Mul", [bn, mb.node("Sigmoid", [bn])])
        mb.output(y)
        mb.output(nrm)
        mb.output(nrv)
        inputs = {"x": rng.standard_normal(shape).astype(npdt),
                  "g": (1 + 0.1 * rng.standard_normal(c)).astype(npdt),
                  "b": (0.1 * rng.standard_normal(c)).astype(npdt),
                  "rm": (0.1 * rng.standard_normal(c)).astype(npdt),
                  "rv": (1 + 0.1 * rng.random(c)).astype(npdt)}
        fwd, dy, grads = _run(mb.doc, inputs, [y, nrm, nrv], ["x", "g", "b"])
        for k, v in inputs.items():
            out[f"bn{tag}_{k}"] = v
        out[f"bn{tag}_y"], out[f"bn{tag}_dy"] = fwd[y], dy
        out[f"bn{tag}_new_rm"], out[f"bn{tag}_new_rv"] = fwd[nrm], fwd[nrv]
        for k, v in grads.items():
            out[f"bn{tag}_d{k}"] = v
    _save(f"norm_sweep_{dtype}", **out)


def golden_known_answers():
    """Single-op reference_apply outputs for the ops the kernels replace,
    on the reference's own test shapes (test_frontend.py:187-305,
    test_lowering.py:188-251)."""
    frontend, _, _ = _import_dfir()
    rng = np.random.default_rng(23)
    out = {}
    # Depthwise conv, padded and strided cases (test_lowering.py:227-246 style)
    for i, (xs, stride, pads) in enumerate([((1, 3, 5, 5), 1, [1, 1, 1, 1]),
                                           ((2, 4, 8, 8), 2, [1, 1, 1, 1]),
                                           ((1, 4, 4, 4), 1, [1, 0, 0, 1])]):
        x = rng.standard_normal(xs)
        w = rng.standard_normal((xs[1], 1, 3, 3))
        (y,) = frontend.reference_apply("Conv", {"group": xs[1], "pads": pads,
                                                 "strides": [stride, stride]}, [x, w])
        out.update({f"dw{i}_x": x, f"dw{i}_w": w, f"dw{i}_y": y,
                    f"dw{i}_stride": stride, f"dw{i}_pads": np.array(pads)})
    # BatchNorm training stats with momentum 0.8 (test_frontend.py:260-276)
    x = rng.standard_normal((4, 3, 2, 2))
    sc, bi, rm, rv = rng.standard_normal(3), rng.standard_normal(3), rng.standard_normal(3), rng.random(3) + 0.5
    y, nm, nv = frontend.reference_apply("BatchNormalization", {"momentum": 0.8}, [x, sc, bi, rm, rv])
    out.update(bn_x=x, bn_scale=sc, bn_bias=bi, bn_rm=rm, bn_rv=rv, bn_y=y, bn_new_rm=nm, bn_new_rv=nv)
    # LayerNorm eps 1e-3 (test_frontend.py:209-217) and softmax (187-192)
    x = rng.standard_normal((4, 5, 8))
    g, b = rng.standard_normal(8), rng.standard_normal(8)
    (y,) = frontend.reference_apply("LayerNormalization", {"epsilon": 1e-3}, [x, g, b])
    out.update(ln_x=x, ln_g=g, ln_b=b, ln_y=y)
    x = rng.standard_normal((3, 5, 7))
    (y,) = frontend.reference_apply("Softmax", {"axis": -1}, [x])
    out.update(sm_x=x, sm_y=y)
    # Gemm alpha/beta/trans (test_frontend.py:219-225)
    a, bb, c = rng.standard_normal((5, 2)), rng.standard_normal((5, 3)), rng.standard_normal(3)
    (y,) = frontend.reference_apply("Gemm", {"alpha": 0.5, "beta": 2.0, "transA": 1}, [a, bb, c])
    out.update(gemm_a=a, gemm_b=bb, gemm_c=c, gemm_y=y)
    # GAP (test_frontend.py:302-305)
    x = rng.standard_normal((2, 3, 4, 5))
    (y,) = frontend.reference_apply("GlobalAveragePool", {}, [x])
    out.update(gap_x=x, gap_y=y)
    _save("known_answers", **out)


def main(only=None):
    if only == "mbconv":
        for dt in ("f64", "f32"):
            golden_mbconv(dtype=dt, stride=1)
        golden_mbconv(dtype="f64", stride=2, Hh=8, Ww=8)
        return
    golden_known_answers()
    for dt in ("f64", "f32"):
        golden_bdrln(dtype=dt)
        golden_softmax(dtype=dt)
        golden_bias_gelu(dtype=dt)
        golden_bert_layer(dtype=dt)
        golden_mbconv(dtype=dt, stride=1)
    golden_mbconv(dtype="f64", stride=2, Hh=8, Ww=8)
    golden_norm_sweep(dtype="f64")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
