"""The reference's training flow on the B200:

    import_model (the reference's own BERT-layer / MBConv / norm-sweep graphs,
    oracle/make_golden.py) -> fuse_to_b200 (dfir_plugin) ->
    autodiff.differentiate_graph -> interp.execute(..., library_eval=library_eval)

Every library node of the forward AND backward states runs on the GPU through
``library_eval`` (zero UnsupportedOp, no CPU fallback); the interpreter runs
only its own glue maps (adjoint zero-fill/accumulation, Reshape copies).
Outputs and all gradients match the reference-generated f32 golden vectors at
1e-4 (interp.compare_outputs metric)."""

import numpy as np
import pytest

from dfir_util import import_dfir
from golden_util import golden

pytestmark = pytest.mark.gpu


def _setup():
    if import_dfir() is None:
        pytest.skip("reference dfir package not available")
    from dfir import autodiff, frontend, interp, ir

    from paper_2110_10802_b200 import dfir_plugin
    from paper_2110_10802_b200.library_eval import library_eval

    dfir_plugin.install()
    return frontend, interp, autodiff, ir, dfir_plugin, library_eval


def _err(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(1.0, float(np.max(np.abs(b)))))


class _Counting:
    def __init__(self, fn):
        self.fn, self.ops = fn, []

    def __call__(self, op, attrs, inputs):
        self.ops.append(op)
        return self.fn(op, attrs, inputs)


def _flow(doc, inputs, out, wrt, dy):
    frontend, interp, autodiff, ir, plugin, le = _setup()
    g, _ = plugin.fuse_to_b200(frontend.import_model(doc))
    res = autodiff.differentiate_graph(g, autodiff.GradientRequest(outputs=(out,), wrt=tuple(wrt), seed="input"))
    full = dict(inputs)
    full[res.adjoints.grads[out]] = dy
    ev = _Counting(le)
    mem, _ = interp.execute(res.graph, full, library_eval=ev)
    lib_nodes = sum(isinstance(n, ir.LibraryNode) for st in res.graph.states for n in st.nodes.values())
    assert len(ev.ops) == lib_nodes  # every library node went through the GPU seam
    return mem, {w: mem[res.adjoints.grads[w]] for w in wrt}, ev.ops


def test_bert_layer_reference_flow_on_gpu():
    from oracle import make_golden as mg

    g0 = golden("bert_layer_f32")
    B, S, H, NH, FF = (int(g0[k]) for k in ("B", "S", "H", "NH", "FF"))
    doc, out, wnames = mg.bert_layer_model(B, S, H, NH, FF, float(g0["eps"]), "f32")
    inputs = {k: g0[k] for k in ["x", "am", "dm", "m1", "m2"] + wnames}
    mem, grads, ops = _flow(doc, inputs, out, ["x"] + wnames, g0["dy"])
    for op in ("BiasDropoutResidualLayerNormGrad", "ScaledMaskedSoftmaxGrad", "BiasGeluGrad", "Einsum", "Gemm"):
        assert op in ops
    assert _err(mem[out], g0["out"]) <= 1e-4
    for w in ["x"] + wnames:
        assert _err(grads[w], g0["d_" + w]) <= 1e-4, w


def test_mbconv_reference_flow_on_gpu():
    from oracle import make_golden as mg

    g0 = golden("mbconv_s1_f32")
    N, C, H, W, SE, st = (int(g0[k]) for k in ("N", "C", "H", "W", "SE", "stride"))
    doc, y, nrm, nrv, wrt = mg.mbconv_model(N, C, H, W, SE, st, float(g0["eps"]), float(g0["momentum"]), "f32")
    inputs = {k: g0[k] for k in ("x", "wdw", "g", "b", "rm", "rv", "wr", "br", "we", "be")}
    mem, grads, ops = _flow(doc, inputs, y, wrt, g0["dy"])
    assert sorted(set(ops)) == ["MBConvBlock", "MBConvBlockGrad"]
    for k, want in ((y, "y"), (nrm, "new_rm"), (nrv, "new_rv")):
        assert _err(mem[k], g0[want]) <= 1e-4, want
    for w in wrt:
        assert _err(grads[w], g0["d_" + w]) <= 1e-4, w


@pytest.mark.parametrize("kind", ["ln", "bn"])
@pytest.mark.parametrize("tag", ["4d", "5d"])
def test_norm_act_reference_flow_on_gpu(kind, tag):
    from oracle import make_golden as mg

    g0 = golden("norm_sweep_f64")
    p = lambda k: g0[f"{kind}{tag}_{k}"].astype(np.float32)  # noqa: E731
    shape = p("x").shape
    mb = mg.ModelBuilder("n", "f32")
    x = mb.inp("x", shape)
    if kind == "ln":
        names = ["x", "g", "b"]
        mb.inp("g", (shape[-1],))
        mb.inp("b", (shape[-1],))
        u = mb.node("LayerNormalization", [x, "g", "b"], epsilon=1e-5, axis=-1)
    else:
        names = ["x", "g", "b", "rm", "rv"]
        for nm in names[1:]:
            mb.inp(nm, (shape[1],))
        u, _, _ = mb.node("BatchNormalization", [x, "g", "b", "rm", "rv"], n_out=3, epsilon=1e-5, momentum=0.9)
    y = mb.node("Mul", [u, mb.node("Sigmoid", [u])])
    mb.output(y)
    mem, grads, ops = _flow(mb.doc, {k: p(k) for k in names}, y, ["x", "g", "b"], p("dy"))
    assert _err(mem[y], g0[f"{kind}{tag}_y"]) <= 1e-4
    for w in ("x", "g", "b"):
        assert _err(grads[w], g0[f"{kind}{tag}_d{w}"]) <= 1e-4, w


def test_reduce_and_reshape_ops():
    _, _, _, _, _, le = _setup()
    from dfir import frontend

    rng = np.random.default_rng(3)
    x = rng.standard_normal((3, 4, 5)).astype(np.float32)
    for op in ("ReduceSum", "ReduceMean"):
        for attrs in ({"axes": [0], "keepdims": 0}, {"axes": [1, 2], "keepdims": 1}, {"axes": None}):
            (got,) = le(op, attrs, [x])
            (want,) = frontend.reference_apply(op, attrs, [x])
            assert got.shape == want.shape and _err(got, want) <= 1e-5, (op, attrs)
    (got,) = le("Reshape", {"shape": [12, 5]}, [x])
    assert got.shape == (12, 5) and np.array_equal(got.reshape(-1), x.reshape(-1))


def test_f64_is_rejected_unless_opted_in():
    from paper_2110_10802_b200.errors import ShapeError
    from paper_2110_10802_b200.library_eval import make_library_eval

    _, _, _, _, _, le = _setup()
    x = np.random.default_rng(0).standard_normal((4, 8))
    with pytest.raises(ShapeError):
        le("Softmax", {"axis": -1}, [x])
    (y,) = make_library_eval(f64="as_f32")("Softmax", {"axis": -1}, [x])
    assert y.dtype == np.float64 and _err(y, np.exp(x) / np.exp(x).sum(-1, keepdims=True)) <= 1e-6
