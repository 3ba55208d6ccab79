"""The dfir plugin contract on the CPU: fused operators with
specs, references, lowerings and manual VJPs installed into the real reference
``dfir``; ``fuse_to_b200`` rewrites the reference's own BERT-layer / MBConv /
norm-sweep graphs (oracle/make_golden.py) and the reference
interpreter + AD still reproduce the golden outputs and gradients.

Everything here runs the reference's ``reference_apply`` (no GPU); the same
flow with ``library_eval`` on the B200 is tests/test_gpu_dfir_flow.py."""

import numpy as np
import pytest

from dfir_util import import_dfir
from golden_util import golden

D = import_dfir()
pytestmark = pytest.mark.skipif(D is None, reason="reference dfir package not available")


def _mods():
    from dfir import autodiff, frontend, interp, lowering, transforms

    from paper_2110_10802_b200 import dfir_plugin

    dfir_plugin.install()
    return frontend, interp, autodiff, lowering, transforms, dfir_plugin


def _mg():
    from oracle import make_golden as mg

    return mg


def _ops(g):
    from dfir import ir

    return sorted(n.op for st in g.states for n in st.nodes.values() if isinstance(n, ir.LibraryNode))


def _err(a, b):
    """interp.compare_outputs metric: max|a-b| / max(|b|, 1) (interp.py:1332-1352)."""
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(1.0, float(np.max(np.abs(b))))) if b.size else 0.0


def _train(g, inputs, out, wrt, dy, library_eval=None):
    """Forward + reverse through the reference (make_golden._run flow)."""
    _, interp, autodiff, _, _, _ = _mods()
    req = autodiff.GradientRequest(outputs=(out,), wrt=tuple(wrt), seed="input")
    res = autodiff.differentiate_graph(g, req)
    full = dict(inputs)
    full[res.adjoints.grads[out]] = dy
    mem, _ = interp.execute(res.graph, full, library_eval=library_eval)
    return mem, {w: mem[res.adjoints.grads[w]] for w in wrt}, res


def test_install_registers_every_fused_op():
    frontend, _, autodiff, lowering, transforms, plugin = _mods()
    from paper_2110_10802_b200.registry import FUSED_OPS

    for spec in FUSED_OPS:
        assert spec.name in frontend.registered_ops()
        if spec.name != "MBConvBlockGrad":
            assert lowering.has_lowering(spec.name), spec.name
        if not spec.name.endswith("Grad"):
            assert autodiff.manual_backward(spec.name) is not None, spec.name
    assert "fuse_to_b200" in transforms.CATALOG
    assert plugin.install() is plugin.install()  # idempotent


def _bert_case(dtype="f64"):
    mg = _mg()
    g0 = golden(f"bert_layer_{dtype}")
    B, S, H, NH, FF = (int(g0[k]) for k in ("B", "S", "H", "NH", "FF"))
    doc, out, wnames = mg.bert_layer_model(B, S, H, NH, FF, float(g0["eps"]), dtype)
    inputs = {k: g0[k] for k in ["x", "am", "dm", "m1", "m2"] + wnames}
    return doc, out, ["x"] + wnames, inputs, g0


@pytest.mark.parametrize("dtype,tol", [("f64", 1e-10), ("f32", 1e-4)])
def test_bert_layer_fused_forward_backward_matches_golden(dtype, tol):
    frontend, interp, _, _, _, plugin = _mods()
    doc, out, wrt, inputs, g0 = _bert_case(dtype)
    g = frontend.import_model(doc)
    fused, n = plugin.fuse_to_b200(g)
    assert n == 4  # 2x BDRLN, scaled-masked softmax, bias-GELU (the FFN1 Gemm bias moves into it)
    ops = _ops(fused)
    assert ops.count("BiasDropoutResidualLayerNorm") == 2
    assert ops.count("ScaledMaskedSoftmax") == 1 and ops.count("BiasGelu") == 1
    for gone in ("Add", "Mul", "Div", "Pow", "Tanh", "Softmax", "LayerNormalization"):
        assert gone not in ops, gone
    fwd, _ = interp.execute(fused, inputs)
    assert _err(fwd[out], g0["out"]) <= tol
    mem, grads, res = _train(fused, inputs, out, wrt, g0["dy"])
    assert not res.lowered_for_ad or set(res.lowered_for_ad) <= {"Reshape"}
    bops = _ops(res.graph)
    for grad_op in ("BiasDropoutResidualLayerNormGrad", "ScaledMaskedSoftmaxGrad", "BiasGeluGrad"):
        assert grad_op in bops
    for w in wrt:
        assert _err(grads[w], g0["d_" + w]) <= tol, w


@pytest.mark.parametrize("name", ["mbconv_s1_f64", "mbconv_s2_f64", "mbconv_s1_f32"])
def test_mbconv_fused_forward_backward_matches_golden(name):
    frontend, interp, _, _, _, plugin = _mods()
    g0 = golden(name)
    tol = 1e-4 if name.endswith("f32") else 1e-9
    N, C, H, W, SE, st = (int(g0[k]) for k in ("N", "C", "H", "W", "SE", "stride"))
    doc, y, nrm, nrv, wrt = _mg().mbconv_model(N, C, H, W, SE, st, float(g0["eps"]), float(g0["momentum"]),
                                                name[-3:])
    g = frontend.import_model(doc)
    fused, n = plugin.fuse_to_b200(g)
    assert n == 1 and _ops(fused) == ["MBConvBlock"]
    inputs = {k: g0[k] for k in ("x", "wdw", "g", "b", "rm", "rv", "wr", "br", "we", "be")}
    fwd, _ = interp.execute(fused, inputs)
    for k, want in ((y, "y"), (nrm, "new_rm"), (nrv, "new_rv")):
        assert _err(fwd[k], g0[want]) <= tol, want
    _, grads, res = _train(fused, inputs, y, wrt, g0["dy"])
    assert "MBConvBlockGrad" in _ops(res.graph) and not res.lowered_for_ad
    for w in wrt:
        assert _err(grads[w], g0["d_" + w]) <= tol, w


@pytest.mark.parametrize("tag", ["4d", "5d"])
@pytest.mark.parametrize("kind", ["ln", "bn"])
def test_norm_act_fused_matches_golden(kind, tag):
    frontend, interp, _, _, _, plugin = _mods()
    mg = _mg()
    g0 = golden("norm_sweep_f64")
    p = lambda k: g0[f"{kind}{tag}_{k}"]  # noqa: E731
    shape = p("x").shape
    mb = mg.ModelBuilder("n", "f64")
    x = mb.inp("x", shape)
    if kind == "ln":
        mb.inp("g", (shape[-1],))
        mb.inp("b", (shape[-1],))
        u = mb.node("LayerNormalization", [x, "g", "b"], epsilon=1e-5, axis=-1)
        names = ["x", "g", "b"]
    else:
        for nm in ("g", "b", "rm", "rv"):
            mb.inp(nm, (shape[1],))
        u, _, _ = mb.node("BatchNormalization", [x, "g", "b", "rm", "rv"], n_out=3, epsilon=1e-5, momentum=0.9)
        names = ["x", "g", "b", "rm", "rv"]
    y = mb.node("Mul", [u, mb.node("Sigmoid", [u])])
    mb.output(y)
    fused, n = plugin.fuse_to_b200(frontend.import_model(mb.doc))
    assert n == 1 and _ops(fused) == [{"ln": "LayerNormAct", "bn": "BatchNormAct"}[kind]]
    inputs = {k: p(k) for k in names}
    _, grads, _ = _train(fused, inputs, y, ["x", "g", "b"], p("dy"))
    assert _err(interp.execute(fused, inputs)[0][y], p("y")) <= 1e-10
    for w in ("x", "g", "b"):
        assert _err(grads[w], p("d" + w)) <= 1e-10, w


def test_fused_graph_lowers_and_matches():
    """lower_all expands every fused operator through its registered lowering
    (only maps and rank-1 nodes remain) and the lowered graph still computes
    the golden forward."""
    frontend, interp, _, lowering, _, plugin = _mods()
    for name, mk in (("bdrln_f64", "bdrln"), ("softmax_f64", "sms"), ("bias_gelu_f64", "gelu")):
        g0 = golden(name)
        mg = _mg()
        if mk == "bdrln":
            mb = mg.ModelBuilder("b", "f64")
            ins = {k: g0[k] for k in ("h", "b", "m", "r", "g", "be")}
            for k, v in ins.items():
                mb.inp(k, v.shape)
            s = mb.node("Add", [mb.node("Mul", [mb.node("Add", ["h", "b"]), "m"]), "r"])
            yname = mb.node("LayerNormalization", [s, "g", "be"], epsilon=float(g0["eps"]), axis=-1)
            want = g0["y"]
        elif mk == "sms":
            mb = mg.ModelBuilder("s", "f64")
            ins = {k: g0[k] for k in ("sc", "am", "dm")}
            for k, v in ins.items():
                mb.inp(k, v.shape)
            z = mb.node("Div", ["sc"], divisor=float(g0["divisor"]))
            yname = mb.node("Mul", [mb.node("Softmax", [mb.node("Add", [z, "am"])], axis=-1), "dm"])
            want = g0["pd"]
        else:
            mb = mg.ModelBuilder("g", "f64")
            ins = {k: g0[k] for k in ("f", "b")}
            for k, v in ins.items():
                mb.inp(k, v.shape)
            yname = mg._gelu_chain(mb, mb.node("Add", ["f", "b"]))
            want = g0["y"]
        mb.output(yname)
        fused, n = plugin.fuse_to_b200(frontend.import_model(mb.doc))
        assert n == 1
        low = lowering.lower_all(fused.clone())
        assert all(op in ("Einsum", "Reduce") for op in _ops(low)), _ops(low)
        got, _ = interp.execute(low, ins)
        assert _err(got[yname], want) <= 1e-10, name


@pytest.mark.parametrize("op", ["BiasDropoutResidualLayerNormGrad", "ScaledMaskedSoftmaxGrad", "BiasGeluGrad",
                                "LayerNormActGrad", "BatchNormActGrad"])
def test_grad_op_lowering_matches_reference(op):
    """Each ...Grad operator's registered lowering (a chain of registry ops
    restating the manual VJP) agrees with its numpy reference."""
    frontend, interp, _, lowering, _, _ = _mods()
    rng = np.random.default_rng(5)
    T, H = 6, 10
    r = lambda *s: rng.standard_normal(s)  # noqa: E731
    if op == "BiasDropoutResidualLayerNormGrad":
        ins = [r(T, H), r(T, H), 1 + 0.1 * r(H), (rng.random((T, H)) > 0.2) / 0.8]
        attrs = {"epsilon": 1e-5}
    elif op == "ScaledMaskedSoftmaxGrad":
        sc = r(2, 3, 4, 5)
        p = np.exp(sc) / np.exp(sc).sum(-1, keepdims=True)
        ins = [r(2, 3, 4, 5), p, (rng.random((2, 3, 4, 5)) > 0.2) / 0.8]
        attrs = {"divisor": 8.0}
    elif op == "BiasGeluGrad":
        ins = [r(T, H), 2 * r(T, H)]
        attrs = {}
    elif op == "LayerNormActGrad":
        ins = [r(2, 3, H), r(2, 3, H), 1 + 0.1 * r(H), 0.1 * r(H)]
        attrs = {"epsilon": 1e-5, "activation": "swish"}
    else:
        ins = [r(4, 3, 2, 5), r(4, 3, 2, 5), 1 + 0.1 * r(3), 0.1 * r(3)]
        attrs = {"epsilon": 1e-5, "activation": "swish"}
    want = frontend.reference_apply(op, attrs, ins)
    names = [f"i{k}" for k in range(len(ins))]
    outs = [f"o{k}" for k in range(len(want))]
    doc = {"version": "dfm-0.1", "inputs": [{"name": n, "shape": list(a.shape), "dtype": "f64"}
                                            for n, a in zip(names, ins)],
           "outputs": outs, "nodes": [{"op": op, "attrs": attrs, "inputs": names, "outputs": outs}]}
    g = lowering.lower_all(frontend.import_model(doc))
    assert op not in _ops(g)
    got, _ = interp.execute(g, dict(zip(names, ins)))
    for o, w in zip(outs, want):
        assert _err(got[o], w) <= 1e-10, o


def test_declined_vjp_falls_back_to_lowering():
    """When the stashed pre-LN sum carries an adjoint the BDRLN VJP declines
    and the reference AD lowers the fused op instead (autodiff.py:1701-1745);
    gradients still match the unfused graph."""
    frontend, interp, autodiff, _, _, _ = _mods()
    g0 = golden("bdrln_f64")
    ins = {k: g0[k] for k in ("h", "b", "m", "r", "g", "be")}
    mk = lambda nodes, outs: {  # noqa: E731
        "version": "dfm-0.1", "inputs": [{"name": k, "shape": list(v.shape), "dtype": "f64"} for k, v in ins.items()],
        "outputs": outs, "nodes": nodes}
    tail = {"op": "Mul", "attrs": {}, "inputs": ["y", "s"], "outputs": ["o"]}
    fused = frontend.import_model(mk([{"op": "BiasDropoutResidualLayerNorm", "attrs": {"epsilon": 1e-12},
                                       "inputs": list(ins), "outputs": ["y", "s"]}, tail], ["o"]))
    plain = frontend.import_model(mk([
        {"op": "Add", "attrs": {}, "inputs": ["h", "b"], "outputs": ["t1"]},
        {"op": "Mul", "attrs": {}, "inputs": ["t1", "m"], "outputs": ["t2"]},
        {"op": "Add", "attrs": {}, "inputs": ["t2", "r"], "outputs": ["s"]},
        {"op": "LayerNormalization", "attrs": {"epsilon": 1e-12}, "inputs": ["s", "g", "be"], "outputs": ["y"]},
        tail], ["o"]))
    dy = np.random.default_rng(1).standard_normal(g0["y"].shape)
    _, gf, res = _train(fused, ins, "o", ["h", "b", "r", "g", "be"], dy)
    assert "BiasDropoutResidualLayerNorm" in res.lowered_for_ad
    _, gp, _ = _train(plain, ins, "o", ["h", "b", "r", "g", "be"], dy)
    for w in gf:
        assert _err(gf[w], gp[w]) <= 1e-12, w


def test_fuse_match_is_a_reference_transformation():
    """find_matches / apply (transforms.py:135-208): matches carry the graph
    hash, stale matches are refused, and the applied graph validates."""
    frontend, _, _, _, transforms, _ = _mods()
    from dfir import ir

    doc, *_ = _bert_case("f64")
    g = frontend.import_model(doc)
    ms = transforms.find_matches(g, "fuse_to_b200")
    assert len(ms) == 4
    g2, diff = transforms.apply(ms[0], g)
    assert diff["removed_nodes"] and not ir.validate(g2)
    with pytest.raises(transforms.StaleMatchError):
        transforms.apply(ms[1], g2)
