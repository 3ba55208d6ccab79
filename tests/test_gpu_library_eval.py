"""The reference-facing seam on the GPU: ``library_eval(op, attrs, inputs)``
against the reference's own ``reference_apply`` (dfir from baseline/_ref when
present, else the oracle), and one dfir graph executed end to end with
``interp.execute(..., library_eval=library_eval)``."""

import numpy as np
import pytest

from dfir_util import import_dfir
from oracle import oracle as O
from golden_util import golden

pytestmark = pytest.mark.gpu

RNG = np.random.default_rng(31)


def le():
    from paper_2110_10802_b200.library_eval import library_eval

    return library_eval


def ref_apply(op, attrs, inputs):
    d = import_dfir()
    if d is not None:
        return d[0].reference_apply(op, attrs, inputs)
    pytest.skip("dfir reference not importable on this box")


def r(*shape, dtype=np.float32):
    return RNG.standard_normal(shape).astype(dtype)


def close(got, want, tol=1e-4):
    for g, w in zip(got, want):
        err = O.compare(g, w)
        assert err <= tol, err


@pytest.mark.parametrize("ta,tb,cshape", [(0, 0, None), (1, 0, (5,)), (0, 1, (7, 5)), (1, 1, (1, 5))])
def test_gemm(ta, tb, cshape):
    a = r(9, 7) if ta else r(7, 9)
    b = r(5, 9) if tb else r(9, 5)
    ins = [a, b] + ([r(*cshape)] if cshape else [])
    attrs = {"alpha": 0.5, "beta": 1.5, "transA": ta, "transB": tb}
    close(le()("Gemm", attrs, ins), ref_apply("Gemm", attrs, ins))


@pytest.mark.parametrize("eq,shapes", [
    ("bsnd,btnd->bnst", [(2, 16, 3, 8), (2, 16, 3, 8)]),
    ("bnst,btnd->bsnd", [(2, 3, 16, 16), (2, 16, 3, 8)]),
    ("ij,jk->ik", [(6, 5), (5, 4)]),
    ("bik,bkj->bij", [(3, 4, 5), (3, 5, 6)]),
    ("ik,jk->ij", [(4, 7), (3, 7)]),
])
def test_einsum(eq, shapes):
    ins = [r(*s) for s in shapes]
    close(le()("Einsum", {"equation": eq}, ins), ref_apply("Einsum", {"equation": eq}, ins))


def test_matmul_broadcast():
    ins = [r(2, 1, 4, 5), r(3, 5, 6)]
    close(le()("MatMul", {}, ins), ref_apply("MatMul", {}, ins))


@pytest.mark.parametrize("axis", [-1, 1])
def test_layernorm(axis):
    x = r(4, 6, 8)
    ns = x.shape[axis % 3:]
    ins = [x, r(*ns), r(*ns)]
    attrs = {"axis": axis, "epsilon": 1e-3}
    close(le()("LayerNormalization", attrs, ins), ref_apply("LayerNormalization", attrs, ins))


@pytest.mark.parametrize("axis", [-1, 0])
def test_softmax(axis):
    ins = [r(5, 7, 3)]
    close(le()("Softmax", {"axis": axis}, ins), ref_apply("Softmax", {"axis": axis}, ins))


def test_batchnorm_training():
    x = r(4, 3, 5, 5)
    ins = [x, r(3), r(3), r(3), (np.abs(r(3)) + 0.5).astype(np.float32)]
    attrs = {"epsilon": 1e-5, "momentum": 0.8}
    close(le()("BatchNormalization", attrs, ins), ref_apply("BatchNormalization", attrs, ins))


@pytest.mark.parametrize("stride,pads", [(1, [1, 1, 1, 1]), (2, [1, 1, 1, 1]), (1, [1, 0, 0, 1])])
def test_depthwise_conv(stride, pads):
    ins = [r(2, 8, 9, 9), r(8, 1, 3, 3)]
    attrs = {"group": 8, "strides": [stride, stride], "pads": pads}
    close(le()("Conv", attrs, ins), ref_apply("Conv", attrs, ins))


def test_fused_row_ops_vs_oracle():
    g = golden("bdrln_f32")
    y, s = le()("BiasDropoutResidualLayerNorm", {"epsilon": float(g["eps"])},
                [g["h"], g["b"], g["m"], g["r"], g["g"], g["be"]])
    close([y], [g["y"]])
    ds, dh, db, dgm, dbe = le()("BiasDropoutResidualLayerNormGrad", {"epsilon": float(g["eps"])},
                                [g["dy"], s, g["g"], g["m"]])
    close([ds, dh, db, dgm, dbe], [g["dr"], g["dh"], g["db"], g["dg"], g["dbe"]])
    g = golden("softmax_f32")
    pd, p = le()("ScaledMaskedSoftmax", {"divisor": float(g["divisor"])}, [g["sc"], g["am"], g["dm"]])
    close([pd, p], [g["pd"], g["p_out"]])
    (dsc,) = le()("ScaledMaskedSoftmaxGrad", {"divisor": float(g["divisor"])}, [g["dy"], p, g["dm"]])
    close([dsc], [g["dsc"]])
    g = golden("bias_gelu_f32")
    y, pre = le()("BiasGelu", {}, [g["f"], g["b"]])
    close([y], [g["y"]])
    dpre, db = le()("BiasGeluGrad", {}, [g["dy"], pre])
    close([dpre, db], [g["df"], g["db"]])


def test_mbconv_block_vs_golden():
    g = golden("mbconv_s1_f32")
    attrs = {"strides": [1, 1], "pads": [1, 1, 1, 1], "epsilon": float(g["eps"]), "momentum": float(g["momentum"])}
    w = [g[k] for k in ("wdw", "g", "b", "rm", "rv", "wr", "br", "we", "be")]
    y, nrm, nrv = le()("MBConvBlock", attrs, [g["x"]] + w)
    close([y, nrm, nrv], [g["y"], g["new_rm"], g["new_rv"]])
    grads = le()("MBConvBlockGrad", attrs, [g["dy"], g["x"]] + w)
    close(grads, [g["d_" + k] for k in ("x", "wdw", "g", "b", "wr", "br", "we", "be")])


def test_norm_sweep_ops_vs_golden():
    g = golden("norm_sweep_f64")
    for tag in ("4d", "5d"):
        p = lambda k: g[f"ln{tag}_{k}"].astype(np.float32)  # noqa: E731
        (y,) = le()("LayerNormAct", {"epsilon": 1e-5}, [p("x"), p("g"), p("b")])
        close([y], [g[f"ln{tag}_y"]])
        q = lambda k: g[f"bn{tag}_{k}"].astype(np.float32)  # noqa: E731
        y, nrm, nrv = le()("BatchNormAct", {"epsilon": 1e-5, "momentum": 0.9},
                           [q("x"), q("g"), q("b"), q("rm"), q("rv")])
        close([y, nrm, nrv], [g[f"bn{tag}_y"], g[f"bn{tag}_new_rm"], g[f"bn{tag}_new_rv"]])


def test_dfir_interpreter_drop_in():
    """interp.execute(g, inputs, library_eval=library_eval): a dfir graph of
    hot-path operators runs on the B200 and matches the reference run."""
    d = import_dfir()
    if d is None:
        pytest.skip("reference dfir package not available")
    frontend, interp = d
    from paper_2110_10802_b200.registry import register_with_dfir

    register_with_dfir(frontend)
    T, H, F = 32, 64, 128
    arr = {"x": r(T, H), "w1": 0.1 * r(F, H), "b1": 0.1 * r(F), "w2": 0.1 * r(H, F), "b2": 0.1 * r(H),
           "m": ((RNG.random((T, H)) > 0.1) / 0.9).astype(np.float32), "g": 1 + 0.1 * r(H), "be": 0.1 * r(H)}
    nodes = [
        {"op": "Gemm", "attrs": {"transB": 1}, "inputs": ["x", "w1"], "outputs": ["f"]},
        {"op": "BiasGelu", "attrs": {}, "inputs": ["f", "b1"], "outputs": ["gl", "pre"]},
        {"op": "Gemm", "attrs": {"transB": 1}, "inputs": ["gl", "w2"], "outputs": ["a"]},
        {"op": "BiasDropoutResidualLayerNorm", "attrs": {"epsilon": 1e-12},
         "inputs": ["a", "b2", "m", "x", "g", "be"], "outputs": ["y", "s"]},
    ]
    model = {"version": "dfm-0.1", "inputs": [{"name": k, "shape": list(v.shape), "dtype": "f32"}
                                              for k, v in arr.items()], "outputs": ["y"], "nodes": nodes}
    gr = frontend.import_model(model)
    want, _ = interp.execute(gr, arr)
    got, counters = interp.execute(gr, arr, library_eval=le())
    assert O.compare(got["y"], want["y"]) <= 1e-4
    assert counters.element_reads  # the interpreter's accounting still runs
