"""Operator-spec contract (mirror of dfir.frontend's registry) — CPU only."""

import numpy as np
import pytest

from dfir_util import import_dfir
from paper_2110_10802_b200 import registry
from paper_2110_10802_b200.errors import ShapeError, UnsupportedOp
from paper_2110_10802_b200.library_eval import SUPPORTED_OPS, library_eval


def test_normalize_attrs_contract():
    """frontend.normalize_attrs (frontend.py:112-129): defaults, unknown names
    rejected, required attributes enforced."""
    assert registry.normalize_attrs("LayerNormalization", {}) == {"axis": -1, "epsilon": 1e-5}
    assert registry.normalize_attrs("Gemm", {"transB": 1})["transB"] == 1
    with pytest.raises(ShapeError):
        registry.normalize_attrs("Softmax", {"axis": -1, "bogus": 3})
    with pytest.raises(ShapeError):
        registry.normalize_attrs("Einsum", {})
    # the per-node implementation selector is accepted (lowering.py:1045-1075)
    assert registry.normalize_attrs("Softmax", {"implementation": "native"}) == {"axis": -1}


def test_registry_refuses_duplicates_and_unknown():
    with pytest.raises(registry.DuplicateOp):
        registry.register_op(registry.OpSpec("Gemm", {}, 2, 3))
    with pytest.raises(UnsupportedOp):
        registry.get_op("NotAnOp")


def test_library_eval_has_no_cpu_fallback():
    """Operators off the hot path raise instead of running on the CPU."""
    for op in ("Add", "Relu", "Sigmoid", "GlobalAveragePool"):
        with pytest.raises(UnsupportedOp):
            library_eval(op, {}, [np.zeros(4, np.float32)])
    assert "BiasDropoutResidualLayerNorm" in SUPPORTED_OPS
    assert all(op in registry.registered_ops() for op in SUPPORTED_OPS)


def test_fused_specs_register_into_dfir():
    """The fused operators install into the real reference registry and their
    reference evaluators (composed from dfir's own operators) match the
    unfused reference graph."""
    d = import_dfir()
    if d is None:
        pytest.skip("reference dfir package not available")
    frontend, interp = d
    registry.register_with_dfir(frontend)
    assert "BiasDropoutResidualLayerNorm" in frontend.registered_ops()
    rng = np.random.default_rng(0)
    T, H = 6, 16
    h, r = rng.standard_normal((T, H)), rng.standard_normal((T, H))
    b, g, be = rng.standard_normal(H), 1 + 0.1 * rng.standard_normal(H), rng.standard_normal(H)
    m = (rng.random((T, H)) > 0.1) / 0.9
    y, s = frontend.reference_apply("BiasDropoutResidualLayerNorm", {"epsilon": 1e-12}, [h, b, m, r, g, be])
    (want,) = frontend.reference_apply("LayerNormalization", {"epsilon": 1e-12}, [(h + b) * m + r, g, be])
    np.testing.assert_allclose(y, want, rtol=1e-12)
    np.testing.assert_allclose(s, (h + b) * m + r, rtol=1e-12)
    # and a graph using it validates and runs in the reference interpreter
    model = {"version": "dfm-0.1", "inputs": [{"name": n, "shape": list(a.shape), "dtype": "f64"}
                                              for n, a in (("h", h), ("b", b), ("m", m), ("r", r), ("g", g),
                                                           ("be", be))],
             "outputs": ["y"], "nodes": [{"op": "BiasDropoutResidualLayerNorm", "attrs": {"epsilon": 1e-12},
                                          "inputs": ["h", "b", "m", "r", "g", "be"], "outputs": ["y", "s"]}]}
    gr = frontend.import_model(model)
    got = interp.run_outputs(gr, dict(h=h, b=b, m=m, r=r, g=g, be=be), outputs=["y"])
    np.testing.assert_allclose(got["y"], want, rtol=1e-12)
