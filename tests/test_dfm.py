"""dfm-0.1 model documents (§8f row 3) on the CPU: the parser restates
frontend.parse_model_json (frontend.py:886-964) with its error messages, the
golden fixtures' model documents parse identically in both, and the fused
documents (model_fused.json) compute the reference's golden values when the
reference itself executes them (dfir + dfir_plugin)."""

import base64

import numpy as np
import pytest

from dfir_util import import_dfir
from golden_util import golden, golden_model

CASES = ["bdrln_f64", "softmax_f64", "bias_gelu_f64", "bert_layer_f64", "mbconv_s1_f64", "mbconv_s2_f64",
         "bdrln_f32", "bert_layer_f32", "mbconv_s1_f32"]


def _parse():
    from paper_2110_10802_b200.dfm import parse_model

    return parse_model


@pytest.mark.parametrize("case", CASES)
def test_golden_documents_parse_like_the_reference(case):
    for fused in (False, True):
        doc = golden_model(case, fused=fused)
        m = _parse()(doc)
        assert m.outputs and m.nodes
        d = import_dfir()
        if d is None or fused:
            continue
        ref = d[0].parse_model_json(doc)
        assert [(n, list(s), t) for n, s, t in m.inputs] == [(n, list(s), t) for n, s, t in ref.inputs]
        assert m.outputs == ref.outputs
        assert [(n.op, n.inputs, n.outputs, n.attrs) for n in m.nodes] == \
            [(n.op, n.inputs, n.outputs, n.attrs) for n in ref.nodes]


def test_parse_errors_match_the_reference():
    from paper_2110_10802_b200.errors import ModelError

    parse = _parse()
    bad = [
        ({"version": "dfm-0.2"}, "unsupported model version 'dfm-0.2'; expected 'dfm-0.1'"),
        ({"version": "dfm-0.1", "inputs": [{"name": "x", "shape": [2]}]}, "inputs[]: missing required keys"),
        ({"version": "dfm-0.1", "inputs": [{"name": "x", "shape": [2], "dtype": "f16"}]}, "unknown dtype 'f16'"),
        ({"version": "dfm-0.1", "inputs": [{"name": "x", "shape": [-1], "dtype": "f32"}]}, "dims must be"),
        ({"version": "dfm-0.1", "initializers": [{"name": "c"}]}, "needs 'file', 'base64', or dtype/dims/data"),
        ({"version": "dfm-0.1", "nodes": [{"op": "Add"}]}, "nodes[0]: missing required keys"),
    ]
    d = import_dfir()
    for doc, msg in bad:
        with pytest.raises(ModelError) as ours:
            parse(doc)
        assert msg in str(ours.value)
        if d is not None:
            with pytest.raises(Exception) as theirs:
                d[0].parse_model_json(doc)
            assert str(theirs.value) == str(ours.value)


def test_initializer_forms(tmp_path):
    from paper_2110_10802_b200 import dtns

    arr = np.arange(6, dtype=np.float32).reshape(2, 3)
    dtns.write_tensor(str(tmp_path / "w.dtns"), arr)
    doc = {"version": "dfm-0.1", "outputs": [], "initializers": [
        {"name": "a", "dtype": "f32", "dims": [2, 3], "data": arr.reshape(-1).tolist()},
        {"name": "b", "base64": base64.b64encode(dtns.encode(arr)).decode()},
        {"name": "c", "file": "w.dtns"}]}
    m = _parse()(doc, base_dir=str(tmp_path))
    for k in "abc":
        assert np.array_equal(m.initializers[k], arr)


def test_device_graph_rejects_operators_off_the_hot_path():
    from paper_2110_10802_b200.dfm import DeviceGraph
    from paper_2110_10802_b200.errors import UnsupportedOp

    with pytest.raises(UnsupportedOp):
        DeviceGraph(golden_model("bdrln_f64"))  # the unfused Add/Mul chain


@pytest.mark.skipif(import_dfir() is None, reason="reference dfir package not available")
@pytest.mark.parametrize("case", CASES)
def test_fused_documents_compute_the_golden_values_in_the_reference(case):
    """The reference interpreter executing model_fused.json (fused operators
    installed by dfir_plugin) reproduces the values it computed for the
    unfused model.json."""
    frontend, interp = import_dfir()
    from paper_2110_10802_b200 import dfir_plugin

    dfir_plugin.install()
    g0 = golden(case)
    doc = golden_model(case, fused=True)
    gr = frontend.import_model(doc)
    ins = {e["name"]: g0[e["name"]] for e in doc["inputs"]}
    got, _ = interp.execute(gr, ins)
    tol = 1e-10 if case.endswith("f64") else 1e-5
    for o in doc["outputs"]:
        want = g0[o]
        err = np.max(np.abs(got[o] - want) / np.maximum(np.abs(want), 1.0))
        assert err <= tol, (o, err)
