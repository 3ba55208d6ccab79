"""dfm-0.1 models executed device-resident (dfm.DeviceGraph): the golden
fixtures' fused model documents with their DTNS inputs, every intermediate in
HBM, against the reference-generated outputs at the fp32 bar 1e-4."""

import numpy as np
import pytest
import torch

from golden_util import golden, golden_model

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", ["bdrln_f32", "softmax_f32", "bias_gelu_f32", "bert_layer_f32", "mbconv_s1_f32"])
def test_fused_model_on_device(case):
    from paper_2110_10802_b200.dfm import DeviceGraph

    g0 = golden(case)
    doc = golden_model(case, fused=True)
    graph = DeviceGraph(doc)
    outs = graph.run({e["name"]: g0[e["name"]] for e in doc["inputs"]})
    torch.cuda.synchronize()
    for name, t in outs.items():
        assert t.is_cuda
        got, want = t.float().cpu().numpy(), g0[name]
        err = np.max(np.abs(got - want) / np.maximum(np.abs(want), 1.0))
        assert err <= 1e-4, (name, err)


def test_f64_inputs_need_an_explicit_policy():
    from paper_2110_10802_b200.dfm import DeviceGraph
    from paper_2110_10802_b200.errors import ShapeError

    g0 = golden("bdrln_f64")
    doc = golden_model("bdrln_f64", fused=True)
    with pytest.raises(ShapeError):
        DeviceGraph(doc).run({e["name"]: g0[e["name"]] for e in doc["inputs"]})
    outs = DeviceGraph(doc, f64="as_f32").run({e["name"]: g0[e["name"]] for e in doc["inputs"]})
    err = np.max(np.abs(outs["y"].double().cpu().numpy() - g0["y"]) / np.maximum(np.abs(g0["y"]), 1.0))
    assert err <= 1e-4
