"""Reference byte accounting of the unfused schedules (measurement reference,
test infrastructure only — never imported by the product package).

Builds the BERT-base encoder layer (C2: B=8, S=512) and the MBConv block (C3:
N=96, 112x112, C=96) as dfm-0.1 graphs from registry operators only (the
golden builders of oracle/make_golden.py), and evaluates the reference's own
``ir.movement_volume`` (ir.py:790-835) on
  * the imported graph (library-node form: one kernel per registry op), and
  * ``lowering.lower_all`` of it (the unfused native map form, lowering.py:1085-1143),
for the forward graph and for the forward + reverse graph of
``autodiff.differentiate_graph`` (autodiff.py:1760-1841).  The reference has no
bf16 (ir.py:49-56): the graphs are f32 and bench.py halves the bytes for the
bf16 comparison.  Writes tests/golden/movement_volume.json; run it here (the
reference is importable in this container, not on the GPU box).

    PYTHONPATH=/root/reference/pkg/src python oracle/movement_volume.py
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle import make_golden as MG  # noqa: E402


def report(doc, out, wrt):
    frontend, interp, autodiff = MG._import_dfir()
    from dfir import ir, lowering  # noqa: WPS433

    g = frontend.import_model(doc)
    res = {"fwd_library_bytes": ir.movement_volume(g).bytes}
    gl = lowering.lower_all(g)
    res["fwd_lowered_bytes"] = ir.movement_volume(gl).bytes
    req = autodiff.GradientRequest(outputs=(out,), wrt=tuple(wrt), seed="input")
    t0 = time.time()
    ad = autodiff.differentiate_graph(g, req).graph
    res["fwd_bwd_library_bytes"] = ir.movement_volume(ad).bytes
    res["ad_seconds"] = round(time.time() - t0, 1)
    return res


def main():
    out = {"note": "reference ir.movement_volume (ir.py:790-835) of the unfused schedules, f32 graphs"}
    doc, o, wnames = MG.bert_layer_model(8, 512, 768, 12, 3072, 1e-12, "f32")
    out["bert_c2"] = report(doc, o, ["x"] + wnames)
    print("bert", out["bert_c2"], flush=True)
    doc, y, _, _, wrt = MG.mbconv_model(96, 96, 112, 112, 4, 1, 1e-3, 0.99, "f32")
    out["mbconv_c3"] = report(doc, y, wrt)
    print("mbconv", out["mbconv_c3"], flush=True)
    path = os.path.join(HERE, "..", "tests", "golden", "movement_volume.json")
    json.dump(out, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
