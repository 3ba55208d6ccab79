"""Shared test helpers (golden fixture loading).

Fixtures are DTNS containers written by the reference's own encoder
(oracle/make_golden.py): tests/golden/<case>/<tensor>.dtns, read here with this
package's decoder (byte-compatible with the reference, tests/test_dtns.py), plus
the case's dfm-0.1 model documents (model.json, model_fused.json)."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def golden(name):
    from paper_2110_10802_b200 import dtns

    d = os.path.join(GOLDEN, name)
    return {f[:-5]: dtns.read_tensor(os.path.join(d, f)) for f in sorted(os.listdir(d)) if f.endswith(".dtns")}


def golden_model(name, fused=False):
    with open(os.path.join(GOLDEN, name, "model_fused.json" if fused else "model.json")) as fh:
        return json.load(fh)
