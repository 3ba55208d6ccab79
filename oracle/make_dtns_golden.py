"""Golden DTNS containers written by the REAL reference encoder.

TEST INFRASTRUCTURE ONLY.  Imports ``dfir.dtns`` from /root/reference/pkg/src
(read-only, build container only), encodes a fixed set of seeded arrays with
``dtns.encode`` (dtns.py:50-68) and stores the bytes under
``tests/golden/dtns/<name>.dtns`` next to ``values.npz`` (the arrays), so
tests/test_dtns.py can check this package's decoder/encoder byte for byte
against the reference without the reference present.

    python oracle/make_dtns_golden.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from dfir import dtns  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "dtns")


def arrays():
    rng = np.random.default_rng(20211020)
    return {
        "f32_4x5": rng.standard_normal((4, 5)).astype(np.float32),
        "f64_3x2x2": rng.standard_normal((3, 2, 2)),
        "i64_7": rng.integers(-(2 ** 40), 2 ** 40, size=(7,), dtype=np.int64),
        "bool_2x3": rng.random((2, 3)) > 0.5,
        "rank0_f64": np.float64(3.5),
        "empty_0x4_f32": np.zeros((0, 4), dtype=np.float32),
        # a BDRLN-shaped operand (a row block of the C1 hidden state) and its keep mask
        "bert_x_8x768_f32": rng.standard_normal((8, 768)).astype(np.float32),
        "bert_keep_8x768_bool": rng.random((8, 768)) >= 0.1,
    }


def main():
    os.makedirs(OUT, exist_ok=True)
    vals = arrays()
    for name, arr in vals.items():
        with open(os.path.join(OUT, name + ".dtns"), "wb") as fh:
            fh.write(dtns.encode(arr))
    np.savez_compressed(os.path.join(OUT, "values.npz"), **{k: np.asarray(v) for k, v in vals.items()})
    print("wrote", len(vals), "containers to", OUT)


if __name__ == "__main__":
    main()
