"""C4 normalisation sweep timing alone (bench.py's measure_norm_sweep_c4: graph
replay, L2 flushed between steps)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

pk = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = bench.measure_norm_sweep_c4(50, flush, pk)
for k, v in res["cases"].items():
    print(f"{k:22s} {v['us_fwd_bwd']:8.2f} us  {v['hbm_frac_effective']:.3f} of HBM")
