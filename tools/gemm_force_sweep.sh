#!/bin/bash
# Time each BERT C2 GEMM shape under every forced tile config (DFX_GEMM_FORCE=cg,bn).
cd "${GRAFT_REPO_ROOT:-.}"
for f in "" 2,256 2,192 2,128 1,256 1,192 1,128; do
  echo "== force '$f'"
  DFX_GEMM_FORCE=$f python - <<'PY'
import os, sys
sys.path.insert(0, ".")
import torch
from tools.gemm_vs_cublas import timeit
from paper_2110_10802_b200 import kernels as K
for name, m, n, k in [("out", 4096, 768, 768), ("qkv", 4096, 2304, 768), ("ffn1", 4096, 3072, 768), ("ffn2", 4096, 768, 3072), ("big", 8192, 8192, 8192)]:
    a = torch.randn(m, k, device="cuda").bfloat16(); b = torch.randn(n, k, device="cuda").bfloat16()
    d = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    us = timeit(lambda: K.gemm(a, b, d), reps=10 if name == "big" else 20)
    print(f"  {name:5s} {us:8.2f} us {2*m*n*k/us/1e6:7.1f} TF/s")
PY
done
