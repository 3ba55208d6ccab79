#!/bin/bash
# A/B of the attention kernels inside the BERT step (bench without extras)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 120 python tools/attn_time.py
for v in "X=1" "DFX_ATTN_BWD_LEGACY=1" "DFX_ATTN_FWD_LEGACY=1 DFX_ATTN_BWD_LEGACY=1"; do
  env $v timeout 240 python bench.py --steps 30 --warmup 5 --no-extra --no-cpu-baseline > gpurun_out/b_ab.json 2> gpurun_out/b_ab.err
  echo "[$v] rc=$?"
  python - <<'P'
import json
d=json.loads(open("gpurun_out/b_ab.json").read().strip().splitlines()[-1])
print(d["ms_per_step"], d["e2e"]["ms_per_step"], {r["kernel"]: r["us_per_call"] for r in d["kernels"] if "attention" in r["kernel"]})
P
done
