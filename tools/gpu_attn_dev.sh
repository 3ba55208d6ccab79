#!/bin/bash
# attention development loop on the GPU: parity tests and timings of the new
# kernels against the legacy ones (DFX_ATTN_*_LEGACY).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 300 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_attention.py ${EXTRA_TESTS} > gpurun_out/attn_test.log 2>&1
echo "tests rc=$?"; tail -15 gpurun_out/attn_test.log
timeout 120 python tools/attn_time.py > gpurun_out/attn_time.txt 2>&1; echo "new rc=$?"; cat gpurun_out/attn_time.txt
DFX_ATTN_BWD_LEGACY=1 timeout 120 python tools/attn_time.py > gpurun_out/attn_time_legacy.txt 2>&1; echo "legacy"; cat gpurun_out/attn_time_legacy.txt
for v in "X=1" "DFX_ATTN_BWD_LEGACY=1"; do
  env $v timeout 240 python bench.py --steps 30 --warmup 5 --no-extra --no-cpu-baseline > gpurun_out/b_ab.json 2> gpurun_out/b_ab.err
  echo "[$v] rc=$?"
  python - <<'P'
import json
d=json.loads(open("gpurun_out/b_ab.json").read().strip().splitlines()[-1])
print(d["ms_per_step"], d["e2e"]["ms_per_step"], {r["kernel"]: r["us_per_call"] for r in d["kernels"] if "attention" in r["kernel"]})
P
done
