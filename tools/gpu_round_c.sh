#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_attention.py tests/test_gpu_dp.py > gpurun_out/attn_test.log 2>&1
echo "tests rc=$?"; tail -15 gpurun_out/attn_test.log
ATTN_ONLY=packed timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/attn_launches.csv python tools/attn_time.py > /dev/null 2>&1
python - <<'P'
import csv
rows=[r for r in csv.reader(open("gpurun_out/attn_launches.csv")) if len(r)>5]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
for r in rows[1:]:
    if "dfx" in r[ki]: print(r[ki][:60], r[vi])
P
timeout 120 python tools/attn_time.py; DFX_ATTN_BWD_LEGACY=1 timeout 120 python tools/attn_time.py | tail -1
VARIANTS="X=1" STEPS=3000 bash tools/gpu_hang.sh
for v in "X=1" "DFX_ATTN_BWD_LEGACY=1"; do
  env $v timeout 240 python bench.py --steps 30 --warmup 5 --no-extra --no-cpu-baseline > gpurun_out/b_ab.json 2> gpurun_out/b_ab.err
  echo "[$v] rc=$?"
  python - <<'P'
import json
d=json.loads(open("gpurun_out/b_ab.json").read().strip().splitlines()[-1])
print(d["ms_per_step"], d["e2e"]["ms_per_step"], {r["kernel"]: r["us_per_call"] for r in d["kernels"] if "attention" in r["kernel"]})
P
done
