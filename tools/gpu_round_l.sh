#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_attention.py tests/test_gpu_bert.py > gpurun_out/round_l_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/round_l_tests.log
for v in "X=1" "DFX_ATTN_DS_TMA=1"; do
  echo "[$v]"; env $v timeout 120 python tools/attn_time.py | tail -1
  env $v PYTHONFAULTHANDLER=1 timeout -s ABRT 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-extra > gpurun_out/b_l.json 2> gpurun_out/b_l.err
  python - <<'P'
import json
d=json.loads(open("gpurun_out/b_l.json").read().strip().splitlines()[-1])
print("bert", d["ms_per_step"], d["e2e"]["ms_per_step"], {r["kernel"]: r["us_per_call"] for r in d["kernels"] if "attention" in r["kernel"]})
P
done
ATTN_ONLY=packed timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/attn_launches.csv python tools/attn_time.py > /dev/null 2>&1
python - <<'P'
import csv
rows=[r for r in csv.reader(open("gpurun_out/attn_launches.csv")) if len(r)>5]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
for r in rows[1:]:
    if "dfx" in r[ki]: print(r[ki][:70], r[vi])
P
