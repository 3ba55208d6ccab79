#!/bin/bash
# build, parity of the changed paths, attention A/B, a short bench, the C5 per-block profile, hang probe
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_attention.py tests/test_gpu_rowops.py tests/test_gpu_bert.py \
  tests/test_gpu_excite_fold.py tests/test_gpu_dp.py tests/test_gpu_dfir_flow.py > gpurun_out/round_e_tests.log 2>&1
echo "tests rc=$?"; tail -20 gpurun_out/round_e_tests.log
timeout 120 python tools/attn_time.py; DFX_ATTN_BWD_LEGACY=1 timeout 120 python tools/attn_time.py | tail -1
ATTN_ONLY=packed timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/attn_launches.csv python tools/attn_time.py > /dev/null 2>&1
python - <<'P'
import csv
rows=[r for r in csv.reader(open("gpurun_out/attn_launches.csv")) if len(r)>5]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
for r in rows[1:]:
    if "dfx" in r[ki]: print(r[ki][:70], r[vi])
P
VARIANTS="X=1" STEPS=3000 bash tools/gpu_hang.sh
for v in "X=1" "DFX_ATTN_BWD_LEGACY=1 DFX_EXCITE_FOLD=0"; do
  env $v PYTHONFAULTHANDLER=1 timeout -s ABRT 600 python bench.py --steps 60 --warmup 5 --no-cpu-baseline > gpurun_out/bench_e.json 2> gpurun_out/bench_e.err
  echo "[$v] bench rc=$?"
  python - <<'P'
import json
d=json.loads(open("gpurun_out/bench_e.json").read().strip().splitlines()[-1])
print("bert", d["ms_per_step"], d["e2e"]["ms_per_step"], d["roofline"]["kernel"], d["roofline"]["frac"])
for r in d["kernels"][:8]: print("  ", r["kernel"], r["us_per_call"], r["frac"])
c5=d["workloads"]["efficientnet_b0_c5"]
print("c5", c5["ms_per_step"], c5["e2e"]["ms_per_step"])
c3=d["workloads"]["mbconv_c3"]; print("c3", c3["ms_per_step"])
P
done
timeout 300 python tools/effnet_profile.py > gpurun_out/effnet_profile.txt 2>&1; head -60 gpurun_out/effnet_profile.txt
