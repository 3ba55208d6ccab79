#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_excite_fold.py tests/test_gpu_dp.py tests/test_gpu_syncbn.py tests/test_gpu_effnet.py tests/test_gpu_mbconv.py > gpurun_out/round_d_tests.log 2>&1
echo "tests rc=$?"; tail -25 gpurun_out/round_d_tests.log
PYTHONFAULTHANDLER=1 timeout -s ABRT 600 python bench.py --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/bench_d.json 2> gpurun_out/bench_d.err
echo "bench rc=$?"
python - <<'P'
import json
d=json.loads(open("gpurun_out/bench_d.json").read().strip().splitlines()[-1])
print("bert", d["ms_per_step"], d["e2e"]["ms_per_step"])
c5=d["workloads"]["efficientnet_b0_c5"]
print("c5", c5["ms_per_step"], c5["e2e"]["ms_per_step"])
for r in c5["kernels"]: print("  ", r["kernel"], r["us_per_call"], r["calls_per_step"], r["frac"])
P
PER_TOOL_TIMEOUT=600 bash tools/sanitize.sh
