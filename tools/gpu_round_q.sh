#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_bert.py tests/test_gpu_attention.py tests/test_gpu_dp.py tests/test_abi.py > gpurun_out/round_q_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/round_q_tests.log
VARIANTS="X=1" STEPS=3000 bash tools/gpu_hang.sh
for i in 1 2; do
PYTHONFAULTHANDLER=1 timeout -s ABRT 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --no-extra > gpurun_out/b_q.json 2> gpurun_out/b_q.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/b_q.json").read().strip().splitlines()[-1])
print("bert", d["ms_per_step"], d["e2e"]["ms_per_step"], d["roofline"]["kernel"], d["roofline"]["frac"])
P
done
