#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
ATTN_ONLY=packed timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/attn_launches.csv python tools/attn_time.py > /dev/null 2>&1
python - <<'P'
import csv
rows=[r for r in csv.reader(open("gpurun_out/attn_launches.csv")) if len(r)>5]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
for r in rows[1:]: print(r[ki][:60], r[vi])
P
VARIANTS="X=1 DFX_ATTN_FWD2_ONE=1" STEPS=3000 bash tools/gpu_hang.sh
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_attention.py tests/test_gpu_dp.py > gpurun_out/attn_test.log 2>&1
echo "tests rc=$?"; tail -15 gpurun_out/attn_test.log
