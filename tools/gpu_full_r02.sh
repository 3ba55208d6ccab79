#!/bin/bash
# One gpurun call at a milestone: the round check (all GPU tests, smoke, bench line of both arms,
# ncu launch list), the ncu DRAM-byte reconciliation of one BERT step, and compute-sanitizer.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
WITH_REF=1 WITH_NCU=1 bash tools/gpu_check_r02.sh
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -c 600 --csv --log-file gpurun_out/dram_step.csv python bench.py --steps 1 --warmup 3 --no-extra --no-cpu-baseline \
  > gpurun_out/dram_step.log 2>&1
python tools/reconcile_bytes.py gpurun_out/dram_step.csv --traffic-out gpurun_out/r02_traffic.json > gpurun_out/reconcile.md 2>&1; echo "reconcile rc=$?"
tail -8 gpurun_out/reconcile.md
[ -n "$WITH_SAN" ] && PER_TOOL_TIMEOUT=600 bash tools/sanitize.sh && python tools/sanitize_summary.py gpurun_out > gpurun_out/sanitize.md
cat gpurun_out/sanitize.md 2>/dev/null
