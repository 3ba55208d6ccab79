#!/bin/bash
# ncu --set full on the kernels matching $1 (regex) of one eager step of
# tools/profile_step.py; reduces the report to CSV pages on the box
# (details, raw, and the SASS source page with per-instruction stalls).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
PAT=$1; TAG=$2; W=${3:-bert}
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"$PAT" \
  -o /tmp/k_$TAG -f python tools/profile_step.py --workload $W > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/k_$TAG.ncu-rep --page details --csv > gpurun_out/ncu_${TAG}_details.csv 2>/dev/null
ncu -i /tmp/k_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_${TAG}_raw.csv 2>/dev/null
for k in $(echo "$PAT" | tr '|' ' '); do
  ncu -i /tmp/k_$TAG.ncu-rep --page source --csv --print-source sass -k regex:"$k" > gpurun_out/ncu_${TAG}_src_$k.csv 2>&1
done
ls -la gpurun_out | tail -8
