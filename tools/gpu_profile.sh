#!/bin/bash
# ncu --set full of every kernel of one eager C2 step and one C3 MBConv step.
# Reports are reduced to CSV on the box (the .ncu-rep files exceed gpurun's
# 64 MiB return limit); pass KEEP=1 to keep a report for a single kernel.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${1:-r01}
for W in ${WORKLOADS:-bert mbconv}; do
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -o /tmp/${W}_$TAG -f python tools/profile_step.py --workload $W > gpurun_out/ncu_${W}_$TAG.log 2>&1
  echo "$W rc=$?"
  ncu -i /tmp/${W}_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_${W}_${TAG}_raw.csv 2>/dev/null
  ncu -i /tmp/${W}_$TAG.ncu-rep --page details --csv > gpurun_out/ncu_${W}_${TAG}_details.csv 2>/dev/null
done
ls -la gpurun_out
