#!/bin/bash
# ncu --set full of every kernel of one eager C2 step and one C3 MBConv step.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${1:-r01}
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -o gpurun_out/bert_step_$TAG -f python tools/profile_step.py --workload bert > gpurun_out/ncu_bert_$TAG.log 2>&1
echo "bert rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -o gpurun_out/mbconv_step_$TAG -f python tools/profile_step.py --workload mbconv > gpurun_out/ncu_mbconv_$TAG.log 2>&1
echo "mbconv rc=$?"
tail -3 gpurun_out/ncu_bert_$TAG.log gpurun_out/ncu_mbconv_$TAG.log
