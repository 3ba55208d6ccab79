#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_excite_fold.py tests/test_gpu_effnet.py > gpurun_out/round_p_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/round_p_tests.log
for v in "X=1" "DFX_EXCITE_FOLD=0"; do
  env $v timeout 300 python tools/effnet_profile.py > gpurun_out/effnet_profile_$v.txt 2>&1; echo "[$v]"; head -1 gpurun_out/effnet_profile_$v.txt
  grep -E "excite_project|project_gemm|bn_swish_se_excite" gpurun_out/effnet_profile_$v.txt | head -8
done
