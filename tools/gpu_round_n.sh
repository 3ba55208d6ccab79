#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_norms.py tests/test_gpu_effnet.py > gpurun_out/round_n_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/round_n_tests.log
timeout 300 python tools/effnet_profile.py > gpurun_out/effnet_profile.txt 2>&1; head -3 gpurun_out/effnet_profile.txt; sed -n '/by kernel type/,$p' gpurun_out/effnet_profile.txt | head -8
grep -E "bn_act_bwd_reduce" gpurun_out/effnet_profile.txt | head -5
