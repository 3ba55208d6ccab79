#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_gemm.py tests/test_gpu_effnet.py tests/test_gpu_excite_fold.py tests/test_gpu_library_eval.py > gpurun_out/round_o_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/round_o_tests.log
for v in "X=1" "DFX_NO_SMALL_GEMM=1"; do
  env $v timeout 300 python tools/effnet_profile.py > gpurun_out/effnet_profile.txt 2>&1; echo "[$v]"; head -1 gpurun_out/effnet_profile.txt
  grep -E "b1.backward/block.expand_dgrad|b1.forward/block.expand_gemm|stem.gemm|b0.backward/block.project_dgrad" gpurun_out/effnet_profile.txt
done
