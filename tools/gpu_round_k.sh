#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_mbconv.py tests/test_gpu_effnet.py tests/test_gpu_library_eval.py > gpurun_out/round_k_tests.log 2>&1
echo "tests rc=$?"; tail -5 gpurun_out/round_k_tests.log
for shp in "56 144 5 2" "112 96 3 2" "14 672 5 2"; do python tools/dw_shape_profile.py $shp; DFX_DW_DX_S2_V2=1 python tools/dw_shape_profile.py $shp; done
timeout 300 python tools/effnet_profile.py > gpurun_out/effnet_profile.txt 2>&1; head -3 gpurun_out/effnet_profile.txt; sed -n '/by kernel type/,$p' gpurun_out/effnet_profile.txt | head -8
