#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_mbconv.py tests/test_gpu_effnet.py tests/test_gpu_library_eval.py tests/test_gpu_excite_fold.py > gpurun_out/round_i_tests.log 2>&1
echo "tests rc=$?"; tail -5 gpurun_out/round_i_tests.log
for shp in "7 1152 5 1" "14 672 5 1" "14 480 5 1" "28 240 5 1" "14 480 3 1" "56 144 5 2" "7 1152 3 1"; do python tools/dw_shape_profile.py $shp; done
timeout 300 python tools/effnet_profile.py > gpurun_out/effnet_profile.txt 2>&1; head -3 gpurun_out/effnet_profile.txt; sed -n '/by kernel type/,$p' gpurun_out/effnet_profile.txt | head -8
timeout 300 python tools/mbconv_time.py 2>&1 | tail -6
