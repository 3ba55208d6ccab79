#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over small
# shapes of every kernel family (GEMM tc + simt, attention, depthwise ring,
# row kernels, norms, MBConv, EfficientNet glue).  One gpurun call:
#   gpurun --timeout 2400 -- bash tools/sanitize.sh
# Logs land in gpurun_out/sanitize_<tool>.log; tools/sanitize_summary.py
# condenses them into profiles/.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
SEL=(
  "tests/test_gpu_gemm.py::test_tc_gemm_layouts[128-64-512-k-k]"
  "tests/test_gpu_gemm.py::test_tc_gemm_layouts[256-320-192-m-n]"
  "tests/test_gpu_gemm.py::test_gemm_epilogues[True-bias_gelu]"
  "tests/test_gpu_gemm.py::test_gemm_epilogues[False-gelu_bwd]"
  "tests/test_gpu_gemm.py::test_gemm_epilogues[True-add]"
  "tests/test_gpu_gemm.py::test_tc_192_tiles[k-k-none-2,192]"
  "tests/test_gpu_gemm.py::test_tc_ragged_m_k[300-96-16-k-k]"
  "tests/test_gpu_gemm.py::test_simt_f32[130-70-33]"
  "tests/test_gpu_excite_fold.py::test_gemm_excite_vs_torch[1-100-24-16]"
  "tests/test_gpu_attention.py::test_attention_vs_oracle[2-2-128]"
  "tests/test_gpu_attention.py::test_qkv_bias_grad_from_strip_partials[2-2-128]"
  "tests/test_gpu_attention.py::test_attention_online_rescale"
  "tests/test_gpu_rowops.py::test_bdrln[37-64-dtype0]"
  "tests/test_gpu_rowops.py::test_bdrln[256-768-dtype1]"
  "tests/test_gpu_rowops.py::test_bdrln_packed_keep_identical[37-64-dtype1]"
  "tests/test_gpu_rowops.py::test_softmax[2-3-16-64-dtype1]"
  "tests/test_gpu_rowops.py::test_bias_gelu"
  "tests/test_gpu_rowops.py::test_colsum_strided"
  "tests/test_gpu_rowops.py::test_sgd_update_vector_and_scalar_paths[1001-0]"
  "tests/test_gpu_mbconv.py::test_vs_oracle[1-pads4-9-dtype0]"
  "tests/test_gpu_mbconv.py::test_vs_oracle[2-pads3-19-dtype1]"
  "tests/test_gpu_mbconv.py::test_5x5_vs_oracle[1-7-144-dtype1]"
  "tests/test_gpu_norms.py::test_golden_ln_bn_swish"
  "tests/test_gpu_library_eval.py::test_batchnorm_training"
  "tests/test_gpu_library_eval.py::test_depthwise_conv"
)
# memcheck / synccheck over the whole selection (one process each)
for tool in ${TOOLS:-memcheck synccheck}; do
  timeout ${PER_TOOL_TIMEOUT:-900} /usr/local/cuda/bin/compute-sanitizer --tool "$tool" \
    --kernel-name-exclude kns=at6native --print-limit 200 --log-file "gpurun_out/sanitize_${tool}.log" \
    python -m pytest -q -p no:cacheprovider "${SEL[@]}" > "gpurun_out/sanitize_${tool}.pytest" 2>&1
  echo "rc=$?" >> "gpurun_out/sanitize_${tool}.pytest"
  tail -1 "gpurun_out/sanitize_${tool}.log"
done
# racecheck / initcheck per test (a hazard count per kernel family, print-limited)
for tool in ${PER_TEST_TOOLS:-racecheck initcheck}; do
  : > "gpurun_out/sanitize_${tool}_per_test.txt"
  for t in "${SEL[@]}"; do
    extra=""
    [ "$tool" = "racecheck" ] && extra="--racecheck-report hazard"
    timeout 300 /usr/local/cuda/bin/compute-sanitizer --tool "$tool" $extra --kernel-name-exclude kns=at6native \
      --print-limit 4 --log-file gpurun_out/san_one.log python -m pytest -q -p no:cacheprovider "$t" > gpurun_out/san_one.pytest 2>&1
    rc=$?
    summ=$(grep -E "(ERROR|RACECHECK) SUMMARY" gpurun_out/san_one.log | tail -1 | sed 's/=========//')
    kern=$(grep -oE "at (void )?dfx::[^(]*" gpurun_out/san_one.log | sed 's/at void //; s/at //; s/dfx:://; s/<unnamed>:://' | sort | uniq -c | sort -rn | head -3 | awk '{c=$1; $1=""; printf "%s(x%s) ", $0, c}')
    echo "$t | rc=$rc | ${summ:-no summary} | ${kern}" >> "gpurun_out/sanitize_${tool}_per_test.txt"
  done
  cat "gpurun_out/sanitize_${tool}_per_test.txt"
done
