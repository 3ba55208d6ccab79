#!/bin/bash
# compute-sanitizer memcheck + racecheck over the attention and normalisation
# tests that exercise the final kernels (persistent attention forward /
# key-strip backward incl. multi-strip grids, LN/BN finalize paths).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
SEL=(
  "tests/test_gpu_attention.py::test_attention_vs_oracle[2-2-128]"
  "tests/test_gpu_attention.py::test_attention_vs_oracle[24-12-128]"
  "tests/test_gpu_attention.py::test_attention_vs_oracle[4-16-384]"
  "tests/test_gpu_attention.py::test_qkv_bias_grad_from_strip_partials[2-2-128]"
  "tests/test_gpu_attention.py::test_attention_online_rescale"
  "tests/test_gpu_norms.py::test_golden_ln_bn_swish"
)
for tool in memcheck racecheck synccheck; do
  : > gpurun_out/sanq_$tool.txt
  for t in "${SEL[@]}"; do
    extra=""; [ "$tool" = racecheck ] && extra="--racecheck-report hazard"
    timeout 900 compute-sanitizer --tool $tool $extra --print-limit 20 python -m pytest -q -x -p no:cacheprovider "$t" > gpurun_out/sanq_one.log 2>&1
    rc=$?
    summ=$(grep -E "(ERROR|RACECHECK) SUMMARY" gpurun_out/sanq_one.log | tail -1)
    echo "$t | rc=$rc | $summ" >> gpurun_out/sanq_$tool.txt
  done
  cat gpurun_out/sanq_$tool.txt
done
