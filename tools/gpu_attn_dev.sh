#!/bin/bash
# attention development loop on the GPU: parity tests (fused backward, then the
# swapped dS-descriptor variant) and timings of the fused vs the legacy pair.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for v in ""; do
  env $v timeout 300 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_attention.py > "gpurun_out/attn_test${v:+_swap}.log" 2>&1
  echo "[$v] rc=$?"; tail -3 "gpurun_out/attn_test${v:+_swap}.log"
done
timeout 120 python tools/attn_time.py > gpurun_out/attn_time.txt 2>&1; echo "fused rc=$?"; cat gpurun_out/attn_time.txt
DFX_ATTN_BWD_LEGACY=1 timeout 120 python tools/attn_time.py > gpurun_out/attn_time_legacy.txt 2>&1; echo "legacy"; cat gpurun_out/attn_time_legacy.txt
timeout 120 python tools/attn_trace.py --fused > gpurun_out/attn_trace_fused.txt 2>&1; cat gpurun_out/attn_trace_fused.txt
