cd "${GRAFT_REPO_ROOT:-.}"
VARIANTS="X=1 DFX_ATTN_FWD_LEGACY=1 DFX_ATTN_BWD_LEGACY=1" STEPS=3000 bash tools/gpu_hang.sh
EXTRA_TESTS="tests/test_gpu_dp.py" bash tools/gpu_attn_dev.sh
