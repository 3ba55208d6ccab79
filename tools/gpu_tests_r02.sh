cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest -s -q -p no:cacheprovider tests/test_gpu_dfir_flow.py tests/test_gpu_syncbn.py "tests/test_gpu_bert.py::test_bert_c2_vs_oracle" "tests/test_gpu_mbconv.py::test_c3_bf16_vs_oracle" "tests/test_gpu_effnet.py::test_bf16_c5_blocks_pinned_to_f64" > gpurun_out/new_tests.log 2>&1
echo "rc=$?" >> gpurun_out/new_tests.log
timeout 1500 python -m pytest -q -p no:cacheprovider tests -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/new_tests.log; tail -3 gpurun_out/pytest_gpu.log
