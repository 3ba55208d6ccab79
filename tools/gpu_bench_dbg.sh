#!/bin/bash
# gpurun helper: build, the data-parallel tests, then bench.py with stderr breadcrumbs and a
# faulthandler traceback if it runs past the limit (SIGABRT)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
if [ -n "$TESTS" ]; then timeout 900 python -m pytest -q -p no:cacheprovider $TESTS > gpurun_out/quick.log 2>&1; echo "rc=$?" >> gpurun_out/quick.log; tail -5 gpurun_out/quick.log; fi
PYTHONFAULTHANDLER=1 timeout -s ABRT ${BENCH_LIMIT:-700} python bench.py $BENCH_ARGS > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
tail -40 gpurun_out/bench.err
head -c 600 gpurun_out/bench.json
