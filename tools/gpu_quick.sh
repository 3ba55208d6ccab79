#!/bin/bash
# gpurun helper: build, then run the pytest node ids given as arguments (-s, output in gpurun_out/quick.log)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout ${QUICK_TIMEOUT:-1200} python -m pytest -s -q -p no:cacheprovider "$@" > gpurun_out/quick.log 2>&1
echo "rc=$?" >> gpurun_out/quick.log
tail -5 gpurun_out/quick.log
