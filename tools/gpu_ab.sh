#!/bin/bash
# A/B of env switches on the BERT C2 bench (short runs, alternating twice) after the given tests;
# a variant joins several VAR=value settings with "+"
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
if [ -n "$TESTS" ]; then timeout 900 python -m pytest -q -x -p no:cacheprovider $TESTS 2>&1 | tail -4; fi
for rep in 1 2; do
for v in "X=1" ${VARIANTS}; do
  env ${v//+/ } timeout 300 python bench.py --steps 60 --warmup 5 --no-extra --no-cpu-baseline > gpurun_out/b_ab.json 2> gpurun_out/b_ab.err
  python - "$v" <<'P'
import json, sys
d = json.loads(open("gpurun_out/b_ab.json").read().strip().splitlines()[-1])
ks = {r["kernel"]: r["us_per_call"] for r in d["kernels"]}
sel = {k: v for k, v in ks.items() if any(t in k for t in (sys.argv[2:] or ["attention", "ffn"]))}
print(f"[{sys.argv[1]}] {d['ms_per_step']} e2e {d['e2e']['ms_per_step']} clk {d['clocks']['sm_mhz']}", sel)
P
done
done
