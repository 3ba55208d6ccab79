#!/bin/bash
# attention development loop on the GPU: parity tests, kernel timings of the
# default path against the A/B switches in $VARIANTS, a hang probe of the
# captured BERT step, and a short bench per variant.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 300 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_attention.py ${EXTRA_TESTS} > gpurun_out/attn_test.log 2>&1
echo "tests rc=$?"; tail -15 gpurun_out/attn_test.log
for v in "X=1" ${VARIANTS}; do
  env $v timeout 120 python tools/attn_time.py > gpurun_out/attn_time_$v.txt 2>&1; echo "[$v] time rc=$?"; cat gpurun_out/attn_time_$v.txt
done
timeout 300 python tools/hang_probe.py ${STEPS:-3000} 20 > gpurun_out/hang.log 2>&1; echo "hang rc=$? $(tail -1 gpurun_out/hang.log)"
for v in "X=1" ${VARIANTS}; do
  env $v timeout 240 python bench.py --steps 30 --warmup 5 --no-extra --no-cpu-baseline > gpurun_out/b_ab.json 2> gpurun_out/b_ab.err
  echo "[$v] bench rc=$?"
  python - <<'P'
import json
d=json.loads(open("gpurun_out/b_ab.json").read().strip().splitlines()[-1])
print(d["ms_per_step"], d["e2e"]["ms_per_step"], {r["kernel"]: r["us_per_call"] for r in d["kernels"] if "attention" in r["kernel"]})
P
done
