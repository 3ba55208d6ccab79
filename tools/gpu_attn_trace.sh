#!/bin/bash
# per-CTA timeline of the persistent key-strip backward, then (WITH_NCU) ncu --set full of it
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 120 python tools/attn_trace.py --kstrip
if [ -n "$WITH_NCU" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:kstrip -c 1 -o /tmp/ks -f python tools/attn_time.py > gpurun_out/ncu_ks.log 2>&1
  ncu -i /tmp/ks.ncu-rep --page raw --csv > gpurun_out/ncu_ks_raw.csv 2>/dev/null
  ncu -i /tmp/ks.ncu-rep --page details --csv > gpurun_out/ncu_ks_details.csv 2>/dev/null
  ncu -i /tmp/ks.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_ks_src.csv 2>/dev/null
fi
