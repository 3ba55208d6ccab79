#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
python tools/dw_shape_profile.py 7 1152 5 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dw_launches.csv python tools/dw_shape_profile.py 7 1152 5 1 > /dev/null 2>&1
python - <<'P'
import csv
rows=[r for r in csv.reader(open("gpurun_out/dw_launches.csv")) if len(r)>5]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value"); gi=h.index("Grid Size"); bi=h.index("Block Size")
seen=0
for r in rows[1:][-14:]:
    print(r[ki][:80], r[gi], r[bi], r[vi])
P
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dw_ring --launch-skip 6 -c 3 -o /tmp/dw -f python tools/dw_shape_profile.py 7 1152 5 1 > gpurun_out/ncu_dw.log 2>&1
ncu -i /tmp/dw.ncu-rep --page details --csv > gpurun_out/ncu_dw_details.csv 2>/dev/null
ncu -i /tmp/dw.ncu-rep --page raw --csv > gpurun_out/ncu_dw_raw.csv 2>/dev/null
ncu -i /tmp/dw.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_dw_src.csv 2>/dev/null
ls -la gpurun_out | grep dw
