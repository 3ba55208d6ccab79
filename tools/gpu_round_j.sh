#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for shp in "56 144 5 2" "112 96 3 2" "28 240 5 1"; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/dw_l.csv python tools/dw_shape_profile.py $shp > /dev/null 2>&1
echo "== $shp"
python - <<'P'
import csv
rows=[r for r in csv.reader(open("gpurun_out/dw_l.csv")) if len(r)>5]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value"); ni=h.index("Metric Name"); gi=h.index("Grid Size"); bi=h.index("Block Size"); ii=h.index("ID")
d={}
order=[]
for r in rows[1:]:
    k=r[ii]
    if k not in d: d[k]={"name":r[ki][:60],"grid":r[gi],"block":r[bi]}; order.append(k)
    d[k][r[ni]]=r[vi]
for k in order[-13:]:
    x=d[k]; print(x["name"], x["grid"], x["block"], x.get("gpu__time_duration.sum"), x.get("dram__bytes_read.sum"), x.get("dram__bytes_write.sum"), x.get("sm__throughput.avg.pct_of_peak_sustained_elapsed"))
P
done
