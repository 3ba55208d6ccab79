cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
ATTN_ONLY=packed timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_ --launch-skip 1 -c 3 -o /tmp/attn6 -f python tools/attn_time.py > gpurun_out/ncu_attn6.log 2>&1
echo rc=$?
ncu -i /tmp/attn6.ncu-rep --page details --csv > gpurun_out/ncu_attn6_details.csv
ncu -i /tmp/attn6.ncu-rep --page raw --csv > gpurun_out/ncu_attn6_raw.csv
for k in attn_fwd attn_bwd_dq attn_bwd_dkdv; do ncu -i /tmp/attn6.ncu-rep --page source --csv --print-source sass -k regex:$k > gpurun_out/ncu_attn6_src_$k.csv 2>&1; done
cp /tmp/attn6.ncu-rep gpurun_out/attn6.ncu-rep
