#!/bin/bash
# ncu --set full of one forward + one backward launch of the fused attention at
# the C2 shape (tools/attn_time.py ATTN_ONLY=packed); TAG names the outputs.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
TAG=${TAG:-attn}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
ATTN_ONLY=packed timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_ --launch-skip ${SKIP:-2} -c ${COUNT:-2} -o /tmp/$TAG -f python tools/attn_time.py > gpurun_out/ncu_$TAG.log 2>&1
echo rc=$?
ncu -i /tmp/$TAG.ncu-rep --page details --csv > gpurun_out/ncu_${TAG}_details.csv
ncu -i /tmp/$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_${TAG}_raw.csv
for k in ${KERNELS:-attn_fwd attn_bwd_kernel}; do ncu -i /tmp/$TAG.ncu-rep --page source --csv --print-source sass -k regex:$k > gpurun_out/ncu_${TAG}_src_$k.csv 2>&1; done
