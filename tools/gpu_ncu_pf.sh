#!/bin/bash
mkdir -p gpurun_out
python tools/pf_one.py > /dev/null 2>&1 || { echo "pf_one failed"; exit 1; }
for k in attn_fwd gemm_tn; do
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:$k -s 1 -c 1 -o gpurun_out/ncu_pf_$k -f python tools/pf_one.py > gpurun_out/ncu_pf_$k.log 2>&1; echo "ncu $k rc=$?"
ncu -i gpurun_out/ncu_pf_$k.ncu-rep --page raw --csv > gpurun_out/ncu_pf_${k}_raw.csv 2>/dev/null
ncu -i gpurun_out/ncu_pf_$k.ncu-rep --page details --csv > gpurun_out/ncu_pf_${k}_details.csv 2>/dev/null
done
