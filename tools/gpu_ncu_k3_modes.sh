#!/bin/bash
# ncu source-level capture of one K3 launch of workload WL in K3 mode M (default h8 / nosm).
mkdir -p gpurun_out
WL=${WL:-h8}; M=${M:-nosm}
CMD="python bench.py --workload $WL --steps 2 --warmup 2 --no-graph --no-e2e --no-cpu-baseline"
TPLA_K3_MODE=$M timeout 600 $CMD > /dev/null 2>&1 || { echo "plain run failed"; exit 1; }
TPLA_K3_MODE=$M timeout 1200 ncu --set full --clock-control none --import-source on -k regex:attn_tc_kernel -s 2 -c 1 \
  -o gpurun_out/k3_${WL}_$M -f $CMD > gpurun_out/k3_${WL}_$M.ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/k3_${WL}_$M.ncu-rep --page source --csv --print-source sass > gpurun_out/k3_${WL}_$M.sass.csv 2>/dev/null
ncu -i gpurun_out/k3_${WL}_$M.ncu-rep --page raw --csv > gpurun_out/k3_${WL}_$M.raw.csv 2>/dev/null
ls -la gpurun_out/k3_${WL}_$M*
