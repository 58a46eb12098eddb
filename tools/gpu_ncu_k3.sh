#!/bin/bash
# ncu --set full of one K3 launch for a workload (WL, default c1), after the same command ran clean.
mkdir -p gpurun_out
WL=${WL:-c1}
CMD="python bench.py --workload $WL --steps 3 --warmup 3 --no-graph --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/k3_$WL.plain.json 2>&1 || { echo "plain run failed"; exit 1; }
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:attn_tc_kernel -s 2 -c 1 \
  -o gpurun_out/k3_$WL -f $CMD > gpurun_out/k3_$WL.ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/k3_$WL.ncu-rep --page source --csv --print-source sass > gpurun_out/k3_$WL.sass.csv 2>/dev/null
ncu -i gpurun_out/k3_$WL.ncu-rep --page raw --csv > gpurun_out/k3_$WL.raw.csv 2>/dev/null
ls -la gpurun_out/k3_$WL*
