#!/bin/bash
# One ncu --set full capture of the decode kernels (K3, K5 W^O, K45), after the same bench command
# has exited 0 without ncu.  Output: gpurun_out/full.ncu-rep (+ raw csv pages).
mkdir -p gpurun_out
CMD="python bench.py --steps 5 --warmup 3 --no-graph --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/full_plain.json 2> gpurun_out/full_plain.err || { echo "plain run failed"; exit 1; }
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"attn_tc_kernel|skinny_tc_kernel|combine_wuv_kernel" -c 5 -o gpurun_out/full -f $CMD \
  > gpurun_out/full_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/full.ncu-rep --page raw --csv > gpurun_out/full_raw.csv 2>/dev/null
ncu -i gpurun_out/full.ncu-rep --page details --csv > gpurun_out/full_details.csv 2>/dev/null
ls -la gpurun_out/full*
