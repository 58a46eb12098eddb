mkdir -p gpurun_out
CMD="python bench.py --workload c1 --steps 3 --warmup 3 --no-graph --no-e2e --no-cpu-baseline"
timeout 600 $CMD > /dev/null 2>&1 || { echo plain failed; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"combine_wuv|skinny_tc" -s 2 -c 2 -o gpurun_out/k45 -f $CMD > gpurun_out/k45.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/k45.ncu-rep --page source --csv --print-source sass -k regex:combine_wuv > gpurun_out/k45_sass.csv 2>/dev/null
ncu -i gpurun_out/k45.ncu-rep --page source --csv --print-source sass -k regex:skinny_tc > gpurun_out/k5_sass.csv 2>/dev/null
ncu -i gpurun_out/k45.ncu-rep --page raw --csv > gpurun_out/k45_raw.csv 2>/dev/null
