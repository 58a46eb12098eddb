#!/bin/bash
# Round profile evidence (one ncu per call; PASS=launches|full):
#   launches: bench.py clean, then the ncu launch list of the same command
#   full:     bench.py clean, then ncu --set full of the first K3, K5 (W^O) and K45 launches
mkdir -p gpurun_out
CMD="python bench.py --steps 20 --warmup 3 --workload ${WL:-c1} --no-cpu-baseline --no-e2e --no-headline"
timeout 900 $CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err || { echo "plain run failed"; tail -5 gpurun_out/prof_plain.err; exit 1; }
cat gpurun_out/prof_plain.json
if [ "$PASS" = "launches" ]; then
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/prof_launches.csv \
    $CMD > gpurun_out/prof_ncu.json 2> gpurun_out/prof_ncu.err; echo "ncu rc=$?"
else
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"attn_tc_kernel|skinny_tc_kernel|combine_wuv_kernel|attn_plan_kernel|nt_gemm_kernel|pre_attn_kernel" \
    -c 5 -o gpurun_out/prof_full -f $CMD > gpurun_out/prof_ncu.json 2> gpurun_out/prof_ncu.err; echo "ncu rc=$?"
  ncu -i gpurun_out/prof_full.ncu-rep --page raw --csv > gpurun_out/prof_full_raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_full.ncu-rep --page source --csv --print-source sass -k regex:attn_tc_kernel > gpurun_out/prof_k3_sass.csv 2>/dev/null
fi
ls -la gpurun_out/prof_*
