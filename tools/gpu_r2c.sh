#!/bin/bash
mkdir -p gpurun_out
bash tools/gpu_sanitize.sh
for w in c2 c3 c1; do for flag in "" "--no-rank-streams"; do
  timeout 300 python bench.py --workload $w --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-headline $flag > gpurun_out/rs_$w$flag.json 2>gpurun_out/rs_$w$flag.err
  python -c "
import json; d=json.load(open('gpurun_out/rs_$w$flag.json')); r=d['roofline']
print('$w $flag step %.1f us  value %.0f  K3 %.1f us hbm %.3f' % (d['ms_per_step']*1e3, d['value'], r['avg_launch_us'], r['hbm_frac']))" || tail -3 gpurun_out/rs_$w$flag.err
done; done
