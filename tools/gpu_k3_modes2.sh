#!/bin/bash
# K3 limiter isolation at one workload: normal / notma / nosm (notma + no softmax) / nomma (notma + no MMA) / nosm_tma
W=${WL:-h8}
for m in normal notma nosm nomma nosm_tma stream; do
  TPLA_K3_MODE=$m timeout 300 python bench.py --workload $W --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/m2_${W}_$m.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/m2_${W}_$m.json')); r=d['roofline']
print('$W %-9s K3 in-step %.1f us iso %.1f  clocks %s' % ('$m', r['avg_launch_us'], r['isolated_avg_launch_us'], d['clocks']['sm_mhz']))"
done
