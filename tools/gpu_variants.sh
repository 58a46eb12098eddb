#!/bin/bash
# A/B: K3 in-step time per library variant (build/variants/libtpla_*.so) and workload, alternated twice.
mkdir -p gpurun_out
for rep in 1 2; do
for v in ${VARIANTS}; do for w in ${WORKLOADS:-c1 c3}; do
  TPLA_LIB=build/variants/libtpla_$v.so timeout 300 python bench.py --workload $w --steps 100 --no-e2e --no-cpu-baseline > gpurun_out/var_${v}_$w.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/var_${v}_$w.json')); r=d['roofline']
print('$v $w step %.1f us  K3 %.1f us (iso %.1f) clk %s' % (d['ms_per_step']*1e3, r['avg_launch_us'], r['isolated_avg_launch_us'], d['clocks']['sm_mhz']))"
done; done; done
