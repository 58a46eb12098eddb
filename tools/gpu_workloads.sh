#!/bin/bash
# Bench line per workload (c1 default, c2 Kimi g4, c3 DSV3 g8 128K) on one GPU.
mkdir -p gpurun_out
for w in ${WORKLOADS:-c1 c2 c3}; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "$w rc=$?"
  python - $w <<'PY'
import json,sys
w=sys.argv[1]
d=json.load(open(f'gpurun_out/bench_{w}.json'))
r=d['roofline']
print('%s value %.0f tok/s  step %.1f us  K3 %.1f us (iso %.1f) bound %s frac %.3f hbm_frac %.3f tc_frac %.3f clocks %s' % (w, d['value'], d['ms_per_step']*1e3, r['avg_launch_us'], r['isolated_avg_launch_us'] or 0, r['bound'], r['frac'], r['hbm_frac'], r['tensor_frac_of_sustained'], d['clocks']['sm_mhz']))
for k,v in d['kernels'].items(): print('  %-20s %7.1f us/step  x%.0f' % (k, v['us_per_step'], v['launches_per_step']))
PY
done
