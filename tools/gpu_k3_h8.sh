#!/bin/bash
# K3 at W_lat = 64 (h8 shape): diagnostic modes and a per-tile trace of one CTA.
mkdir -p gpurun_out
W=${WL:-h8}
for m in normal nold notma stream; do
  TPLA_K3_MODE=$m timeout 300 python bench.py --workload $W --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/m_${W}_$m.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/m_${W}_$m.json')); r=d['roofline']
print('$W $m K3 in-step %.1f us iso %.1f  clocks %s' % (r['avg_launch_us'], r['isolated_avg_launch_us'], d['clocks']['sm_mhz']))"
done
for m in trace trace_notma; do
TPLA_K3_MODE=$m TPLA_K3_TRACE_CTA=${TRACE_CTA:-5} timeout 300 python bench.py --workload $W --steps 1 --warmup 3 --no-graph --no-e2e --no-cpu-baseline > /dev/null 2> gpurun_out/trace_${W}_$m.log; echo "$m rc=$?"
done
