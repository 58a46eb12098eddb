#!/bin/bash
# K3 change check: attention/e2e/mtp parity, then bench lines (no e2e/cpu) and one trace.
mkdir -p gpurun_out
TAG=${TAG:-k3}
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "attention or e2e or multi_token or determin" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
for wl in ${WLS:-h8 c3 c1 c2}; do
  timeout 600 python bench.py --workload $wl --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_${wl}.json 2> gpurun_out/${TAG}_${wl}.err; echo "bench $wl rc=$?"
python - gpurun_out/${TAG}_${wl}.json <<'PY'
import json, sys
d=json.load(open(sys.argv[1]))
r=d['roofline']
print('%s value %.0f tok/s step %.1f us K3 %.1f us (iso %s) frac %.3f (%s) hbm %.3f clocks %s' % (sys.argv[1], d['value'], d['ms_per_step']*1e3, r['avg_launch_us'], r['isolated_avg_launch_us'], r['frac'], r['bound'], r['hbm_frac'], d['clocks'].get('sm_mhz')))
PY
done
TPLA_K3_MODE=trace TPLA_K3_TRACE_CTA=5 timeout 300 python bench.py --workload ${TRACE_WL:-h8} --steps 1 --warmup 3 --no-graph --no-e2e --no-cpu-baseline > /dev/null 2> gpurun_out/trace_$TAG.log; echo "trace rc=$?"
grep "k3 start" gpurun_out/trace_$TAG.log | tail -1; grep "k3 cta\]" gpurun_out/trace_$TAG.log | grep -E "traced|span|  5 start" | tail -3
