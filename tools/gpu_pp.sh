#!/bin/bash
# PP softmax check: attention / e2e / multi-token parity, then the W_lat <= 128 workloads.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "attention or e2e or multi_token or determin" > gpurun_out/pytest_pp.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_pp.log
summ() {
python - "$1" <<'PY'
import json, sys
d=json.load(open(sys.argv[1]))
r=d['roofline']
print('%s value %.0f tok/s step %.1f us K3 %.1f us (iso %s) frac %.3f (%s) hbm %.3f clocks %s' % (sys.argv[1], d['value'], d['ms_per_step']*1e3, r['avg_launch_us'], r['isolated_avg_launch_us'], r['frac'], r['bound'], r['hbm_frac'], d['clocks'].get('sm_mhz')))
PY
}
for wl in ${WLS:-h8 c3 c2 c2mtp}; do
  timeout 600 python bench.py --workload $wl --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/pp_${wl}.json 2> gpurun_out/pp_${wl}.err; echo "bench $wl rc=$?"
  summ gpurun_out/pp_${wl}.json
done
TPLA_K3_MODE=trace TPLA_K3_TRACE_CTA=5 timeout 300 python bench.py --workload h8 --steps 1 --warmup 3 --no-graph --no-e2e --no-cpu-baseline > /dev/null 2> gpurun_out/trace_pp_h8.log; echo "trace rc=$?"
