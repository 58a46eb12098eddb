#!/bin/bash
# Quick GPU check: gpu parity tests, one K3 trace, default bench line.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
TPLA_K3_MODE=trace TPLA_K3_TRACE_CTA=${TRACE_CTA:-5} timeout 300 python bench.py --steps 2 --warmup 3 --no-graph --no-e2e --no-cpu-baseline > /dev/null 2> gpurun_out/trace.log; echo "trace rc=$?"
grep "span" gpurun_out/trace.log | tail -2
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench.json'))
r=d['roofline']
print('value %.0f tok/s  step %.1f us  e2e %.0f  K3 %.1f us (iso %.1f) hbm_frac %.3f tc_frac %.3f clocks %s' % (d['value'], d['ms_per_step']*1e3, d['e2e']['value'] if d.get('e2e') else 0, r['avg_launch_us'], r['isolated_avg_launch_us'] or 0, r['hbm_frac'], r['tensor_frac_of_sustained'], d['clocks']))
for k,v in d['kernels'].items(): print('  %-20s %7.1f us/step' % (k, v['us_per_step']))
PY
