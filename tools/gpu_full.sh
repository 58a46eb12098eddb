#!/bin/bash
# Full check: smoke, the GPU parity suite, the default bench line.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -14 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_default.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_default.json')); r=d['roofline']; h=d.get('headline') or {}
print('value %.0f step %.1f us e2e %.0f | K3 %.1f us hbm %.3f frac %.3f (%s %s) | headline %.1f us hbm %.3f clk %s | cpu %.2f tok/s parity %.2e' % (
  d['value'], d['ms_per_step']*1e3, d['e2e']['value'], r['avg_launch_us'], r['hbm_frac'], r['frac'], r['bound'], r['tensor_peak_choice'],
  h.get('us_per_launch',0), h.get('hbm_frac',0), (h.get('clocks') or {}).get('sm_mhz'), d['cpu_baseline']['value'], d['cpu_baseline']['parity_max_row_rel_err']))
print('clocks', d['clocks'], d['clocks_sustained'])
PY
