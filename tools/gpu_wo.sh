#!/bin/bash
# f2(ii) check: new parity tests, then bench with per-rank vs group-shared W^O on c1 / h8 / c3.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "shared_wo or project_out or nccl" > gpurun_out/pytest_wo.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_wo.log
summ() {
python - "$1" <<'PY'
import json, sys
d=json.load(open(sys.argv[1]))
r=d['roofline']
print('%s value %.0f tok/s step %.1f us e2e %.0f K3 %.1f us frac %.3f (%s) clocks %s' % (sys.argv[1], d['value'], d['ms_per_step']*1e3, d['e2e']['value'] if d.get('e2e') else 0, r['avg_launch_us'], r['frac'], r['bound'], d['clocks'].get('sm_mhz')))
print('   ', {k: round(v['us_per_step'],1) for k,v in d['kernels'].items()})
PY
}
for wl in c1 h8 c3; do
  for wo in rank shared; do
    timeout 600 python bench.py --workload $wl --wo $wo --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/wo_${wl}_${wo}.json 2> gpurun_out/wo_${wl}_${wo}.err; echo "bench $wl $wo rc=$?"
    summ gpurun_out/wo_${wl}_${wo}.json
  done
done
