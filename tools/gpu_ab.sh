#!/bin/bash
# A/B of library variants: parity subset on the first variant, then K3 in-step / isolated per variant and workload.
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then
  timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "$TESTS" > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/ab_tests.log
fi
for rep in 1 2; do
for v in ${VARIANTS}; do for w in ${WORKLOADS:-h8 c3}; do
  TPLA_LIB=build/variants/libtpla_$v.so timeout 300 python bench.py --workload $w --steps ${STEPS:-50} --warmup 5 --no-e2e --no-cpu-baseline --no-headline > gpurun_out/var_${v}_$w.json 2>gpurun_out/var_${v}_$w.err
  python -c "
import json; d=json.load(open('gpurun_out/var_${v}_$w.json')); r=d['roofline']
print('$v $w step %.1f us  K3 %.1f us (iso %.1f) hbm %.3f clk %s/%s' % (d['ms_per_step']*1e3, r['avg_launch_us'], r['isolated_avg_launch_us'], r['hbm_frac'], d['clocks']['sm_mhz'], d['clocks_sustained']['sm_mhz']))" || tail -3 gpurun_out/var_${v}_$w.err
done; done; done
