#!/bin/bash
# A/B of library variants on the per-kernel breakdown (event-bracketed, one stream) and the step time.
# VARIANTS="a b" WORKLOADS="c1 h8" KERNELS="K45_combine_W_UV K2_absorb_q" [TESTS=...] bash tools/gpu_ab_k.sh
# A variant "lib:VAR=1" runs build/variants/libtpla_lib.so with the environment variable VAR=1.
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then
  timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "$TESTS" > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/ab_tests.log
fi
for rep in 1 2; do
for v in ${VARIANTS}; do for w in ${WORKLOADS:-c1 h8}; do
  lib=${v%%:*}; envv=""; [ "$lib" != "$v" ] && envv=${v#*:}
  env $envv TPLA_LIB=build/variants/libtpla_$lib.so timeout 300 python bench.py --workload $w --steps ${STEPS:-50} --warmup 5 --no-e2e --no-cpu-baseline --no-headline $BENCH_ARGS > gpurun_out/vk_${v//[:=]/_}_$w.json 2>gpurun_out/vk_${v//[:=]/_}_$w.err
  KERNELS="$KERNELS" python -c "
import json, os; d=json.load(open('gpurun_out/vk_${v//[:=]/_}_$w.json')); ks=d['kernels']
sel=os.environ['KERNELS'].split() or list(ks)
print('$v $w step %.1f us clk %s | ' % (d['ms_per_step']*1e3, d['clocks']['sm_mhz']) + '  '.join('%s %.1f' % (k, ks[k]['us_per_step']) for k in sel if k in ks))" || tail -3 gpurun_out/vk_${v//[:=]/_}_$w.err
done; done; done
