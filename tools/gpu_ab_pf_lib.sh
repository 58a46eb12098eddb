#!/bin/bash
# A/B of library variants on the prefill forward (tools/prefill_bench.py mla_fwd): per device us, TFLOP/s, K8.
for rep in 1 2; do for v in ${VARIANTS}; do
  TPLA_LIB=build/variants/libtpla_$v.so timeout 300 python tools/prefill_bench.py --L ${LS:-1024 4096} --iters 10 --fwd-only 2>/dev/null | python -c "
import json,sys
for line in sys.stdin:
    try: d=json.loads(line)
    except Exception: continue
    m=d.get('mla_fwd')
    if m: print('$v', d['L'], round(m['fwd_us_per_device'],1), round(m['fwd_tflops']), 'K8', m['fwd_kernels_us_per_device'].get('K8_prefill_fa'))
"
done; done
