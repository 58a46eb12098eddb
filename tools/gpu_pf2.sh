#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/prefill_bench.py --L 4096 --iters 5 > gpurun_out/pf_bench.log 2>&1; echo "bench rc=$?"
python -c "
import json
for l in open('gpurun_out/pf_bench.log'):
    if l.startswith('{'):
        d=json.loads(l)['mla_fwd']; print(d['L'], 'fwd us/dev %.0f  TF %.0f attn TF %.0f' % (d['fwd_us_per_device'], d['fwd_tflops'], d['attn_tflops'])); print(d['fwd_kernels_us_per_device'])
"
