#!/bin/bash
# K3 grid floor (TPLA_K3_MIN_BOXES) over small-batch shapes: step time per (context, batch, floor).
mkdir -p gpurun_out
for S in 4096 32768 65536; do for B in 1 2 8; do for mb in 4 8 16; do
  TPLA_K3_MIN_BOXES=$mb timeout 300 python bench.py --workload c1 --batch $B --seq-len $S --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-headline > gpurun_out/mb_${S}_${B}_$mb.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/mb_${S}_${B}_$mb.json')); ks=d['kernels']
print('S=$S B=$B min_boxes=$mb step %.1f us  K3 %.1f  K45 %.1f' % (d['ms_per_step']*1e3, ks['K3_attn_tc']['us_per_step'], ks['K45_combine_W_UV']['us_per_step']))" || echo "S=$S B=$B mb=$mb failed"
done; done; done
