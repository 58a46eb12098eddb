#!/bin/bash
# K3 balance at HEAD: per-CTA (smid, tiles, segments, end) for h8 and c1, plus the per-tile trace of a
# two-segment CTA (TRACE_CTA) to show the segment switch.
mkdir -p gpurun_out
for W in h8 c1; do
  TPLA_K3_MODE=trace TPLA_K3_TRACE_CTA=${TRACE_CTA:-4} timeout 300 python bench.py --workload $W --steps 1 --warmup 3 --no-graph --no-e2e --no-cpu-baseline --no-headline > /dev/null 2> gpurun_out/bal2_$W.log; echo "trace $W rc=$?"
  grep "ctainfo\] [0-9]" gpurun_out/bal2_$W.log | tail -888 > gpurun_out/bal2_${W}_cta.txt
done
