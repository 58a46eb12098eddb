#!/bin/bash
# K3 per-CTA balance: (smid, tiles, segments, start, end) of every CTA of the last traced launch.
mkdir -p gpurun_out
for W in ${WLS:-h8 c1}; do
  TPLA_K3_MODE=trace TPLA_K3_TRACE_CTA=5 timeout 300 python bench.py --workload $W --steps 1 --warmup 3 --no-graph --no-e2e --no-cpu-baseline --no-headline > /dev/null 2> gpurun_out/bal_$W.log; echo "trace $W rc=$?"
  grep "ctainfo\] [0-9]" gpurun_out/bal_$W.log | tail -1000 > gpurun_out/bal_${W}_cta.txt
done
