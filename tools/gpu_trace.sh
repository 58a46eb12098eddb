#!/bin/bash
# K3 per-tile / startup trace of one CTA for a workload (eager, no graph).
mkdir -p gpurun_out
W=${WL:-h8}
TPLA_K3_MODE=trace TPLA_K3_TRACE_CTA=${TRACE_CTA:-5} timeout 300 python bench.py --workload $W --steps 1 --warmup 3 --no-graph --no-e2e --no-cpu-baseline --no-headline > /dev/null 2> gpurun_out/trace_$W.log; echo "trace rc=$?"
grep "k3 start" gpurun_out/trace_$W.log | tail -4
