#!/bin/bash
# K3 startup trace per library variant (eager, h8): prints the startup events of the last launches.
mkdir -p gpurun_out
for v in ${VARIANTS}; do
TPLA_LIB=build/variants/libtpla_$v.so TPLA_K3_MODE=trace TPLA_K3_TRACE_CTA=${TRACE_CTA:-5} timeout 300 python bench.py --workload ${WL:-h8} --steps 1 --warmup 3 --no-graph --no-e2e --no-cpu-baseline --no-headline > /dev/null 2> gpurun_out/trace_$v.log; echo "$v trace rc=$?"
grep "k3 start" gpurun_out/trace_$v.log | tail -4
grep "span" gpurun_out/trace_$v.log | tail -2
done
