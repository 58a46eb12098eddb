#!/bin/bash
# A/B of library variants: K3 in-step (normal) and iso (nosm) on workloads
VARIANTS="${VARIANTS}" WORKLOADS="${WORKLOADS:-h8 c3 c1}" bash tools/gpu_variants.sh
for v in ${VARIANTS}; do TPLA_LIB=build/variants/libtpla_$v.so TPLA_K3_MODE=nosm timeout 300 python bench.py --workload h8 --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/nosm_$v.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/nosm_$v.json')); r=d['roofline']; print('$v nosm iso', r['isolated_avg_launch_us'])"; done
