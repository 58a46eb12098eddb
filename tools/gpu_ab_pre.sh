#!/bin/bash
# A/B: fused K3p + K2 launch vs the separate kernels (TPLA_PRE_SPLIT=1), same library.
TESTS="${TESTS-e2e or full_size or mtp or decode_v or attention}" VARIANTS="pre:TPLA_PRE_SPLIT=1 pre" WORKLOADS="c1 h8" KERNELS="K3p_attn_plan K2_absorb_q K3p_K2_pre_attn" STEPS=30 bash tools/gpu_ab_k.sh
TESTS= VARIANTS="pre:TPLA_PRE_SPLIT=1 pre" WORKLOADS="c1" BENCH_ARGS="--batch 1" KERNELS="K3p_attn_plan K2_absorb_q K3p_K2_pre_attn" STEPS=30 bash tools/gpu_ab_k.sh
for v in 1 0; do
TPLA_PRE_SPLIT=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"attn_plan|nt_gemm|pre_attn" -c 6 --csv python bench.py --workload c1 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-headline 2>/dev/null | grep -E "attn_plan|nt_gemm|pre_attn" | awk -F'","' -v v=$v '{print "split=" v, $5, $(NF-2), $NF}' | tr -d '"' | cut -c1-150 | tail -6
done
