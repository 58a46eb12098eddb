#!/bin/bash
# A/B for the small-batch step: K45 warps-per-row split (k45d vs pre) and the K3 grid floor (TPLA_K3_MIN_BOXES).
TESTS="${TESTS-e2e or full_size or mtp or decode_v or attention}" VARIANTS="pre k45d" WORKLOADS="c1 h8" KERNELS="K45_combine_W_UV K3_attn_tc" STEPS=30 bash tools/gpu_ab_k.sh
for B in 1 4; do
TESTS= VARIANTS="pre k45d k45d:TPLA_K3_MIN_BOXES=8 k45d:TPLA_K3_MIN_BOXES=16" WORKLOADS="c1" BENCH_ARGS="--batch $B" KERNELS="K45_combine_W_UV K3_attn_tc" STEPS=30 bash tools/gpu_ab_k.sh
done
