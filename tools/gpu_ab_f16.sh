#!/bin/bash
# A/B: fp16 normalised split-K partials (f16) vs fp32 partials (base).
TESTS="${TESTS-attention or e2e or full_size or mtp or decode_v or prefill or c_example or smoke}" VARIANTS="base f16" WORKLOADS="c1 h8 c3" KERNELS="K3_attn_tc K45_combine_W_UV" STEPS=30 bash tools/gpu_ab_k.sh
TESTS= VARIANTS="base f16" WORKLOADS="c1" BENCH_ARGS="--batch 1" KERNELS="K3_attn_tc K45_combine_W_UV" STEPS=30 bash tools/gpu_ab_k.sh
