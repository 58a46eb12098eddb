#!/bin/bash
# Re-entry session evidence at HEAD: GPU suite, smoke, default + h8 bench lines, the W_lat = 64
# per-sequence cost A/B, the c1 launch list and one ncu --set full of the h8 K3.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/final_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/final_smoke.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --workload h8 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/final_bench_h8.json 2> gpurun_out/final_bench_h8.err; echo "bench h8 rc=$?"
VARIANTS="head5 sc640" WORKLOADS="h8 c3" STEPS=50 bash tools/gpu_ab.sh
PASS=launches WL=c1 bash tools/gpu_profile_round.sh > gpurun_out/prof_launches.log 2>&1; echo "launches rc=$?"
M=normal WL=h8 bash tools/gpu_ncu_k3_modes.sh > gpurun_out/ncu_h8.log 2>&1; echo "ncu h8 rc=$?"
