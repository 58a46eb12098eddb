#!/bin/bash
# Round evidence: gpu tests, smoke, default bench, per-workload bench lines, ncu launch list,
# ncu --set full of the c1 kernels and of the h8 K3.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
for wl in c2 c3 h8 h8g2 c2mtp mla1 mla2; do
  timeout 600 python bench.py --workload $wl --no-cpu-baseline > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err; echo "bench $wl rc=$?"
done
PASS=launches bash tools/gpu_profile_round.sh > gpurun_out/prof_launches.log 2>&1; echo "launches rc=$?"
bash tools/gpu_ncu_full.sh > gpurun_out/ncu_full_c1.log 2>&1; echo "ncu c1 rc=$?"
M=normal WL=h8 bash tools/gpu_ncu_k3_modes.sh > gpurun_out/ncu_h8.log 2>&1; echo "ncu h8 rc=$?"
