#!/bin/bash
# Round-2 evidence at HEAD: default bench line, launch list of the bench command, ncu --set full of the
# decode kernels (c1 and h8) and of the prefill kernels, prefill TTFT at 1K / 4K.
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
PASS=launches bash tools/gpu_profile_round.sh > gpurun_out/prof_launches.log 2>&1; echo "launches rc=$?"
cp gpurun_out/prof_launches.csv gpurun_out/r02_launches.csv 2>/dev/null
cp gpurun_out/prof_plain.json gpurun_out/r02_launches_cmd.json 2>/dev/null
PASS=full bash tools/gpu_profile_round.sh > gpurun_out/prof_full_c1.log 2>&1; echo "full c1 rc=$?"
cp gpurun_out/prof_full_raw.csv gpurun_out/r02_full_c1_raw.csv; cp gpurun_out/prof_k3_sass.csv gpurun_out/r02_k3_c1_sass.csv
WL=h8 PASS=full bash tools/gpu_profile_round.sh > gpurun_out/prof_full_h8.log 2>&1; echo "full h8 rc=$?"
cp gpurun_out/prof_full_raw.csv gpurun_out/r02_full_h8_raw.csv; cp gpurun_out/prof_k3_sass.csv gpurun_out/r02_k3_h8_sass.csv
if [ -z "$NO_PREFILL" ]; then
bash tools/gpu_ncu_pf.sh > gpurun_out/prof_pf.log 2>&1; echo "prefill ncu rc=$?"
timeout 600 python tools/prefill_bench.py --L 1024 4096 --iters 10 > gpurun_out/r02_prefill.jsonl 2>&1; echo "prefill bench rc=$?"
fi
ls -la gpurun_out/r02_*
