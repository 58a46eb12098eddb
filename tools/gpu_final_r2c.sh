#!/bin/bash
# Final evidence at HEAD (after the K45 shift change): GPU suite, smoke, default bench line.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final2_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/final2_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/final2_smoke.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/final2_bench.json 2> gpurun_out/final2_bench.err; echo "bench rc=$?"
