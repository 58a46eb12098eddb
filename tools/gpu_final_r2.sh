#!/bin/bash
# End-of-round evidence at HEAD: GPU suite, smoke, the default bench line, the prefill TTFT table.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/final_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/final_smoke.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
timeout 900 python tools/prefill_bench.py --L 1024 4096 --iters 10 > gpurun_out/r02_prefill.jsonl 2> gpurun_out/r02_prefill.err; echo "prefill rc=$?"
