#!/bin/bash
# Re-entry check at HEAD: gpu tests, smoke, default bench line, h8 bench line.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py --steps 20 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --workload h8 --steps 20 --no-cpu-baseline > gpurun_out/bench_h8.json 2> gpurun_out/bench_h8.err; echo "bench h8 rc=$?"
