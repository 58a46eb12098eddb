#!/bin/bash
# Round 2, first GPU pass: smoke, the GPU parity suite, the default bench line, and an h8 K3 trace.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_c1.err
timeout 300 python bench.py --workload h8 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-headline > gpurun_out/bench_h8.json 2> gpurun_out/bench_h8.err; echo "bench h8 rc=$?"
TPLA_K3_MODE=trace TPLA_K3_TRACE_CTA=5 timeout 300 python bench.py --workload h8 --steps 1 --warmup 3 --no-graph --no-e2e --no-cpu-baseline --no-headline > /dev/null 2> gpurun_out/trace_h8.log; echo "trace rc=$?"
