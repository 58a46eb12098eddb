#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill_mla_forward" > gpurun_out/pf_tests.log 2>&1; echo "tests rc=$?"; grep -E "^E  |passed|failed|Error" gpurun_out/pf_tests.log | head -8
timeout 600 python tools/prefill_bench.py --L 1024 4096 --iters 10 > gpurun_out/pf_bench.log 2>&1; echo "bench rc=$?"; tail -4 gpurun_out/pf_bench.log
