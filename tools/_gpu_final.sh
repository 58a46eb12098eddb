set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests=$?
timeout 600 python bench.py > gpurun_out/bench_final.log 2>&1; echo bench=$?
tail -3 gpurun_out/gputests.log; tail -2 gpurun_out/bench_final.log
