#!/bin/bash
# rank streams A/B on the bench + parity for the co-located sum path + compute-sanitizer on small shapes
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "group_shared or duplicated or project_out or large_batch" > gpurun_out/t_sum.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_sum.log
for w in c1 h8; do for flag in "" "--no-rank-streams"; do
  timeout 300 python bench.py --workload $w --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-headline $flag > gpurun_out/rs_$w$flag.json 2>gpurun_out/rs_$w$flag.err
  python -c "
import json; d=json.load(open('gpurun_out/rs_$w$flag.json')); r=d['roofline']
print('$w $flag step %.1f us  value %.0f  K3 %.1f us hbm %.3f' % (d['ms_per_step']*1e3, d['value'], r['avg_launch_us'], r['hbm_frac']))" || tail -3 gpurun_out/rs_$w$flag.err
done; done
for B in 1 8; do for flag in "" "--no-rank-streams"; do
  timeout 300 python bench.py --workload c1 --batch $B --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-headline $flag > gpurun_out/rsb$B$flag.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/rsb$B$flag.json'))
print('c1 B=$B $flag step %.1f us' % (d['ms_per_step']*1e3))"
done; done
