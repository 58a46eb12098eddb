#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "two_stages" > gpurun_out/t_stage.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/t_stage.log
for rep in 1 2; do for w in c1 h8 c3; do for m in pre full off; do
  timeout 300 python bench.py --workload $w --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-headline --rank-streams $m > gpurun_out/rs_$w$m.json 2>gpurun_out/rs_$w$m.err
  python -c "
import json; d=json.load(open('gpurun_out/rs_$w$m.json')); r=d['roofline']
print('$w $m step %.1f us  value %.0f  K3 %.1f us clk %s' % (d['ms_per_step']*1e3, d['value'], r['avg_launch_us'], d['clocks']['sm_mhz']))" || tail -3 gpurun_out/rs_$w$m.err
done; done; done
