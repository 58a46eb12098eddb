#!/bin/bash
# Bench lines of the other workloads at HEAD (K3 in-step per shard), and batch 1 at 32K / 4K (g = 2).
mkdir -p gpurun_out
for wl in c2 c3 h8g2 c2mtp; do
  timeout 600 python bench.py --workload $wl --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-headline > gpurun_out/wl_$wl.json 2> gpurun_out/wl_$wl.err; echo "bench $wl rc=$?"
done
for S in 32768 4096; do
  timeout 600 python bench.py --workload c1 --batch 1 --seq-len $S --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-headline > gpurun_out/wl_b1_$S.json 2> gpurun_out/wl_b1_$S.err; echo "bench b1 $S rc=$?"
done
for f in gpurun_out/wl_*.json; do python -c "
import json; d=json.load(open('$f')); r=d['roofline']
print('$f', 'step %.1f us' % (d['ms_per_step']*1e3), 'tok/s %.0f' % d['value'], 'K3 %.1f us hbm %.3f' % (r['avg_launch_us'], r['hbm_frac']), 'clk', d['clocks']['sm_mhz'])" || tail -2 ${f%.json}.err; done
