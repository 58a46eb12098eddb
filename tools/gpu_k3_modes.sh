for w in c1 c3; do for m in normal nold notma stream; do
  TPLA_K3_MODE=$m timeout 300 python bench.py --workload $w --steps 50 --no-e2e --no-cpu-baseline > gpurun_out/m_$w_$m.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/m_$w_$m.json')); r=d['roofline']
print('$w $m K3 in-step %.1f us iso %.1f  clocks %s' % (r['avg_launch_us'], r['isolated_avg_launch_us'], d['clocks']['sm_mhz']))"
done; done
