for cta in 5 77; do
TPLA_K3_MODE=trace TPLA_K3_TRACE_CTA=$cta timeout 300 python bench.py --workload h8 --steps 1 --warmup 3 --no-graph --no-e2e --no-cpu-baseline > /dev/null 2> gpurun_out/trace_pp_h8_$cta.log; echo "trace rc=$?"
grep "k3 cta\]" gpurun_out/trace_pp_h8_$cta.log | grep -E "traced| $cta start|span|  0 start"; grep "k3 start" gpurun_out/trace_pp_h8_$cta.log
done
