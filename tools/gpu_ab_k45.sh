TESTS="e2e or full_size or mtp or decode_v" VARIANTS="base k45b k45c" WORKLOADS="c1 h8 c2mtp" KERNELS="K45_combine_W_UV" STEPS=30 bash tools/gpu_ab_k.sh
for v in base k45b k45c; do for w in c1 h8; do
TPLA_LIB=build/variants/libtpla_$v.so timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:combine_wuv -c 6 --csv python bench.py --workload $w --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-headline 2>/dev/null | grep combine_wuv | awk -F'","' -v v=$v -v w=$w '{print v, w, $(NF-2), $NF}' | tr -d '"' | tail -4
done; done
