#!/bin/bash
mkdir -p gpurun_out
for v in sp nosp; do
  TPLA_LIB=build/variants/libtpla_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "full_size" > gpurun_out/fs_$v.log 2>&1; echo "$v full_size rc=$?"; grep -E "^E  |passed|failed" gpurun_out/fs_$v.log | head -4
done
