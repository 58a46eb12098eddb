#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python tools/sweep.py --tp 2 > gpurun_out/sweep_tp2.log 2>&1; echo "tp2 rc=$?"; tail -24 gpurun_out/sweep_tp2.log
timeout 1200 python tools/sweep.py --tp 4 --batches 1,32,128 --contexts 8192,32768 > gpurun_out/sweep_tp4.log 2>&1; echo "tp4 rc=$?"; tail -10 gpurun_out/sweep_tp4.log
