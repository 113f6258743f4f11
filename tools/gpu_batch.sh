#!/bin/bash
# scratch batch for one gpurun call (edited per call)
mkdir -p gpurun_out
timeout 300 python tools/small_engine_ncu.py > gpurun_out/se_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_spmv|k_tiny|k_chain" --launch-count 14 -o gpurun_out/small_engines -f python tools/small_engine_ncu.py > gpurun_out/se_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/se_ncu.log
