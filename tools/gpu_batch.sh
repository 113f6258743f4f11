#!/bin/bash
# scratch batch for one gpurun call (edited per call)
mkdir -p gpurun_out
{
for rep in 1 2; do
for v in "" kfd3 kfd4; do
  echo "variant=${v:-default} rep=$rep"
  KR_CUDA_LIB_VARIANT=$v timeout 300 python tools/kf_probe.py 2 3
done
done
} > gpurun_out/kf_depth.log 2>&1
