#!/bin/bash
# scratch batch for one gpurun call (edited per call)
mkdir -p gpurun_out
{
for rep in 1 2; do
for v in "" ku6 ku10 ku12; do echo "variant=${v:-ku8} rep=$rep"; KR_CUDA_LIB_VARIANT=$v timeout 300 python tools/pair_probe.py; done
done
} > gpurun_out/ku_c3.log 2>&1
