#!/bin/bash
# scratch batch for one gpurun call (edited per call)
mkdir -p gpurun_out
{
for rep in 1 2; do
echo "default rep=$rep"; timeout 300 python tools/pair_probe.py
echo "deep-all rep=$rep"; KR_DEEP_BLOCKS=1000000000 timeout 300 python tools/pair_probe.py
echo "nodeep rep=$rep"; KR_DEEP_KU=0 timeout 300 python tools/pair_probe.py
done
} > gpurun_out/deep_c3.log 2>&1
