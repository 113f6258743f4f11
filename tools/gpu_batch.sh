#!/bin/bash
# scratch batch for one gpurun call (edited per call)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_headline.py tests/test_gpu_solver.py -x -q -p no:cacheprovider > gpurun_out/lean_tests.log 2>&1; echo "rc=$?" >> gpurun_out/lean_tests.log
{
for rep in 1 2; do
for v in "" lean1 lean8; do echo "variant=${v:-default4} rep=$rep"; KR_CUDA_LIB_VARIANT=$v timeout 300 python tools/pair_probe.py; done
echo "variant=nolean rep=$rep"; KR_NO_LEAN=1 timeout 300 python tools/pair_probe.py
done
} > gpurun_out/lean_probe.log 2>&1
