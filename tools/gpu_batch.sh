#!/bin/bash
# scratch batch for one gpurun call (edited per call)
mkdir -p gpurun_out
KR_ASYNC=1 timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_solver.py tests/test_gpu_factors_device.py -x -q -p no:cacheprovider > gpurun_out/async_tests.log 2>&1; echo "rc=$?" >> gpurun_out/async_tests.log
KR_ASYNC=1 KR_CUDA_LIB_VARIANT=checked timeout 900 python -m pytest tests/test_gpu_engine.py -x -q -p no:cacheprovider >> gpurun_out/async_tests.log 2>&1; echo "rc=$?" >> gpurun_out/async_tests.log
{
PROBE_LABEL=regs KR_ASYNC=0 timeout 120 python tools/config1_iteration_probe.py
PROBE_LABEL=async KR_ASYNC=1 timeout 120 python tools/config1_iteration_probe.py
timeout 600 python tools/tiny_probe.py '[["regs", {"KR_ASYNC": "0"}], ["async", {"KR_ASYNC": "1"}]]'
} > gpurun_out/async_probe.log 2>&1
