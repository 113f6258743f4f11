#!/bin/bash
# scratch batch for one gpurun call (edited per call)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tiny_product.py tests/test_gpu_engine.py -x -q -p no:cacheprovider > gpurun_out/tiny3.log 2>&1; echo "rc=$?" >> gpurun_out/tiny3.log
KR_CUDA_LIB_VARIANT=checked timeout 600 python -m pytest tests/test_gpu_tiny_product.py -x -q -p no:cacheprovider >> gpurun_out/tiny3.log 2>&1; echo "rc=$?" >> gpurun_out/tiny3.log
