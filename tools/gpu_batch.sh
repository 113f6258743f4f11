#!/bin/bash
# scratch batch for one gpurun call (edited per call)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_tiny_product.py tests/test_gpu_solver.py -x -q -p no:cacheprovider > gpurun_out/deep_tests2.log 2>&1; echo "rc=$?" >> gpurun_out/deep_tests2.log
