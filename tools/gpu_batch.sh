#!/bin/bash
# scratch batch for one gpurun call (edited per call)
mkdir -p gpurun_out
KR_CUDA_LIB_VARIANT=checked timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/checked_full.log 2>&1; echo "rc=$?" >> gpurun_out/checked_full.log
