#!/bin/bash
# scratch batch for one gpurun call (edited per call)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_factors_device.py tests/test_gpu_headline.py tests/test_gpu_engine.py -x -q -p no:cacheprovider > gpurun_out/dev_lr.log 2>&1; echo "rc=$?" >> gpurun_out/dev_lr.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/dev_lr_bench.json 2> gpurun_out/dev_lr_bench.err; echo "bench rc=$?" >> gpurun_out/dev_lr.log
