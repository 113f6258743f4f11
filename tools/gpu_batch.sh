#!/bin/bash
# scratch batch for one gpurun call (edited per call)
mkdir -p gpurun_out
KR_CUDA_LIB_VARIANT=checked timeout 600 python -m pytest tests/test_gpu_tiny_product.py -x -q -p no:cacheprovider > gpurun_out/tiny_checked.log 2>&1; echo "rc=$?" >> gpurun_out/tiny_checked.log
timeout 1200 python tools/tiny_probe.py > gpurun_out/tiny_probe.log 2>&1; echo "probe exit $?" >> gpurun_out/tiny_probe.log
for t in "0 8" "1000000 8" "1000000 16"; do set -- $t
  KR_TINY=$1 KR_TINY_CLUSTER=$2 timeout 300 python tools/graph_product_probe.py 2>&1 | grep -E "RESULT|Error|error" >> gpurun_out/graph_probe.log
done
TAG=r02z8 bash tools/round_end_run.sh
