#!/bin/bash
# scratch batch for one gpurun call (edited per call)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_turn.py -x -q -p no:cacheprovider -s > gpurun_out/turn_tight.log 2>&1; echo "rc=$?" >> gpurun_out/turn_tight.log
TAG=r02z9 bash tools/round_end_run.sh
