#!/bin/bash
# scratch batch for one gpurun call (edited per call)
TAG=r02z12 bash tools/round_end_run.sh
