#!/bin/bash
# scratch batch for one gpurun call (edited per call)
TAG=${TAG:-r02z} bash tools/round_end_run.sh
