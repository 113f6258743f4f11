# ad-hoc GPU batch (edited per call): tests, then the sanitizer sweep
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r02a_gpu.txt
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02a_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r02a_pytest_gpu.log
TAG=r02a bash tools/sanitize_run.sh
