# ad-hoc GPU batch (edited per call)
T=r02l
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=15 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_gpu.log
tail -n 25 gpurun_out/${T}_pytest_gpu.log
