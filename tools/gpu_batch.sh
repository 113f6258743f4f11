# ad-hoc GPU batch (edited per call)
T=r02z
timeout 600 python -m pytest tests/test_gpu_checked.py -q -p no:cacheprovider > gpurun_out/${T}_checked_selftest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_checked_selftest.log
tail -5 gpurun_out/${T}_checked_selftest.log
