# ad-hoc GPU batch (edited per call)
T=r02z
KR_CUDA_LIB_VARIANT=checked timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_checked_pytest2.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_checked_pytest2.log
tail -4 gpurun_out/${T}_checked_pytest2.log
