# ad-hoc GPU batch (edited per call)
T=r02z
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_pytest_jit_all.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_jit_all.log
tail -5 gpurun_out/${T}_pytest_jit_all.log
