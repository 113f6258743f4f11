timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02z_pytest_all5.log 2>&1; echo "rc=$?" >> gpurun_out/r02z_pytest_all5.log
tail -3 gpurun_out/r02z_pytest_all5.log
