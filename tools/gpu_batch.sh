# ad-hoc GPU batch (edited per call)
T=r02z
timeout 900 python -m pytest tests/test_gpu_jit_step.py -q -x -p no:cacheprovider > gpurun_out/${T}_jit3_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_jit3_pytest.log
tail -2 gpurun_out/${T}_jit3_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for i in 1 2; do timeout 300 python tools/solver_probe.py kron 400 2>&1; done
