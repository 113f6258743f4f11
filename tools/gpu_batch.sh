# ad-hoc GPU batch (edited per call)
T=r02z
timeout 900 python -m pytest tests/test_gpu_jit_step.py -q -x -p no:cacheprovider > gpurun_out/${T}_ov_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_ov_pytest.log
tail -3 gpurun_out/${T}_ov_pytest.log
for ov in 0 1; do
  KR_OVERLAP=$ov timeout 300 python tools/solver_probe.py kron 400 2>&1 | sed "s/^/[overlap $ov] /"
  KR_OVERLAP=$ov timeout 300 python tools/solver_probe.py kfactored 200 2>&1 | sed "s/^/[overlap $ov] /"
done
