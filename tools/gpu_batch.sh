# ad-hoc GPU batch (edited per call)
T=r02z
timeout 900 python -m pytest tests/test_gpu_jit_step.py -q -x -p no:cacheprovider > gpurun_out/${T}_kfseq_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_kfseq_pytest.log
tail -12 gpurun_out/${T}_kfseq_pytest.log
for v in 0 1; do KR_KFSEQ=$v timeout 300 python tools/solver_probe.py kfactored 300 2>&1 | sed "s/^/[kfseq $v] /"; done
timeout 300 python tools/solver_probe.py kron 400 2>&1 | sed "s/^/[k7] /"
