timeout 900 python -m pytest tests/test_gpu_jit_step.py tests/test_gpu_headline.py tests/test_gpu_solver.py -q -p no:cacheprovider 2>&1 | tail -3
for i in 1 2; do timeout 300 python tools/solver_probe.py kron 400 2>&1 | sed "s/^/[k7] /"; done
timeout 300 python tools/solver_probe.py kfactored 300 2>&1 | sed "s/^/[kf] /"
