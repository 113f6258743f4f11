timeout 600 python -m pytest tests/test_gpu_jit_step.py -q -p no:cacheprovider -k "spilling or turn12_jit" 2>&1 | tail -2
timeout 300 python tools/solver_probe.py kron 400 2>&1 | tail -1
