# ad-hoc GPU batch (edited per call)
T=r02z
timeout 900 python -m pytest tests/test_gpu_jit_step.py -q -x -p no:cacheprovider -k forced 2>&1 | tail -3
