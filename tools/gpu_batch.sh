# ad-hoc GPU batch (edited per call)
T=r02z
timeout 900 python -m pytest tests/test_gpu_jit_step.py tests/test_gpu_turn.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 300 python tools/turn_probe.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('turn', d['iters_per_s'])"
timeout 300 python tools/solver_probe.py kron 400
