for v in 0 1; do KR_TURN_JIT_SMALL=$v timeout 300 python tools/turn_probe.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tiny $v turn', d['iters_per_s'], d['exploitability'])"; done
timeout 900 python -m pytest tests/test_gpu_turn.py -q -p no:cacheprovider 2>&1 | tail -2
