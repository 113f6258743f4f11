timeout 900 python -m pytest tests/test_gpu_turn.py -q -p no:cacheprovider 2>&1 | tail -1
for i in 1 2; do timeout 300 python tools/turn_probe.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('turn', d['iters_per_s'], d['trace'])"; done
