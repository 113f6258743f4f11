timeout 900 python -m pytest tests/test_gpu_kfengine.py -q -p no:cacheprovider 2>&1 | tail -1
for cfg in "KR_KF_ROUNDS_A=4 KR_KF_ROUNDS_T=4" "X=1" "KR_KF_ROUNDS_A=4 KR_KF_ROUNDS_T=4" "X=1"; do env $cfg timeout 600 python tools/kf_probe.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg config3', d['kf_ax_us'], d['kf_atx_us'], d['kf_pair_us'])"; done
for cfg in "KR_KF_ROUNDS_A=4 KR_KF_ROUNDS_T=4" "X=1"; do env $cfg timeout 300 python tools/solver_probe.py kfactored 300 2>&1 | tail -1 | sed "s/^/[$cfg] /"; done
