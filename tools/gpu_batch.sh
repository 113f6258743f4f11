timeout 900 python -m pytest tests/test_gpu_kfengine.py -q -p no:cacheprovider 2>&1 | tail -2
for v in 0 1 0 1; do KR_KF_SPLITF=$v timeout 600 python tools/kf_probe.py 2>&1 | head -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('splitF $v config2', d['kf_ax_us'], d['kf_atx_us'], d['kf_pair_us'], d['bitwise_vs_device_built'])"; done
for v in 0 1; do KR_KF_SPLITF=$v BOARDS=1 timeout 300 python tools/solver_probe.py kfactored 2000 2>&1 | tail -1 | sed "s/^/[splitF $v] /"; done
