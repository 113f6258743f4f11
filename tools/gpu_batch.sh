for v in 0 1 0 1; do KR_KF_PIPE=$v timeout 600 python tools/kf_probe.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pipe $v', d['kf_ax_us'], d['kf_atx_us'], d['kf_pair_us'], d['bitwise_vs_device_built'])"; done
for v in 0 1; do KR_KF_PIPE=$v timeout 300 python tools/solver_probe.py kfactored 300 2>&1 | tail -1 | sed "s/^/[kf pipe $v] /"; done
