# ad-hoc GPU batch (edited per call)
T=r02z
for t in 32 64 128 32; do KR_KF_TILE=$t timeout 600 python tools/kf_probe.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tile $t', d['kf_ax_us'], d['kf_atx_us'], d['kf_pair_us'], d['bitwise_vs_device_built'])"; done
KR_KF_TILE=64 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_kf_seqmajor -c 4 --csv python tools/kf_probe.py 2>/dev/null | grep gpu__time | awk -F'","' '{print $NF}' | head -4
