for v in "" kfw4 kfw16 ""; do KR_CUDA_LIB_VARIANT=$v timeout 600 python tools/kf_probe.py 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('[$v]', d['config'], d['kf_ax_us'], d['kf_atx_us'], d['kf_pair_us'], d['bitwise_vs_device_built'])"; done
