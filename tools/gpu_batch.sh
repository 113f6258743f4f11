# ad-hoc GPU batch (edited per call)
T=r02z
timeout 600 python tools/pair_mode_probe.py 2>&1 | tail -4
KR_PAIR_SERIAL_GB=100 timeout 600 python tools/pair_mode_probe.py 2>&1 | tail -2 | sed 's/^/[forced concurrent] /'
