# ad-hoc GPU batch (edited per call)
T=r02z
for g in 2 4; do KR_JIT_GROUPS_ALL=1 KR_JIT_GROUPS=$g timeout 300 python tools/solver_probe.py kron 400 2>&1 | sed "s/^/[config3 groups $g] /"; done
KR_K7SEQ=0 timeout 300 python tools/solver_probe.py kron 400 2>&1 | sed "s/^/[config3 one-thread hand-major] /"
for g in 2 4; do KR_JIT_GROUPS_ALL=1 KR_JIT_GROUPS=$g timeout 300 python tools/solver_probe.py kfactored 200 2>&1 | sed "s/^/[config3 kf groups $g] /"; done
timeout 300 python tools/solver_probe.py kfactored 200 2>&1 | sed "s/^/[config3 kf one-thread] /"
