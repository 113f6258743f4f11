# ad-hoc GPU batch (edited per call)
T=r02z
for cfg in "0 2" "6000 2" "10000 2" "15000 2" "4000 3" "6000 3" "3000 4" "5000 4"; do set -- $cfg; KR_JIT_STAGGER=$1 KR_JIT_STAGGER_K=$2 timeout 300 python tools/solver_probe.py kron 400 2>&1 | sed "s/^/[stagger $1 k $2] /"; done
