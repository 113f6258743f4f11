for w in 0 1 0 1; do KR_K7_WIDE=$w timeout 300 python tools/solver_probe.py kron 400 2>&1 | tail -1 | sed "s/^/[wide $w] /"; done
