# ad-hoc GPU batch (edited per call)
T=r02z
timeout 600 python -m pytest tests/test_gpu_jit_step.py -q -x -p no:cacheprovider -k "why" 2>&1 | tail -1
for g in 4 6 8 12; do KR_JIT_GROUPS=$g BOARDS=1 timeout 300 python tools/solver_probe.py kron 2000 2>&1 | sed "s/^/[config2 groups $g] /"; done
for g in 4 8; do KR_JIT_GROUPS=$g timeout 300 python -c "
import sys, time; sys.path.insert(0,'.')
from paper_2112_03804_b200 import host as H
from paper_2112_03804_b200.solver import DcfrParams, solver_for
p = H.builtin('twenty_card'); f = p.sparsify('b', True)
s = solver_for([(p, f)]); s.run(DcfrParams.cfr_plus(max_iters=20, checkpoint_every=1))
r = s.run(DcfrParams.cfr_plus(max_iters=1000, checkpoint_every=1)); print('[config1 groups $g]', 1000 / r.seconds, 'it/s', s.step_kind(0))
"; done
KR_JIT_GROUPS=0 timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_2112_03804_b200 import host as H
from paper_2112_03804_b200.solver import DcfrParams, solver_for
p = H.builtin('twenty_card'); f = p.sparsify('b', True)
s = solver_for([(p, f)]); s.run(DcfrParams.cfr_plus(max_iters=20, checkpoint_every=1))
r = s.run(DcfrParams.cfr_plus(max_iters=1000, checkpoint_every=1)); print('[config1 team]', 1000 / r.seconds, 'it/s')
"
