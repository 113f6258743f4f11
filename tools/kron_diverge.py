"""Iteration-by-iteration divergence of DCFR averages, implicit vs factored engine."""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2112_03804_b200 import host as H
from paper_2112_03804_b200.solver import DcfrParams, solver_for
nb = int(sys.argv[1]) if len(sys.argv) > 1 else 4
boards = H.turn_instances("Ks7d4c2h", nboards=nb, tree=3)
si, sf = solver_for(boards, implicit=True), solver_for(boards)
si.begin(DcfrParams()); sf.begin(DcfrParams())
for t in range(1, 101):
    si.iterate(1); sf.iterate(1)
    a1, a2 = si.averages(); b1, b2 = sf.averages()
    d = max(np.abs(a1 - b1).max(), np.abs(a2 - b2).max())
    if t <= 10 or t % 10 == 0 or d > 1e-6:
        print(t, f"{d:.3e}", flush=True)
    if d > 1e-3:
        i = np.argmax(np.abs(a1 - b1)); j = np.argmax(np.abs(a2 - b2))
        print("p1 idx", i, a1[i], b1[i], "p2 idx", j, a2[j], b2[j])
        break
