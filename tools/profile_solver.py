"""Profile target (development tool): DCFR on the first N boards of the
config-3 turn (default 48), a few iterations with one checkpoint, so ncu can
capture the solver-step kernels next to the engine's."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2112_03804_b200 import host as H  # noqa: E402
from paper_2112_03804_b200.solver import DcfrParams, solver_for  # noqa: E402


def main():
    nb = int(sys.argv[sys.argv.index("--turn") + 1]) if "--turn" in sys.argv else 48
    iters = int(sys.argv[sys.argv.index("--iters") + 1]) if "--iters" in sys.argv else 6
    s = solver_for(H.turn_instances(nboards=nb))
    r = s.run(DcfrParams(max_iters=iters, checkpoint_every=iters))
    torch.cuda.synchronize()
    print("ok", r.iterations, r.exploitability, r.seconds, r.launches)


if __name__ == "__main__":
    main()
