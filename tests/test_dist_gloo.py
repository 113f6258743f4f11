"""The N>1 path on CPU: boards sharded over 2 ranks (gloo), the local solver
state held per rank, gap scalars gathered in board order at checkpoints.
The global trace must be bitwise identical to the single-process run (the
rank count cannot change the result), including the early-stop decision.
The local solver here is the oracle's incremental DCFR (the GPU ranks run
CudaSolver behind the same begin / iterate / checkpoint interface)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2112_03804_b200.dist import DistributedDcfr, exploitability_from_boards, shard

POT = 2 * 1875.0
NBOARDS = 5


def boards(indices):
    import pyoracle as po
    out = []
    for b in indices:
        inst = po.Instance.builtin("random_small", seed=100 + b)
        out.append((inst, inst.sparsify("b", True)))
    return out


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, kw, out):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "oracle")]
    import pyoracle as po
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        local = po.DcfrBoards(boards(shard(NBOARDS, rank, world)))
        r = DistributedDcfr(local, NBOARDS, POT, rank, world).run(**kw)
        out[rank] = (r["trace_expl"].tobytes(), r["board_br1"].tobytes(), r["iterations"])
    finally:
        dist.destroy_process_group()


def run_world(world, **kw):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), kw, out), nprocs=world, join=True)
    return dict(out)


def test_shard_is_contiguous_and_complete():
    for nb in (1, 5, 48):
        for world in (1, 2, 3, 4, 8):
            got = [b for r in range(world) for b in shard(nb, r, world)]
            assert got == list(range(nb))
    assert [len(shard(48, r, 8)) for r in range(8)] == [6] * 8


def test_single_board_matches_reference_formula():
    assert exploitability_from_boards([3.0], [5.0], 4.0) == (3.0 + 5.0) / 2 / 4.0


@pytest.mark.parametrize("kw", [dict(max_iters=40, checkpoint_every=10),
                                dict(max_iters=2000, checkpoint_every=5, target=0.02),
                                dict(max_iters=40, checkpoint_every=10, alpha=float("inf"), beta=float("-inf"),
                                     gamma=1.0, rule=1)])
def test_two_ranks_match_one(kw):
    import pyoracle as po
    single = DistributedDcfr(po.DcfrBoards(boards(range(NBOARDS))), NBOARDS, POT).run(**kw)
    got = run_world(2, **kw)
    assert len(got) == 2
    for rank in (0, 1):
        expl, br1, iters = got[rank]
        assert iters == single["iterations"]
        assert expl == single["trace_expl"].tobytes()
        assert br1 == single["board_br1"].tobytes()
    if kw.get("target"):
        assert single["iterations"] < kw["max_iters"]
