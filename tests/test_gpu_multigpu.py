"""Board sharding through the library's transports.

The turn payoff is block diagonal over river boards, so each rank holds a
contiguous shard of boards and nothing crosses ranks in the products.  What
does cross (per-board best-response values at checkpoints, the turn solver's
per-board river values every half-iteration) is all-gathered and folded in
global board order by libkrcuda — the one-GPU fold — so every result must be
BITWISE the one-rank result, for any rank count:

* the NCCL path at world 1 (kr_comm over one GPU: the collectives are real
  ncclAllGather calls, enqueued on the solver stream and captured into the
  iteration graphs) against the solver without a communicator;
* two ranks on one GPU through a host (gloo) process group (each rank's
  kernels are independent; only the host exchange synchronises them);
* `multigpu`: two ranks on two GPUs over NCCL (skipped below two GPUs)."""
import os

import numpy as np
import pytest

from conftest import bits_equal
from paper_2112_03804_b200 import CudaEngine
from paper_2112_03804_b200 import host as H
from paper_2112_03804_b200.dist import Comm, DistributedDcfr, boards_per_rank, shard
from paper_2112_03804_b200.solver import CudaSolver, DcfrParams
from paper_2112_03804_b200.turn import TurnGame, TurnSolver

pytestmark = pytest.mark.gpu

NB = 6


def solver_on(boards, engine="factored"):
    insts = [i for i, _ in boards]
    eng = CudaEngine([f for _, f in boards]) if engine == "factored" else (
        CudaEngine.kfactored(insts) if engine == "kfactored" else CudaEngine.kron(insts))
    i0 = insts[0]
    return CudaSolver(eng, i0.treeplex(0), i0.treeplex(1), [i.m1 for i in insts], [i.m2 for i in insts], i0.pot)


@pytest.mark.parametrize("engine", ["factored", "kfactored", "implicit"])
@pytest.mark.parametrize("no_graph", [False, True], ids=["graph", "launches"])
def test_dcfr_nccl_world1_bitwise(engine, no_graph, monkeypatch):
    if no_graph:
        monkeypatch.setenv("KR_NO_GRAPH", "1")
    boards = H.turn_instances(nboards=NB, factors=engine == "factored")
    prm = DcfrParams(max_iters=60, checkpoint_every=20)
    ref = solver_on(boards, engine).run(prm)
    s = solver_on(boards, engine)
    comm = Comm.single(0)
    s.set_comm(comm, [NB])
    r = s.run(prm)
    assert bits_equal(r.trace_expl, ref.trace_expl)
    assert bits_equal(r.board_br1, ref.board_br1) and bits_equal(r.board_br2, ref.board_br2)
    assert bits_equal(r.avg1, ref.avg1) and bits_equal(r.avg2, ref.avg2)
    # early stop (host checkpoints through kr_solver_checkpoint)
    t = 10 * ref.trace_expl[1]
    s2 = solver_on(boards, engine)
    s2.set_comm(comm, [NB])
    r2 = s2.run(DcfrParams(max_iters=60, checkpoint_every=20, target_exploitability=t))
    r3 = solver_on(boards, engine).run(DcfrParams(max_iters=60, checkpoint_every=20, target_exploitability=t))
    assert r2.iterations == r3.iterations and bits_equal(r2.trace_expl, r3.trace_expl)


@pytest.fixture(scope="module")
def game():
    return TurnGame()


def test_turn_nccl_world1_bitwise(game):
    ref = TurnSolver(game).run(max_iters=40, checkpoint_every=10, want_avg=True)
    s = TurnSolver(game, comm=Comm.single(0), boards_per_rank=[len(game.rivers)])
    r = s.run(max_iters=40, checkpoint_every=10, want_avg=True)
    for k in ("trace_expl", "trace_br1", "trace_br2", "avg1", "avg2"):
        assert bits_equal(r[k], ref[k]), k


def _turn_rank(rank, world, port, nb, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = TurnGame(boards=list(shard(nb, rank, world)))
        r = TurnSolver(g, group=dist.group.WORLD).run(max_iters=30, checkpoint_every=3)
        q.put((rank, r["trace_br1"].tobytes(), r["trace_br2"].tobytes()))
    finally:
        dist.destroy_process_group()


def test_turn_two_gloo_ranks_bitwise():
    """22 river boards over two ranks on one GPU (host collectives): the trace
    is bitwise the one-rank trace (board-order fold of all-gathered values)."""
    import torch.multiprocessing as mp
    g = TurnGame()
    nb = len(g.rivers)
    ref = TurnSolver(g).run(max_iters=30, checkpoint_every=3)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_turn_rank, args=(r, 2, 29641, nb, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = [q.get(timeout=900) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for _, b1, b2 in out:
        assert b1 == ref["trace_br1"].tobytes() and b2 == ref["trace_br2"].tobytes()


def _dcfr_rank(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = list(shard(NB, rank, world))
        boards = H.turn_instances(nboards=NB, indices=mine)
        drv = DistributedDcfr(solver_on(boards), NB, boards[0][0].pot, rank, world, device=torch.device("cpu"))
        r = drv.run(max_iters=40, checkpoint_every=10)
        q.put((rank, r["trace_expl"].tobytes()))
    finally:
        dist.destroy_process_group()


def test_dcfr_two_gloo_ranks_bitwise():
    import torch.multiprocessing as mp
    ref = solver_on(H.turn_instances(nboards=NB)).run(DcfrParams(max_iters=40, checkpoint_every=10))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_dcfr_rank, args=(r, 2, 29643, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = [q.get(timeout=900) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for _, te in out:
        assert te == ref.trace_expl.tobytes()


# ---------------------------------------------------------------- 2 GPUs ----
def _nccl_rank(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)  # only to share the NCCL id
    try:
        comm = Comm.from_process_group(rank)
        bpr = boards_per_rank(NB, world)
        boards = H.turn_instances(nboards=NB, indices=list(shard(NB, rank, world)))
        insts = [i for i, _ in boards]
        eng = CudaEngine([f for _, f in boards], device=rank)
        i0 = insts[0]
        s = CudaSolver(eng, i0.treeplex(0), i0.treeplex(1), [i.m1 for i in insts], [i.m2 for i in insts], i0.pot)
        s.set_comm(comm, bpr)
        r = s.run(DcfrParams(max_iters=40, checkpoint_every=10))
        g = TurnGame(boards=list(shard(22, rank, world)))
        tr = TurnSolver(g, device=rank, comm=comm, boards_per_rank=boards_per_rank(22, world)).run(
            max_iters=20, checkpoint_every=5)
        q.put((rank, r.trace_expl.tobytes(), tr["trace_expl"].tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.multigpu
def test_two_gpus_nccl_bitwise():
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    ref = solver_on(H.turn_instances(nboards=NB)).run(DcfrParams(max_iters=40, checkpoint_every=10))
    tref = TurnSolver(TurnGame()).run(max_iters=20, checkpoint_every=5)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_nccl_rank, args=(r, 2, 29645, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = [q.get(timeout=900) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for _, te, tt in out:
        assert te == ref.trace_expl.tobytes() and tt == tref["trace_expl"].tobytes()
