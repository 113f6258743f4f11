"""Multi-GPU: the chance (board) dimension sharded over ranks.

The turn payoff is block diagonal over river cards, so a
board's Ax / ATx reads and writes only that board's slices: the products
need no communication at all.  Each rank holds a contiguous range of boards
(engine + solver state for those boards only).  The one collective is at
checkpoints: the per-board best-response values are all-gathered and summed
in board order on every rank, so the exploitability trace — and hence the
early-stop decision — is bitwise identical for any number of ranks (an
all-reduce would reorder the sum with the world size).

One process per GPU (torchrun); the process group is NCCL on GPUs, gloo in
the CPU tests (tests/test_dist_gloo.py).
"""
from __future__ import annotations

import numpy as np


def shard(nboards, rank, world):
    """Contiguous board range of `rank`: boards split as evenly as possible,
    earlier ranks take the remainder (48 boards -> 48/24/12/6 at 1/2/4/8)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(nboards, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def gather_boards(local, nboards, world, group=None, device=None):
    """All-gather per-board float64 values held by each rank (contiguous
    shards, rank order == board order) into the full board vector."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return np.asarray(local, np.float64)
    width = max(len(shard(nboards, r, world)) for r in range(world))
    buf = torch.zeros(width, dtype=torch.float64, device=device)
    buf[:len(local)] = torch.as_tensor(np.asarray(local, np.float64), device=device)
    parts = [torch.zeros(width, dtype=torch.float64, device=device) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    out = [p[:len(shard(nboards, r, world))].cpu().numpy() for r, p in enumerate(parts)]
    return np.concatenate(out)


def exploitability_from_boards(br1, br2, pot):
    """exploitability (solver.hpp:325-331) of the turn game: a board's value
    (br1_b + br2_b) / 2 / pot averaged over boards in board order (the chance
    root picks a board uniformly); one board reproduces the reference."""
    if len(br1) == 1:
        return (br1[0] + br2[0]) / 2 / pot
    total = 0.0
    for a, b in zip(br1, br2):
        total += (a + b) / 2 / pot
    return total / len(br1)


class DistributedDcfr:
    """dcfrSolve (solver.hpp:343-404) over boards sharded across ranks.

    `local` is a begin / iterate / checkpoint object over this rank's boards
    (CudaSolver on a GPU; the oracle's DcfrBoards in CPU tests)."""

    def __init__(self, local, nboards, pot, rank=0, world=1, group=None, device=None):
        self.local, self.nboards, self.pot = local, nboards, pot
        self.rank, self.world, self.group, self.device = rank, world, group, device

    def run(self, alpha=1.5, beta=0.0, gamma=2.0, max_iters=1000, target=0.0, checkpoint_every=50, rule=0):
        if max_iters < 1 or checkpoint_every < 1:
            raise ValueError("iteration budget and checkpoint period must be positive")
        from .solver import CudaSolver, DcfrParams
        if isinstance(self.local, CudaSolver):
            self.local.begin(DcfrParams(alpha=alpha, beta=beta, gamma=gamma, rule=rule))
        else:  # the oracle's DcfrBoards (CPU tests)
            self.local.begin(alpha, beta, gamma, rule)
        t = 0
        trace = {"iter": [], "expl": [], "br1": [], "br2": []}
        while t < max_iters:
            nxt = min(max_iters, (t // checkpoint_every + 1) * checkpoint_every)
            self.local.iterate(nxt - t)
            t = nxt
            b1, b2 = self.local.checkpoint()
            g1 = gather_boards(b1, self.nboards, self.world, self.group, self.device)
            g2 = gather_boards(b2, self.nboards, self.world, self.group, self.device)
            expl = exploitability_from_boards(g1, g2, self.pot)
            trace["iter"].append(t)
            trace["expl"].append(expl)
            trace["br1"].append(g1)
            trace["br2"].append(g2)
            if target > 0 and expl <= target:
                break
        return {"iterations": t, "exploitability": trace["expl"][-1], "trace_iter": np.array(trace["iter"]),
                "trace_expl": np.array(trace["expl"]), "board_br1": np.array(trace["br1"]),
                "board_br2": np.array(trace["br2"])}
