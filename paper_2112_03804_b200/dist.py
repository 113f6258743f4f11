"""Multi-GPU: the chance (board) dimension sharded over ranks.

The turn payoff is block diagonal over river cards, so a
board's Ax / ATx reads and writes only that board's slices: the products
need no communication at all.  Each rank holds a contiguous range of boards
(engine + solver state for those boards only).  The one collective is at
checkpoints: the per-board best-response values are all-gathered and summed
in board order on every rank, so the exploitability trace — and hence the
early-stop decision — is bitwise identical for any number of ranks (an
all-reduce would reorder the sum with the world size).

One process per GPU (torchrun).  On GPUs the transport is the library's own
NCCL communicator (kr_comm, `Comm` below): the per-board values are
all-gathered in-stream by libkrcuda and folded there, inside the solver's
captured iteration graphs.  A host process group (gloo: the CPU tests, and a
multi-rank smoke on a one-GPU box) drives the same all-gather from Python.
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


def boards_per_rank(nboards, world):
    return np.ascontiguousarray([len(shard(nboards, r, world)) for r in range(world)], np.int32)


class Comm:
    """kr_comm: an NCCL communicator owned by libkrcuda, one rank per GPU
    (kr_comm_init_rank from a unique id shared over a torch process group,
    or kr_comm_init_all over a device list in one process)."""

    ID_BYTES = 128

    def __init__(self, handle, device):
        from . import _native as N
        self._h = handle
        self.device = device
        self.rank = int(N.cuda().kr_comm_rank(handle))
        self.size = int(N.cuda().kr_comm_size(handle))

    @classmethod
    def from_process_group(cls, device, group=None):
        """Every rank of `group` calls this; rank 0's unique id travels over
        the group (one broadcast), then NCCL takes over."""
        import ctypes as C

        import torch.distributed as dist

        from . import _native as N
        L = N.cuda()
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = (C.c_uint8 * cls.ID_BYTES)()
        if rank == 0:
            N.check(L.kr_comm_unique_id(uid))
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0, group=group)
        uid = (C.c_uint8 * cls.ID_BYTES).from_buffer_copy(obj[0])
        h = C.c_void_p()
        N.check(L.kr_comm_init_rank(uid, world, rank, device, C.byref(h)))
        return cls(h, device)

    @classmethod
    def single(cls, device=0):
        """A one-rank communicator (the NCCL path on one GPU)."""
        import ctypes as C

        from . import _native as N
        L = N.cuda()
        uid = (C.c_uint8 * cls.ID_BYTES)()
        N.check(L.kr_comm_unique_id(uid))
        h = C.c_void_p()
        N.check(L.kr_comm_init_rank(uid, 1, 0, device, C.byref(h)))
        return cls(h, device)

    @classmethod
    def init_all(cls, devices):
        """One communicator per device, all in this process."""
        import ctypes as C

        from . import _native as N
        devs = np.ascontiguousarray(devices, np.int32)
        hs = (C.c_void_p * len(devs))()
        N.check(N.cuda().kr_comm_init_all(len(devs), N.ptr(devs), hs))
        return [cls(C.c_void_p(hs[i]), int(devs[i])) for i in range(len(devs))]

    @property
    def handle(self):
        return self._h

    def close(self):
        from . import _native as N
        if getattr(self, "_h", None) is not None and self._h.value:
            N.cuda().kr_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


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
        if isinstance(self.local, CudaSolver) and self.local.comm is not None:
            # the library's NCCL path: kr_solver_run with the checkpoint
            # all-gathers in-stream, iterations replayed as graphs
            r = self.local.run(DcfrParams(alpha=alpha, beta=beta, gamma=gamma, max_iters=max_iters,
                                          target_exploitability=target, checkpoint_every=checkpoint_every,
                                          rule=rule), want_avg=False)
            return {"iterations": r.iterations, "exploitability": r.exploitability, "trace_iter": r.trace_iter,
                    "trace_expl": r.trace_expl, "board_br1": r.board_br1, "board_br2": r.board_br2}
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
