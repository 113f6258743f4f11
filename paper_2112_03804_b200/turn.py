"""Turn endgames: a betting round on the turn above the river boards
(beyond the reference, whose instances are single
river endgames).

Game.  Turn board (4 cards); every hand not touching it for both players
(C(48,2) = 1,128 with the 52-card deck); beliefs mu_p; lambda_p = mu_p /
sqrt(beta), beta = sum over disjoint hand pairs of mu1 mu2 (the river's
normalisation, kron.hpp:160-163, over turn hands).  The turn betting tree is
built by the river skeleton builder (skeleton.hpp) from the turn
configuration: its fold leaves pay as on the river, and its "showdown" leaves
are the river continuations t, each reached by one sequence pair (sigma1(t),
sigma2(t)) with both players' contribution c_t (the S entry).  Continuation t
deals the river card b uniformly among the cards not on the board and not in
either hand (1/44 with the 52-card deck) and plays the river subgame built
from (stack - (c_t - pot), c_t) with the river menus; after an all-in call
(no stack left) that subgame is a check-check showdown at stakes c_t.

Payoff.  With pi_ij = lambda1_i lambda2_j [i, j disjoint]:
  turn block   A[(i, s1), (j, s2)] = pi_ij F_turn[s1, s2]
  river block  A[(t, b, i, r1), (t, b, j, r2)] = pi_ij / K (F_t + W^b_ij S_t)[r1, r2]
               for i, j not holding b (K = cards left for the river),
so A is block diagonal: one implicit Kronecker board for the turn (S empty)
and, per continuation, one K7 engine over the river boards with lambda / sqrt(K)
in each board's strength order.  The turn and the rivers are coupled only
through the treeplex: river root nodes hang under sigma_p(t).

Vector layout per player p: [turn block: m x n_turn] then, per continuation t,
per board b (ascending card id): [m_b x n_t] in board b's hand order.
"""
from __future__ import annotations

import itertools

import numpy as np

from . import host as H

RANKS, SUITS = "23456789TJQKA", "cdhs"


def card_id(code):
    return RANKS.index(code[0]) * 4 + SUITS.index(code[1])


def deck_cards(deck):
    if deck == 26:
        return [r * 4 + s for r in range(13) for s in range(2)]
    return list(range(52))


class TurnGame:
    """Host-side description of a turn endgame (see the module docstring)."""

    def __init__(self, turn="Kc9d7c4d", deck=26, seed=1, stack=18125.0, pot=1875.0, turn_menu=(0.5,),
                 turn_raise_cap=1, river_menu=(0.5, 1.0), river_raise_cap=1, boards=None, turn_all_in=False):
        """boards: indices of the river cards this object holds (a rank's
        contiguous shard, dist.shard); default all."""
        self.deck = deck
        self.turn = [card_id(turn[i:i + 2]) for i in range(0, 8, 2)]
        cards = [c for c in deck_cards(deck) if c not in self.turn]
        self.all_rivers = cards
        self.rivers = cards if boards is None else [cards[i] for i in boards]  # board cards b, ascending id
        self.K = len(cards) - 4                              # river cards left given two hands
        self.hands = np.array([(max(a, b), min(a, b)) for a, b in itertools.combinations(cards, 2)], np.uint8)
        self.m = len(self.hands)
        rng = np.random.default_rng(seed)
        self.mu = [rng.uniform(0.25, 1.0, self.m), rng.uniform(0.25, 1.0, self.m)]
        masks = np.array([(1 << int(h[0])) | (1 << int(h[1])) for h in self.hands], dtype=object)
        disjoint = np.array([[(int(a) & int(b)) == 0 for b in masks] for a in masks])
        self.disjoint = disjoint
        self.beta = float(self.mu[0] @ disjoint @ self.mu[1])
        self.lam = [self.mu[0] / np.sqrt(self.beta), self.mu[1] / np.sqrt(self.beta)]
        self.stack, self.pot = float(stack), float(pot)
        self.river_menu, self.river_raise_cap = list(river_menu), int(river_raise_cap)
        # turn tree: the builder on a placeholder river card (only F, S and the
        # treeplex are used; no showdown happens on the turn)
        dummy = self.rivers[0]
        free = [h for h in self.hands if dummy not in h]
        h1 = free[0]
        h2 = next(h for h in free if not set(h.tolist()) & set(h1.tolist()))
        self.turn_inst = H.custom_instance(self.turn + [dummy], deck, np.array([h1], np.uint8), [1.0],
                                           np.array([h2], np.uint8), [1.0], stack, pot, list(turn_menu),
                                           turn_all_in, turn_raise_cap)
        v = self.turn_inst.kron_view()
        self.n_turn = (v.n1, v.n2)
        self.F_turn = _csr(v.F, v.n2)
        S = _csr(v.S, v.n2)
        self.conts = [(r + 1, c + 1, S[r, c]) for r, c in zip(*np.nonzero(S))]  # (sigma1, sigma2, c_t)
        self.tree_turn = [self.turn_inst.treeplex(0), self.turn_inst.treeplex(1)]
        # river continuations: one instance per (t, b); per-board hand order
        self.river = []       # [t] -> list over boards of Instance
        self.order = []       # [b] -> turn-hand index of each river hand (board order)
        for ti, (_, _, c) in enumerate(self.conts):
            insts = []
            for bi, b in enumerate(self.rivers):
                keep = np.array([b not in h for h in self.hands])
                idx = np.flatnonzero(keep)
                left = stack - (c - pot)
                if left > 0:
                    cfg = (left, c, self.river_menu, True, river_raise_cap)
                else:  # all-in on the turn: no river betting, a showdown at stakes c (check-check)
                    cfg = (1.0, c, [], False, 0)
                inst = H.custom_instance(self.turn + [b], deck, self.hands[idx], self.mu[0][idx], self.hands[idx],
                                         self.mu[1][idx], *cfg)
                if ti == 0:
                    code = {tuple(sorted(h)): i for i, h in enumerate(self.hands.tolist())}
                    self.order.append(np.array([code[tuple(sorted((card_id(s[:2]), card_id(s[2:]))))]
                                                for s in inst.hands(0)]))
                insts.append(inst)
            self.river.append(insts)
        self.n_river = [(r[0].n1, r[0].n2) for r in self.river]
        self.tree_river = [[r[0].treeplex(0), r[0].treeplex(1)] for r in self.river]
        self.mb = [len(o) for o in self.order]
        # vector offsets per player
        self.off = []
        for p in range(2):
            o = [self.m * self.n_turn[p]]
            for ti in range(len(self.conts)):
                o.append(o[-1] + sum(self.mb) * self.n_river[ti][p])
            self.off.append(o)
        self.size = [self.off[0][-1], self.off[1][-1]]

    # -- the payoff blocks as K7 boards ----------------------------------------
    def turn_board(self):
        """kr_kron_board of the turn block: keys all equal (no showdown), S empty."""
        from . import _native as N
        v = self.turn_inst.kron_view()
        keep = []
        b = N.kr_kron_board()
        b.m1 = b.m2 = self.m
        b.n1, b.n2 = self.n_turn
        z = np.zeros(self.m, np.uint32)
        cards = np.ascontiguousarray(self.hands, np.uint8)
        l1, l2 = np.ascontiguousarray(self.lam[0]), np.ascontiguousarray(self.lam[1])
        keep += [z, cards, l1, l2]
        b.key1 = b.key2 = z.ctypes.data
        b.cards1 = b.cards2 = cards.ctypes.data
        b.lambda1, b.lambda2 = l1.ctypes.data, l2.ctypes.data
        b.F = v.F
        so = np.zeros(b.n1 + 1, np.int64)
        keep.append(so)
        b.S = N.kr_compressed(b.n1, so.ctypes.data, None, None)
        return b, keep

    def river_boards(self, t):
        """kr_kron_board per river board of continuation t, lambda / sqrt(K) in
        each board's hand order."""
        out, keep = [], []
        s = 1.0 / np.sqrt(self.K)
        for bi, inst in enumerate(self.river[t]):
            v = inst.kron_view()
            idx = self.order[bi]
            l1 = np.ascontiguousarray(self.lam[0][idx] * s)
            l2 = np.ascontiguousarray(self.lam[1][idx] * s)
            keep += [l1, l2, inst]
            v.lambda1, v.lambda2 = l1.ctypes.data, l2.ctypes.data
            out.append(v)
        return out, keep

    def kron_pieces(self, t=None):
        """(keys, cards, lambdas, F, S) per block as numpy, for the CPU checker."""
        if t is None:
            z = np.zeros(self.m, np.uint32)
            return [dict(key=[z, z], cards=[self.hands, self.hands], lam=self.lam, F=self.F_turn,
                         S=np.zeros_like(self.F_turn))]
        s = 1.0 / np.sqrt(self.K)
        out = []
        for bi, inst in enumerate(self.river[t]):
            v = inst.kron_view()
            idx = self.order[bi]
            k1 = np.ctypeslib.as_array(_cast(v.key1, "u4"), (v.m1,)).copy()
            k2 = np.ctypeslib.as_array(_cast(v.key2, "u4"), (v.m2,)).copy()
            c = self.hands[idx]
            out.append(dict(key=[k1, k2], cards=[c, c], lam=[self.lam[0][idx] * s, self.lam[1][idx] * s],
                            F=_csr(v.F, v.n2), S=_csr(v.S, v.n2)))
        return out


def _cast(p, kind):
    import ctypes as C
    return C.cast(p, C.POINTER({"u4": C.c_uint32}[kind]))


def _csr(c, ncols):
    import ctypes as C
    no = c.outer_size
    outer = np.ctypeslib.as_array(C.cast(c.outer, C.POINTER(C.c_int64)), (no + 1,)).copy()
    nnz = int(outer[-1])
    dense = np.zeros((no, ncols))
    if nnz:
        inner = np.ctypeslib.as_array(C.cast(c.inner, C.POINTER(C.c_int32)), (nnz,))
        val = np.ctypeslib.as_array(C.cast(c.val, C.POINTER(C.c_double)), (nnz,))
        for r in range(no):
            for e in range(outer[r], outer[r + 1]):
                dense[r, inner[e]] += val[e]
    return dense


class TurnSolver:
    """DCFR over a TurnGame on the device (kr_turn_solver): implicit Kronecker
    engines for the turn block and each continuation's river boards, the
    turn treeplex composed with the river treeplexes."""

    def __init__(self, game: TurnGame, device=0, group=None, comm=None, boards_per_rank=None, engine="implicit"):
        """Board sharding (each rank builds its TurnGame with boards=shard):
        comm, a dist.Comm (NCCL in-stream, graph-captured), or group, a host
        torch.distributed process group (gloo), carries the per-board river
        values of every half-iteration; the library folds them in global board
        order, so the solve is bitwise the one-rank solve (see shard()).
        engine: "implicit" (K7, the fastest; products within 1e-12) or
        "kfactored" (each block as Technique B post from its Kronecker
        factors: products bitwise the reference's factored matvec, so the
        whole solve is bitwise its CPU restatement)."""
        import ctypes as C

        from . import _native as N
        from .engine import CudaEngine
        self.game = game
        tb, keep = game.turn_board()
        self.turn_eng = CudaEngine.from_kron_boards([tb], device, kind=engine)
        self.river_eng = []
        for t in range(len(game.conts)):
            rb, k2 = game.river_boards(t)
            self.river_eng.append(CudaEngine.from_kron_boards(rb, device, kind=engine))
        del keep
        keepalive = []
        tt = (N.kr_treeplex * 2)(*[game.tree_turn[p].struct(keepalive) for p in range(2)])
        rt = (N.kr_treeplex * (2 * len(game.conts)))(
            *[game.tree_river[t][p].struct(keepalive) for t in range(len(game.conts)) for p in range(2)])
        engs = (C.c_void_p * len(self.river_eng))(*[e.handle.value for e in self.river_eng])
        mb = np.ascontiguousarray(game.mb, np.int32)
        r2t = np.ascontiguousarray(np.concatenate(game.order), np.int32)
        sig = np.ascontiguousarray([int(game.conts[t][p]) for t in range(len(game.conts)) for p in range(2)],
                                   np.int32)
        h = C.c_void_p()
        N.check(N.cuda().kr_turn_solver_create(self.turn_eng.handle, len(game.conts), engs, tt, rt, game.m,
                                               len(game.rivers), N.ptr(mb), N.ptr(r2t), N.ptr(sig), 2 * game.pot,
                                               C.byref(h)))
        self._h = h
        self.comm = None
        if group is not None or comm is not None:
            self.shard(group=group, comm=comm, boards_per_rank=boards_per_rank)

    def shard(self, group=None, comm=None, boards_per_rank=None):
        """Attach the board-sharding transport.  boards_per_rank defaults to
        this rank's board count gathered over the group."""
        import ctypes as C

        import torch

        from . import _native as N
        L = N.cuda()
        nb = len(self.game.rivers)
        if comm is not None:
            if boards_per_rank is None:
                raise ValueError("an NCCL communicator needs boards_per_rank")
            bpr = np.ascontiguousarray(boards_per_rank, np.int32)
            N.check(L.kr_turn_solver_set_comm(self._h, comm.handle, N.ptr(bpr)))
            self.comm = comm
            return
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        if boards_per_rank is None:
            counts = [None] * world
            dist.all_gather_object(counts, nb, group=group)
            boards_per_rank = counts
        bpr = np.ascontiguousarray(boards_per_rank, np.int32)
        sz = np.zeros(4, np.int64)
        N.check(L.kr_turn_solver_sizes(self._h, N.ptr(sz)))
        count = int(sz[2]) * int(bpr.max())
        dev = torch.device("cuda", torch.cuda.current_device())
        self.send = torch.zeros(count, dtype=torch.float64, device=dev)
        self.recv = torch.zeros(world * count, dtype=torch.float64, device=dev)
        host = dist.get_backend(group) != "nccl"

        def exchange(_user):
            if host:  # gloo: through host memory
                src = self.send.cpu()
                parts = [torch.empty_like(src) for _ in range(world)]
                dist.all_gather(parts, src, group=group)
                self.recv.copy_(torch.cat(parts))
            else:
                dist.all_gather_into_tensor(self.recv, self.send, group=group)
            torch.cuda.synchronize(dev)

        self._cb = C.CFUNCTYPE(None, C.c_void_p)(exchange)
        N.check(L.kr_turn_solver_set_exchange(self._h, C.cast(self._cb, C.c_void_p), None, world, rank, N.ptr(bpr),
                                              C.c_void_p(self.send.data_ptr()), C.c_void_p(self.recv.data_ptr())))

    def close(self):
        from . import _native as N
        if getattr(self, "_h", None) and self._h.value:
            N.cuda().kr_turn_solver_destroy(self._h)
            self._h = None
        self.send = self.recv = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run(self, max_iters=100, checkpoint_every=10, alpha=1.5, beta=0.0, gamma=2.0, want_avg=False, rule=0):
        import ctypes as C

        from . import _native as N
        cap = max_iters // checkpoint_every + 2
        ti = np.zeros(cap, np.int32)
        te, b1, b2 = np.zeros(cap), np.zeros(cap), np.zeros(cap)
        a1 = np.zeros(self.game.size[0]) if want_avg else None
        a2 = np.zeros(self.game.size[1]) if want_avg else None
        prm = N.kr_dcfr_params(alpha, beta, gamma, max_iters, 0.0, checkpoint_every, rule)
        res = N.kr_dcfr_result(0, 0.0, 0, 0, cap, N.ptr(ti), N.ptr(te), N.ptr(b1), N.ptr(b2), None, None,
                               N.ptr(a1), N.ptr(a2), 0.0)
        N.check(N.cuda().kr_turn_solver_run(self._h, C.byref(prm), C.byref(res)))
        n = min(res.trace_len, cap)
        return {"iterations": res.iterations, "exploitability": res.exploitability, "trace_iter": ti[:n],
                "trace_expl": te[:n], "trace_br1": b1[:n], "trace_br2": b2[:n], "seconds": res.seconds,
                "avg1": a1, "avg2": a2}
