"""Device DCFR solver (reference solver.hpp:145-414) through the kr_solver C ABI.

CudaSolver binds a CudaEngine to the two players' treeplexes and runs
dcfrSolve / bestResponseValue / exploitability on the B200.  Per-hand walks
replay the reference's arithmetic order, so with the engine's ordered
products the whole trace is bitwise equal to the reference's.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as N


@dataclass
class Treeplex:
    """One player's decision nodes in preorder (skeleton.hpp:89-126)."""
    n_seq: int
    parent: np.ndarray      # [nodes] parent sequence id (0 = empty sequence)
    action_ptr: np.ndarray  # [nodes+1]
    action_seq: np.ndarray  # [actions] 1-based sequence ids

    @classmethod
    def from_flat(cls, n_seq, flat):
        """[parent, nActions, seq...] per node (oracle/product export format)."""
        parent, ptr, seqs = [], [0], []
        q = 0
        flat = list(int(v) for v in flat)
        while q < len(flat):
            parent.append(flat[q])
            cnt = flat[q + 1]
            seqs.extend(flat[q + 2:q + 2 + cnt])
            ptr.append(ptr[-1] + cnt)
            q += 2 + cnt
        return cls(n_seq, np.array(parent, np.int32), np.array(ptr, np.int32), np.array(seqs, np.int32))

    def struct(self, keep):
        arrs = [np.ascontiguousarray(a, np.int32) for a in (self.parent, self.action_ptr, self.action_seq)]
        keep += arrs
        return N.kr_treeplex(self.n_seq, len(self.parent), *(N.ptr(a) for a in arrs))


def jit_step_source(tree: Treeplex, rule=0):
    """The CUDA C of the player step compiled for `tree` (kr_jit_step_source)."""
    keep = []
    t = tree.struct(keep)
    L = N.cuda()
    n = L.kr_jit_step_source(C.byref(t), int(rule), None, 0)
    if n < 0:
        raise N.InvalidInputError(1, "treeplex is not level-ordered")
    buf = C.create_string_buffer(int(n) + 1)
    L.kr_jit_step_source(C.byref(t), int(rule), buf, int(n) + 1)
    return buf.value.decode()


RULE_DCFR, RULE_CFRP, RULE_PRMP = 0, 1, 2


@dataclass
class DcfrParams:
    """DcfrParams (solver.hpp:101-109) plus the update rule (kr_engine.h
    KR_RULE_*): 0 is the reference's DCFR; CFR+ and PRM+ are presets beyond
    the reference (its SPEC.md:438 lists CFR+ as a non-goal)."""
    alpha: float = 1.5
    beta: float = 0.0
    gamma: float = 2.0
    max_iters: int = 1000
    target_exploitability: float = 0.0
    checkpoint_every: int = 50
    rule: int = RULE_DCFR

    @classmethod
    def cfr_plus(cls, **kw):
        """CFR+: regret matching+ (R <- max(R + r, 0)), linear averaging."""
        return cls(alpha=math.inf, beta=-math.inf, gamma=1.0, rule=RULE_CFRP, **kw)

    @classmethod
    def prm_plus(cls, **kw):
        """Predictive regret matching+ (strategy from R + last regret), linear averaging."""
        return cls(alpha=math.inf, beta=-math.inf, gamma=1.0, rule=RULE_PRMP, **kw)


@dataclass
class DcfrResult:
    """DcfrResult (solver.hpp:133-140) plus per-board best-response values."""
    iterations: int
    exploitability: float
    gradient_flops: int
    trace_iter: np.ndarray
    trace_expl: np.ndarray
    trace_br1: np.ndarray
    trace_br2: np.ndarray
    board_br1: np.ndarray
    board_br2: np.ndarray
    avg1: np.ndarray
    avg2: np.ndarray
    seconds: float
    launches: int = 0
    extra: dict = field(default_factory=dict)


class CudaSolver:
    def __init__(self, engine, tree1: Treeplex, tree2: Treeplex, hands1, hands2, pot):
        L = N.cuda()
        keep = []
        t1, t2 = tree1.struct(keep), tree2.struct(keep)
        h1 = np.ascontiguousarray(np.atleast_1d(hands1), np.int32)
        h2 = np.ascontiguousarray(np.atleast_1d(hands2), np.int32)
        if len(h1) != len(h2):
            raise N.InvalidInputError(1, "hand-count lists differ in length")
        h = C.c_void_p()
        N.check(L.kr_solver_create(engine.handle, C.byref(t1), C.byref(t2), len(h1), N.ptr(h1), N.ptr(h2),
                                   C.c_double(pot), C.byref(h)))
        self._h = h
        self.engine = engine  # keep alive: the solver borrows the engine (solver.hpp:32 ownership rule)
        self.nboards = len(h1)
        self.nb_out = self.nboards   # boards reported per checkpoint (all ranks' with a comm)
        self.comm = None
        self.pot = float(pot)
        self.rows, self.cols = engine.rows, engine.cols

    def step_kind(self, player):
        """(kind, why): 2 = the step compiled for this player's treeplex
        (NVRTC), 1 = the generic team kernel, 0 = the generic per-hand kernel;
        `why` says why the compiled step is not used."""
        why = C.c_char_p()
        k = N.cuda().kr_solver_step_kind(self._h, int(player), C.byref(why))
        return int(k), (why.value or b"").decode()

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            N.cuda().kr_solver_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def launches(self):
        return int(N.cuda().kr_solver_launches(self._h))

    def set_comm(self, comm, boards_per_rank):
        """kr_solver_set_comm: this solver's boards are `comm.rank`'s shard of
        boards_per_rank; runs and checkpoints then report every board in
        global order, checkpoint values all-gathered over NCCL in-stream."""
        bpr = np.ascontiguousarray(boards_per_rank, np.int32)
        N.check(N.cuda().kr_solver_set_comm(self._h, comm.handle if comm else None, N.ptr(bpr) if comm else None))
        self.comm = comm
        self.nb_out = int(bpr.sum()) if comm else self.nboards

    def run(self, params: DcfrParams = None, want_avg=True) -> DcfrResult:
        p = params or DcfrParams()
        cap = max(p.max_iters, 0) // max(p.checkpoint_every, 1) + 2  # the C ABI validates the params
        ti = np.zeros(cap, np.int32)
        te, b1, b2 = np.zeros(cap), np.zeros(cap), np.zeros(cap)
        nb = self.nb_out
        bb1, bb2 = np.zeros(cap * nb), np.zeros(cap * nb)
        a1 = np.zeros(self.rows) if want_avg else None
        a2 = np.zeros(self.cols) if want_avg else None
        prm = N.kr_dcfr_params(p.alpha, p.beta, p.gamma, p.max_iters, p.target_exploitability, p.checkpoint_every,
                               p.rule)
        res = N.kr_dcfr_result(0, 0.0, 0, 0, cap, N.ptr(ti), N.ptr(te), N.ptr(b1), N.ptr(b2), N.ptr(bb1),
                               N.ptr(bb2), N.ptr(a1), N.ptr(a2), 0.0)
        launches0 = self.launches() + self.engine.launches()
        N.check(N.cuda().kr_solver_run(self._h, C.byref(prm), C.byref(res)))
        n = min(res.trace_len, cap)
        return DcfrResult(res.iterations, res.exploitability, res.gradient_flops, ti[:n], te[:n], b1[:n], b2[:n],
                          bb1[:n * nb].reshape(n, nb), bb2[:n * nb].reshape(n, nb), a1, a2, res.seconds,
                          self.launches() + self.engine.launches() - launches0)

    # -- incremental interface (multi-rank drivers, dist.py) ----------------
    def begin(self, params: DcfrParams = None):
        p = params or DcfrParams()
        N.check(N.cuda().kr_solver_set_rule(self._h, p.rule))
        N.check(N.cuda().kr_solver_begin(self._h, p.alpha, p.beta, p.gamma))

    def iterate(self, n):
        N.check(N.cuda().kr_solver_iterate(self._h, int(n)))

    def checkpoint(self):
        """Per-board best-response values (br1, br2) of the current averages."""
        b1, b2 = np.zeros(self.nb_out), np.zeros(self.nb_out)
        N.check(N.cuda().kr_solver_checkpoint(self._h, N.ptr(b1), N.ptr(b2)))
        return b1, b2

    def averages(self):
        a1, a2 = np.zeros(self.rows), np.zeros(self.cols)
        N.check(N.cuda().kr_solver_averages(self._h, N.ptr(a1), N.ptr(a2)))
        return a1, a2

    @property
    def iteration(self):
        return int(N.cuda().kr_solver_iteration(self._h))

    def best_response(self, player, opp, per_board=False):
        """bestResponseValue (solver.hpp:292-321) against a host strategy."""
        opp = np.ascontiguousarray(opp, np.float64)
        v = C.c_double()
        bv = np.zeros(self.nboards)
        N.check(N.cuda().kr_solver_best_response(self._h, player, N.ptr(opp), len(opp), C.byref(v), N.ptr(bv)))
        return (v.value, bv) if per_board else v.value

    def best_responses(self, x1, x2):
        """The two best-response values (br1 against x2, br2 against x1),
        summed over boards; their sum is the saddle-point gap."""
        return self.best_response(0, x2), self.best_response(1, x1)

    def exploitability(self, x1, x2):
        """exploitability (solver.hpp:325-331): (br1 + br2) / 2 / pot, with the
        chance root's 1/nboards over a multi-board engine (kr_solver_run's rule)."""
        br1, br2 = self.best_responses(x1, x2)
        return (br1 + br2) / 2 / self.pot / self.nboards


def solver_for(boards, device=0, implicit=False):
    """Engine + solver over one or more (Instance, Factors) boards that share a
    betting tree (product host objects, paper_2112_03804_b200.host).  With
    implicit=True the gradient runs on the implicit Kronecker engine
    (CudaEngine.kron) and the factors are not needed (entries may be bare
    Instances)."""
    from .engine import CudaEngine
    insts = [b[0] if isinstance(b, (tuple, list)) else b for b in boards]
    eng = CudaEngine.kron(insts, device=device) if implicit else CudaEngine([b[1] for b in boards], device=device)
    i0 = insts[0]
    return CudaSolver(eng, i0.treeplex(0), i0.treeplex(1), [i.m1 for i in insts], [i.m2 for i in insts], i0.pot)


def dcfr_solve(instance, factors, params: DcfrParams = None, device=0) -> DcfrResult:
    """dcfrSolve(kp, FactoredEngine(s), params) (solver.hpp:343-414) on the B200."""
    return solver_for([(instance, factors)], device).run(params)
