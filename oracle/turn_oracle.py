"""CPU checker for turn endgames (TEST INFRASTRUCTURE: only tests/ import it).

The turn betting round is beyond the reference: kronriver solves
single river endgames.  This module restates, for the game defined in
paper_2112_03804_b200/turn.py, the reference's own pieces composed through
the turn treeplex:
  - every payoff block is the block formula of referenceMatvec /
    referenceMatvecT (kron.hpp:211-254), Y = P X F^T + (P o W) X S^T with
    P_ij = lambda1_i lambda2_j [disjoint] and W_ij = sign(key1_i - key2_j),
    written as dense numpy products;
  - the solver is dcfrSolve (solver.hpp:343-404), with cfrSweep (222-260),
    regretMatch (166-194), sequenceForm (197-218), discount and averaging
    applied per hand.  River subtrees are swept first.  Each river subtree's
    root value (the sum of its root nodes' values, descending node order, as
    seqVal[0] accumulates them) is summed over the boards (ascending card) into
    the turn sequence sigma_p(t).  The turn sweep adds that sum after the turn
    children (ev = g + (children + river)).  Each river sequence form runs with
    mass 1 and is then scaled by the turn reach of sigma_p(t);
  - bestResponseValue (292-321) composes the same way.
Products: `products="block"` applies each block by the block formula
(dense numpy); `products="factored"` applies it by the reference's own
factored matvec / matvecTranspose (engine.hpp:58-133) over Technique B with
postprocessing built from the block's pieces (the oracle's techniqueB +
postprocess, or_sparsify_pieces).  The device's Kronecker-factored engine
reproduces the latter bit for bit, so a turn solve driven by it is checked
bitwise; the K7 engine differs by summation order and is held to tolerances
stated in the tests.
"""
import numpy as np


def _disjoint(c1, c2):
    m1 = (1 << c1[:, 0].astype(np.int64)) | (1 << c1[:, 1].astype(np.int64))
    m2 = (1 << c2[:, 0].astype(np.int64)) | (1 << c2[:, 1].astype(np.int64))
    return (m1[:, None] & m2[None, :]) == 0


class Block:
    def __init__(self, piece, products="block"):
        self.factored = products == "factored"
        if self.factored:
            import pyoracle as po
            self.sp = po.Sparsification.from_pieces(piece)
            return
        k1, k2 = [np.asarray(k, np.int64) for k in piece["key"]]
        self.P = piece["lam"][0][:, None] * piece["lam"][1][None, :] * _disjoint(*piece["cards"])
        self.PW = self.P * np.sign(k1[:, None] - k2[None, :])
        self.F, self.S = piece["F"], piece["S"]

    def ax(self, x):  # x: (m2, n2) -> (m1, n1)
        if self.factored:
            return self.sp.matvec(np.ascontiguousarray(x).ravel())
        return self.P @ x @ self.F.T + self.PW @ x @ self.S.T

    def atx(self, y):  # y: (m1, n1) -> (m2, n2)
        if self.factored:
            return self.sp.matvec_t(np.ascontiguousarray(y).ravel())
        return self.P.T @ y @ self.F + self.PW.T @ y @ self.S


class Tree:
    """Treeplex of one player (skeleton.hpp:114-126): nodes in preorder."""

    def __init__(self, tp):
        self.n = int(tp.n_seq)
        self.parent = [int(v) for v in tp.parent]
        ap = [int(v) for v in tp.action_ptr]
        self.acts = [[int(s) for s in tp.action_seq[ap[v]:ap[v + 1]]] for v in range(len(self.parent))]


def regret_match(R, seqs):  # solver.hpp:166-194
    r = [R[s - 1] for s in seqs]
    best = r[0]
    max_abs = abs(best)
    for v in r[1:]:
        best = max(best, v)
        max_abs = max(max_abs, abs(v))
    tol = 1e-9 * (1 + max_abs)
    if best > tol:
        sp = 0.0
        for v in r:
            if v > 0:
                sp += v
        return [v / sp if v > 0 else 0.0 for v in r]
    ties = sum(1 for v in r if v >= best - tol)
    return [1.0 / ties if v >= best - tol else 0.0 for v in r]


def sweep(tree, R, g, extra=None, inst=None):
    """cfrSweep of one hand (solver.hpp:227-245); returns the root value.
    inst: receives each sequence's instantaneous regret (ev - nodeVal)."""
    sv = [0.0] * (tree.n + 1)
    for v in range(len(tree.parent) - 1, -1, -1):
        seqs = tree.acts[v]
        probs = regret_match(R, seqs)
        node = 0.0
        evs = []
        for a, s in enumerate(seqs):
            cs = sv[s] + extra[s - 1] if extra is not None else sv[s]
            ev = g[s - 1] + cs
            sv[s] = ev
            evs.append(ev)
            node += probs[a] * ev
        for s in seqs:
            d = sv[s] - node
            R[s - 1] += d
            if inst is not None:
                inst[s - 1] = d
        sv[tree.parent[v]] += node
    return sv[0]


def factor(t, e):
    """t^e / (t^e + 1), with the limits 1 / 0 at e = +-inf (kr_dcfr_params)."""
    if np.isinf(e):
        return 1.0 if e > 0 else 0.0
    te = t ** e
    return te / (te + 1)


def seq_form(tree, R):
    """sequenceForm of one hand with root mass 1 (solver.hpp:202-215)."""
    reach = [0.0] * (tree.n + 1)
    reach[0] = 1.0
    for v in range(len(tree.parent)):
        probs = regret_match(R, tree.acts[v])
        mass = reach[tree.parent[v]]
        for a, s in enumerate(tree.acts[v]):
            reach[s] = mass * probs[a]
    return np.array(reach[1:])


def br_walk(tree, g, extra=None):
    """bestResponseValue walk of one hand (solver.hpp:304-318)."""
    sv = [0.0] * (tree.n + 1)
    for v in range(len(tree.parent) - 1, -1, -1):
        best, first = 0.0, True
        for s in tree.acts[v]:
            cs = sv[s] + extra[s - 1] if extra is not None else sv[s]
            ev = g[s - 1] + cs
            if first or ev > best:
                best = ev
            first = False
        sv[tree.parent[v]] += best
    return sv[0]


class TurnOracle:
    def __init__(self, game, products="block"):
        self.g = game
        self.turn = Block(game.kron_pieces(None)[0], products)
        self.river = [[Block(pc, products) for pc in game.kron_pieces(t)] for t in range(len(game.conts))]
        self.tt = [Tree(game.tree_turn[p]) for p in range(2)]
        self.tr = [[Tree(game.tree_river[t][p]) for p in range(2)] for t in range(len(game.conts))]
        self.boff = np.concatenate([[0], np.cumsum(game.mb)])

    # -- products -----------------------------------------------------------
    def ax(self, x2):
        g = self.g
        out = np.zeros(g.size[0])
        n1, n2 = g.n_turn
        out[:g.off[0][0]] = self.turn.ax(x2[:g.off[1][0]].reshape(g.m, n2)).ravel()
        for t, blocks in enumerate(self.river):
            r1, r2 = g.n_river[t]
            for b, blk in enumerate(blocks):
                lo1 = g.off[0][t] + self.boff[b] * r1
                lo2 = g.off[1][t] + self.boff[b] * r2
                mb = g.mb[b]
                out[lo1:lo1 + mb * r1] = blk.ax(x2[lo2:lo2 + mb * r2].reshape(mb, r2)).ravel()
        return out

    def atx(self, y1):
        g = self.g
        out = np.zeros(g.size[1])
        n1, n2 = g.n_turn
        out[:g.off[1][0]] = self.turn.atx(y1[:g.off[0][0]].reshape(g.m, n1)).ravel()
        for t, blocks in enumerate(self.river):
            r1, r2 = g.n_river[t]
            for b, blk in enumerate(blocks):
                lo1 = g.off[0][t] + self.boff[b] * r1
                lo2 = g.off[1][t] + self.boff[b] * r2
                mb = g.mb[b]
                out[lo2:lo2 + mb * r2] = blk.atx(y1[lo1:lo1 + mb * r1].reshape(mb, r1)).ravel()
        return out

    # -- one player's half-iteration ---------------------------------------------
    def _river_slices(self, p, t):
        g = self.g
        n = g.n_river[t][p]
        for b in range(len(g.rivers)):
            for r in range(g.mb[b]):
                lo = g.off[p][t] + (self.boff[b] + r) * n
                yield b, r, slice(lo, lo + n)

    def _hand(self, tree, R, X, grad, sl, extra, rule, pos, neg):
        """One hand's sweep and strategy under the update rule (the river
        oracle's playerUpdate): 0 DCFR; 1 CFR+ (discount, then match the
        discounted regrets); 2 PRM+ (match R + the last regret)."""
        d = np.zeros(sl.stop - sl.start) if rule == 2 else None
        Rs = R[sl]
        root = sweep(tree, Rs, grad[sl], extra, d)
        if rule != 0:
            Rs *= np.where(Rs > 0, pos, neg)
        R[sl] = Rs
        X[sl] = seq_form(tree, Rs + d if rule == 2 else Rs)
        return root

    def update(self, p, R, X, grad, mode1=True, rule=0, pos=1.0, neg=0.0):
        """Regrets R and strategy X (full vectors) of player p from gradient
        grad (already negated for player 2); mode1=False: initial strategy."""
        g = self.g
        nt = g.n_turn[p]
        extra = np.zeros(g.m * nt)
        for t in range(len(g.conts)):
            tree = self.tr[t][p]
            sigma = int(g.conts[t][p])
            root = np.zeros(sum(g.mb))
            for b, r, sl in self._river_slices(p, t):
                if mode1:
                    root[self.boff[b] + r] = self._hand(tree, R, X, grad, sl, None, rule, pos, neg)
                else:
                    X[sl] = seq_form(tree, R[sl])
            # sum over boards (ascending) per turn hand
            acc = np.zeros(g.m)
            for b in range(len(g.rivers)):
                for r, h in enumerate(g.order[b]):
                    acc[h] += root[self.boff[b] + r]
            extra[np.arange(g.m) * nt + sigma - 1] += acc
        for h in range(g.m):
            sl = slice(h * nt, (h + 1) * nt)
            if mode1:
                self._hand(self.tt[p], R, X, grad, sl, extra[sl], rule, pos, neg)
            else:
                X[sl] = seq_form(self.tt[p], R[sl])
        # river strategies: turn reach of sigma_p(t) times the mass-1 form
        for t in range(len(g.conts)):
            sigma = int(g.conts[t][p])
            for b, r, sl in self._river_slices(p, t):
                h = g.order[b][r]
                X[sl] = X[h * nt + sigma - 1] * X[sl]

    def best_response(self, p, opp):
        g = self.g
        grad = self.ax(opp) if p == 0 else -self.atx(opp)
        nt = g.n_turn[p]
        extra = np.zeros(g.m * nt)
        for t in range(len(g.conts)):
            tree = self.tr[t][p]
            sigma = int(g.conts[t][p])
            acc = np.zeros(g.m)
            for b, r, sl in self._river_slices(p, t):
                acc[g.order[b][r]] += br_walk(tree, grad[sl])
            extra[np.arange(g.m) * nt + sigma - 1] += acc
        total = 0.0
        for h in range(g.m):
            sl = slice(h * nt, (h + 1) * nt)
            total += br_walk(self.tt[p], grad[sl], extra[sl])
        return total

    def dcfr(self, iters, alpha=1.5, beta=0.0, gamma=2.0, checkpoint_every=1, rule=0):
        """dcfrSolve over the turn game; returns (trace of (br1, br2, expl), avgs)."""
        g = self.g
        R = [np.zeros(g.size[0]), np.zeros(g.size[1])]
        A = [np.zeros(g.size[0]), np.zeros(g.size[1])]
        X = [np.zeros(g.size[0]), np.zeros(g.size[1])]
        self.update(0, R[0], X[0], None, mode1=False)
        self.update(1, R[1], X[1], None, mode1=False)
        ws = 0.0
        trace = []
        pot = 2 * g.pot
        for t in range(1, iters + 1):
            pos, neg = factor(t, alpha), factor(t, beta)
            shrink = (t / (t + 1)) ** gamma
            self.update(0, R[0], X[0], self.ax(X[1]), rule=rule, pos=pos, neg=neg)
            self.update(1, R[1], X[1], -self.atx(X[0]), rule=rule, pos=pos, neg=neg)
            for p in range(2):
                if rule == 0:
                    R[p] *= np.where(R[p] > 0, pos, neg)
                A[p] = (A[p] + X[p]) * shrink
            ws = (ws + 1) * shrink
            if t % checkpoint_every == 0 or t == iters:
                a1, a2 = A[0] / ws, A[1] / ws
                b1, b2 = self.best_response(0, a2), self.best_response(1, a1)
                trace.append((t, b1, b2, (b1 + b2) / 2 / pot))
        return trace, (A[0] / ws, A[1] / ws)
