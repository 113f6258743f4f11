"""ctypes wrapper over the CPU ORACLE (oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg, always as the checker.  The product package
(paper_2112_03804_b200) never imports this module.

The oracle is a C++20 restatement of the reference `kronriver` library
(/root/reference/proj/include/kronriver/*.hpp); see oracle/kr_oracle.hpp
for the file:line each function follows.  It is pinned by the reference's
published golden numbers (README.md:75-82), tests/test_oracle_golden.py.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

CONTEXTS = ["first_action", "facing_check", "facing_bet", "after_one_raise", "after_multiple_raises"]

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C")


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{code}: {msg}")
        self.code = code


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.or_last_error.restype = C.c_char_p
        L.or_last_code.restype = C.c_char_p
        L.or_inst_beta.restype = C.c_double
        L.or_dense_nnz.restype = C.c_int64
        L.or_time_pairs.restype = C.c_double
        L.or_time_pairs_multi.restype = C.c_double
        _LIB = L
    return _LIB


def _check(rc):
    if rc != 0:
        L = lib()
        raise OracleError(L.or_last_code().decode(), L.or_last_error().decode())


class Instance:
    """Oracle RiverInstance + KronPayoff (kron.hpp:18-166)."""

    def __init__(self, handle):
        self.h = C.c_void_p(handle)
        d = np.zeros(14, np.int64)
        lib().or_inst_dims(self.h, d.ctypes.data_as(C.c_void_p))
        (self.m1, self.m2, self.n1, self.n2, self.rows, self.cols, self.nodes, self.dec0, self.dec1,
         self.terminals, self.folds, self.showdowns, self.nnzF, self.nnzS) = [int(v) for v in d]

    def __del__(self):
        if _LIB is not None and getattr(self, "h", None):
            _LIB.or_instance_free(self.h)
            self.h = None

    @classmethod
    def builtin(cls, name, seed=1, hands=0, shared=0, board="", deck=52, tree=1):
        out = C.c_void_p()
        _check(lib().or_builtin(name.encode(), C.c_uint64(seed), hands, shared, board.encode(), deck, tree,
                                C.byref(out)))
        return cls(out.value)

    @classmethod
    def from_json(cls, path_or_obj):
        """Mirror of instanceFromJson (instance_io.hpp:103-229) for the fields used."""
        j = path_or_obj
        if isinstance(path_or_obj, (str, os.PathLike)):
            with open(path_or_obj) as f:
                j = json.load(f)
        deck = None if j["deck"] == "standard52" else "".join(j["deck"]).encode()
        board = "".join(j["board"]).encode()
        hands, weights = [], []
        for p in range(2):
            items = sorted(j["beliefs"][p].items())
            hands.append("".join(k for k, _ in items).encode())
            weights.append(np.array([float(v) for _, v in items], np.float64))
        counts, values = [], []
        for p in range(2):
            menu = j["betting"]["menus"][p]
            for c in CONTEXTS:
                vals = menu.get(c, [])
                counts.append(len(vals))
                values.extend(float(v) for v in vals)
        counts = np.array(counts, np.int32)
        values = np.array(values if values else [0.0], np.float64)
        rc = j["betting"]["raise_cap"]
        out = C.c_void_p()
        _check(lib().or_instance(board, deck, len(weights[0]), hands[0], weights[0].ctypes.data_as(C.c_void_p),
                                 len(weights[1]), hands[1], weights[1].ctypes.data_as(C.c_void_p),
                                 C.c_double(j["stacks"][0]), C.c_double(j["stacks"][1]),
                                 C.c_double(j["pot_contribution"]), counts.ctypes.data_as(C.c_void_p),
                                 values.ctypes.data_as(C.c_void_p), int(bool(j["betting"]["all_in"])),
                                 -1 if rc is None else int(rc), C.byref(out)))
        return cls(out.value)

    @property
    def beta(self):
        return lib().or_inst_beta(self.h)

    def hands(self, player):
        n = self.m1 if player == 0 else self.m2
        buf = C.create_string_buffer(4 * n)
        lib().or_inst_hands(self.h, player, buf)
        raw = buf.raw.decode()
        return [raw[4 * i:4 * i + 4] for i in range(n)]

    def vectors(self):
        mu1, mu2 = np.zeros(self.m1), np.zeros(self.m2)
        l1, l2 = np.zeros(self.m1), np.zeros(self.m2)
        lib().or_inst_vectors(self.h, *(a.ctypes.data_as(C.c_void_p) for a in (mu1, mu2, l1, l2)))
        return mu1, mu2, l1, l2

    def W(self):
        W = np.zeros((self.m1, self.m2))
        H = np.zeros((self.m1, self.m2))
        lib().or_inst_W(self.h, W.ctypes.data_as(C.c_void_p), H.ctypes.data_as(C.c_void_p))
        return W, H

    def terminals_table(self):
        n = self.terminals
        ints = np.zeros((n, 4), np.int32)
        qs = np.zeros((n, 2))
        paths = C.create_string_buffer(64 * n)
        lib().or_inst_terminals(self.h, ints.ctypes.data_as(C.c_void_p), qs.ctypes.data_as(C.c_void_p), paths, 64)
        raw = paths.raw
        names = [raw[64 * t:64 * t + 64].split(b"\0", 1)[0].decode() for t in range(n)]
        return ints, qs, names

    def treeplex(self, player):
        n = lib().or_inst_treeplex(self.h, player, None)
        out = np.zeros(n, np.int32)
        lib().or_inst_treeplex(self.h, player, out.ctypes.data_as(C.c_void_p))
        return out

    def FS(self, which):
        n1, n2 = self.n1, self.n2
        nnz = self.nnzF if which == 0 else self.nnzS
        o = np.zeros(n1 + 1, np.int64)
        i = np.zeros(max(nnz, 1), np.int32)
        v = np.zeros(max(nnz, 1))
        lib().or_inst_FS(self.h, which, o.ctypes.data_as(C.c_void_p), i.ctypes.data_as(C.c_void_p),
                         v.ctypes.data_as(C.c_void_p))
        return o, i[:nnz], v[:nnz]

    def dense_nnz(self):
        return int(lib().or_dense_nnz(self.h))

    def dense(self, guard=5e7):
        A = np.zeros((self.rows, self.cols))
        _check(lib().or_dense_expand(self.h, C.c_double(guard), A.ctypes.data_as(C.c_void_p)))
        return A

    def reference_matvec(self, x):
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(self.rows)
        _check(lib().or_reference_matvec(self.h, x.ctypes.data_as(C.c_void_p), C.c_int64(len(x)),
                                         y.ctypes.data_as(C.c_void_p)))
        return y

    def reference_matvec_t(self, y):
        y = np.ascontiguousarray(y, np.float64)
        x = np.zeros(self.cols)
        _check(lib().or_reference_matvec_t(self.h, y.ctypes.data_as(C.c_void_p), C.c_int64(len(y)),
                                           x.ctypes.data_as(C.c_void_p)))
        return x

    def uniform(self, player):
        out = np.zeros(self.rows if player == 0 else self.cols)
        _check(lib().or_uniform(self.h, player, out.ctypes.data_as(C.c_void_p)))
        return out

    def sparsify(self, technique="b", post=True, peel_iters=1000):
        out = C.c_void_p()
        _check(lib().or_sparsify(self.h, 0 if technique.lower() == "a" else 1, int(post), peel_iters, C.byref(out)))
        return Sparsification(out.value)


class Sparsification:
    """Oracle Sparsification (sparsify.hpp:110-121): Ahat CSR, U CSR, M CSC, V CSC."""

    NAMES = ("ahat", "u", "m", "v")

    def __init__(self, handle):
        self.h = C.c_void_p(handle)
        d = np.zeros(9, np.int64)
        lib().or_sp_sizes(self.h, d.ctypes.data_as(C.c_void_p))
        self.rows, self.cols, self.k, nA, nU, nM, nV, tech, post = [int(v) for v in d]
        self.nnz = {"ahat": nA, "u": nU, "m": nM, "v": nV}
        self.technique = "a" if tech == 0 else "b"
        self.postprocessed = bool(post)

    def __del__(self):
        if _LIB is not None and getattr(self, "h", None):
            _LIB.or_sp_free(self.h)
            self.h = None

    def size_total(self):
        return sum(self.nnz.values())

    def flops_per_matvec(self):
        ident = self.nnz["m"] == self.k  # isIdentity holds for every factor the builders emit with nnz(M)==k
        return self.nnz["v"] + self.nnz["u"] + self.nnz["ahat"] + (0 if ident else self.nnz["m"] - self.k)

    def export(self, name):
        which = self.NAMES.index(name)
        outer_n = {"ahat": self.rows, "u": self.rows, "m": self.k, "v": self.k}[name]
        nnz = self.nnz[name]
        o = np.zeros(outer_n + 1, np.int64)
        i = np.zeros(max(nnz, 1), np.int32)
        v = np.zeros(max(nnz, 1))
        lib().or_sp_export(self.h, which, o.ctypes.data_as(C.c_void_p), i.ctypes.data_as(C.c_void_p),
                           v.ctypes.data_as(C.c_void_p))
        return o, i[:nnz], v[:nnz]

    def factors(self):
        return {n: self.export(n) for n in self.NAMES}

    @classmethod
    def from_pieces(cls, piece):
        """Technique B post (sparsify.hpp:246-406) of one Kronecker block from
        raw pieces: dict(key=[k1, k2], cards=[c1, c2], lam=[l1, l2], F, S)
        with F, S dense (n1 x n2) arrays (or_sparsify_pieces)."""
        k1, k2 = [np.ascontiguousarray(k, np.uint32) for k in piece["key"]]
        c1, c2 = [np.ascontiguousarray(c, np.uint8).reshape(-1) for c in piece["cards"]]
        l1, l2 = [np.ascontiguousarray(v, np.float64) for v in piece["lam"]]

        def csr(D):
            D = np.asarray(D, np.float64)
            ptr, col, val = [0], [], []
            for r in range(D.shape[0]):
                nz = np.nonzero(D[r])[0]
                col += nz.tolist()
                val += D[r, nz].tolist()
                ptr.append(len(col))
            return (np.ascontiguousarray(ptr, np.int64), np.ascontiguousarray(col, np.int32),
                    np.ascontiguousarray(val, np.float64))

        F, S = csr(piece["F"]), csr(piece["S"])
        n1, n2 = np.asarray(piece["F"]).shape
        out = C.c_void_p()
        p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        _check(lib().or_sparsify_pieces(len(k1), len(k2), n1, n2, p(k1), p(k2), p(c1), p(c2), p(l1), p(l2),
                                        p(F[0]), p(F[1]), p(F[2]), p(S[0]), p(S[1]), p(S[2]), C.byref(out)))
        sp = cls(out.value)
        sp._keep = (k1, k2, c1, c2, l1, l2, F, S)
        return sp

    @classmethod
    def from_arrays(cls, rows, cols, k, f, technique="b", post=True, validate=True):
        args = []
        for n in cls.NAMES:
            o, i, v = f[n]
            args += [np.ascontiguousarray(o, np.int64), np.ascontiguousarray(i, np.int32),
                     np.ascontiguousarray(v, np.float64)]
        out = C.c_void_p()
        _check(lib().or_sp_from_arrays(C.c_int64(rows), C.c_int64(cols), C.c_int64(k),
                                       *(a.ctypes.data_as(C.c_void_p) for a in args),
                                       0 if technique == "a" else 1, int(post), int(validate), C.byref(out)))
        return cls(out.value)

    def postprocess(self):
        out = C.c_void_p()
        _check(lib().or_postprocess(self.h, C.byref(out)))
        return Sparsification(out.value)

    def matvec(self, x):
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(self.rows)
        fl = C.c_int64()
        _check(lib().or_matvec(self.h, x.ctypes.data_as(C.c_void_p), C.c_int64(len(x)),
                               y.ctypes.data_as(C.c_void_p), C.byref(fl)))
        self.last_flops = fl.value
        return y

    def matvec_t(self, y):
        y = np.ascontiguousarray(y, np.float64)
        x = np.zeros(self.cols)
        fl = C.c_int64()
        _check(lib().or_matvec_t(self.h, y.ctypes.data_as(C.c_void_p), C.c_int64(len(y)),
                                 x.ctypes.data_as(C.c_void_p), C.byref(fl)))
        self.last_flops = fl.value
        return x

    def time_pairs(self, x, y, reps):
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        sink = C.c_double()
        sec = lib().or_time_pairs(self.h, x.ctypes.data_as(C.c_void_p), y.ctypes.data_as(C.c_void_p), reps,
                                  C.byref(sink))
        return sec


def time_pairs_multi(sps, threads, reps):
    arr = (C.c_void_p * len(sps))(*[s.h.value for s in sps])
    sink = C.c_double()
    return lib().or_time_pairs_multi(arr, len(sps), threads, reps, C.byref(sink))


def time_dcfr_multi(pairs, threads, iters):
    """Wall seconds of `iters` DCFR iterations on each (Instance, Sparsification)
    board, one board per thread at a time."""
    ia = (C.c_void_p * len(pairs))(*[i.h.value for i, _ in pairs])
    sa = (C.c_void_p * len(pairs))(*[s.h.value for _, s in pairs])
    sink = C.c_double()
    lib().or_time_dcfr_multi.restype = C.c_double
    return lib().or_time_dcfr_multi(ia, sa, len(pairs), threads, iters, C.byref(sink))


def peel(W, max_iters=1000):
    """sparsifyW (sparsify.hpp:68-103): (rank, nnz What, nnz U, nnz V)."""
    W = np.ascontiguousarray(W, np.float64)
    out = np.zeros(4, np.int64)
    _check(lib().or_peel(W.ctypes.data_as(C.c_void_p), W.shape[0], W.shape[1], max_iters,
                         out.ctypes.data_as(C.c_void_p)))
    return tuple(int(v) for v in out)


def best_response(inst, sp, player, opp):
    opp = np.ascontiguousarray(opp, np.float64)
    out = C.c_double()
    _check(lib().or_best_response(inst.h, sp.h, player, opp.ctypes.data_as(C.c_void_p), C.byref(out)))
    return out.value


class DcfrBoards:
    """Incremental oracle DCFR over independent boards (same interface as the
    product's CudaSolver begin/iterate/checkpoint; multi-rank test stand-in)."""

    def __init__(self, pairs):
        self.pairs = pairs  # keep (Instance, Sparsification) alive
        self.nboards = len(pairs)
        self.hs = []
        for inst, sp in pairs:
            out = C.c_void_p()
            _check(lib().or_dcfr_state_create(inst.h, sp.h, C.byref(out)))
            self.hs.append(out)

    def __del__(self):
        if _LIB is not None:
            for h in getattr(self, "hs", []):
                _LIB.or_dcfr_state_free(h)
            self.hs = []

    def begin(self, alpha=1.5, beta=0.0, gamma=2.0, rule=0):
        for h in self.hs:
            _check(lib().or_dcfr_begin(h, C.c_double(alpha), C.c_double(beta), C.c_double(gamma), int(rule)))

    def iterate(self, n):
        for h in self.hs:
            _check(lib().or_dcfr_iterate(h, int(n)))

    def checkpoint(self):
        b1, b2 = np.zeros(self.nboards), np.zeros(self.nboards)
        for i, h in enumerate(self.hs):
            x, y = C.c_double(), C.c_double()
            _check(lib().or_dcfr_checkpoint(h, C.byref(x), C.byref(y)))
            b1[i], b2[i] = x.value, y.value
        return b1, b2


def dcfr(inst, sp=None, engine="factored", alpha=1.5, beta=0.0, gamma=2.0, max_iters=1000, target=0.0,
         checkpoint_every=50, rule=0):
    """dcfrSolve (solver.hpp:343-404).  Returns a dict with the trace."""
    kind = {"factored": 0, "reference": 1, "dense": 2}[engine]
    cap = max_iters // checkpoint_every + 2
    ti = np.zeros(cap, np.int32)
    te, tb1, tb2 = np.zeros(cap), np.zeros(cap), np.zeros(cap)
    it, ex, fl, nt, sec = C.c_int(), C.c_double(), C.c_int64(), C.c_int(), C.c_double()
    a1, a2 = np.zeros(inst.rows), np.zeros(inst.cols)
    _check(lib().or_dcfr(inst.h, sp.h if sp is not None else None, kind, C.c_double(alpha), C.c_double(beta),
                         C.c_double(gamma), max_iters, C.c_double(target), checkpoint_every, C.byref(it),
                         C.byref(ex), C.byref(fl), ti.ctypes.data_as(C.c_void_p), te.ctypes.data_as(C.c_void_p),
                         tb1.ctypes.data_as(C.c_void_p), tb2.ctypes.data_as(C.c_void_p), cap, C.byref(nt),
                         a1.ctypes.data_as(C.c_void_p), a2.ctypes.data_as(C.c_void_p), C.byref(sec), int(rule)))
    n = min(nt.value, cap)
    return {"iterations": it.value, "exploitability": ex.value, "gradient_flops": fl.value,
            "trace_iter": ti[:n], "trace_expl": te[:n], "trace_br1": tb1[:n], "trace_br2": tb2[:n],
            "avg1": a1, "avg2": a2, "seconds": sec.value}
