"""Host side of the product, bound from libkrhost.so (include/kr_host.h).

Python mirror of the reference interfaces upstream of the gradient oracle
(/root/reference/proj/include/kronriver/):
    read_instance(path)            readInstance          instance_io.hpp:237-247
    builtin(name, ...)             instances.hpp constructors
    Instance                       RiverInstance + KronPayoff (kron.hpp:18-166)
    Instance.sparsify(t, post)     techniqueA/techniqueB (+ postprocess)
    Factors.postprocess()          postprocess            sparsify.hpp:318-406
    Factors.write_bundle / read_bundle   bundle_io.hpp:27-94
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _native as N
from . import build as _build

_HOST = None

HOST_SYMBOLS = [
    "krh_instance_from_json", "krh_instance_builtin", "krh_instance_free", "krh_instance_dims", "krh_instance_beta",
    "krh_instance_pot", "krh_instance_hands", "krh_instance_vectors", "krh_instance_treeplex", "krh_dense_nnz",
    "krh_sparsify", "krh_postprocess", "krh_factors_from_arrays", "krh_factors_free", "krh_factors_dims",
    "krh_factors_view", "krh_factors_validate", "krh_bundle_write", "krh_bundle_read", "krh_last_error",
    "krh_instance_kron_view", "krh_instance_custom",
]


def host_lib_path():
    return os.path.join(_build.LIBDIR, "libkrhost.so")


def host():
    global _HOST
    if _HOST is None:
        path = host_lib_path()
        if not os.path.exists(path):
            _build.build_host()
        L = C.CDLL(path)
        L.krh_last_error.restype = C.c_char_p
        L.krh_last_error.argtypes = [C.POINTER(C.c_int)]
        L.krh_instance_beta.restype = C.c_double
        L.krh_instance_pot.restype = C.c_double
        L.krh_dense_nnz.restype = C.c_int64
        for f in ("krh_instance_beta", "krh_instance_pot", "krh_dense_nnz", "krh_instance_free", "krh_factors_free",
                  "krh_factors_validate"):
            getattr(L, f).argtypes = [C.c_void_p]
        L.krh_instance_builtin.argtypes = [C.c_char_p, C.c_uint64, C.c_int, C.c_int, C.c_char_p, C.c_int, C.c_int,
                                           C.POINTER(C.c_void_p)]
        L.krh_instance_from_json.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        L.krh_instance_dims.argtypes = [C.c_void_p, C.c_void_p]
        L.krh_instance_hands.argtypes = [C.c_void_p, C.c_int, C.c_char_p]
        L.krh_instance_vectors.argtypes = [C.c_void_p] + [C.c_void_p] * 4
        L.krh_instance_treeplex.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        L.krh_instance_kron_view.argtypes = [C.c_void_p, C.POINTER(N.kr_kron_board)]
        L.krh_instance_custom.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                          C.c_int, C.c_double, C.c_double, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                          C.POINTER(C.c_void_p)]
        L.krh_sparsify.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.krh_postprocess.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)]
        L.krh_factors_from_arrays.argtypes = [C.POINTER(N.kr_factors), C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.krh_factors_dims.argtypes = [C.c_void_p, C.c_void_p]
        L.krh_factors_view.argtypes = [C.c_void_p, C.POINTER(N.kr_factors)]
        L.krh_bundle_write.argtypes = [C.c_void_p, C.c_char_p]
        L.krh_bundle_read.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        _HOST = L
    return _HOST


def _check(rc):
    if rc != 0:
        code = C.c_int()
        msg = host().krh_last_error(C.byref(code)).decode()
        raise N._ERR_CLASS.get(rc, N.KrError)(rc, msg)


class Instance:
    """RiverInstance + KronPayoff (kron.hpp:18-166), strength-sorted hands."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle)
        d = np.zeros(16, np.int64)
        _check(host().krh_instance_dims(self._h, N.ptr(d)))
        (self.m1, self.m2, self.n1, self.n2, self.rows, self.cols, self.nodes, self.dec1, self.dec2, self.terminals,
         self.folds, self.showdowns, self.nnzF, self.nnzS, self.actions1, self.actions2) = [int(v) for v in d]

    def __del__(self):
        if _HOST is not None and getattr(self, "_h", None) and self._h.value:
            _HOST.krh_instance_free(self._h)
            self._h = C.c_void_p()

    @property
    def beta(self):
        return host().krh_instance_beta(self._h)

    @property
    def pot(self):
        """2 * potContribution (solver.hpp:329)."""
        return host().krh_instance_pot(self._h)

    def hand_count(self, player):
        return self.m1 if player == 0 else self.m2

    def hands(self, player):
        n = self.hand_count(player)
        buf = C.create_string_buffer(4 * n + 1)
        _check(host().krh_instance_hands(self._h, player, buf))
        raw = buf.raw[:4 * n].decode()
        return [raw[4 * i:4 * i + 4] for i in range(n)]

    def vectors(self):
        mu1, mu2, l1, l2 = np.zeros(self.m1), np.zeros(self.m2), np.zeros(self.m1), np.zeros(self.m2)
        _check(host().krh_instance_vectors(self._h, N.ptr(mu1), N.ptr(mu2), N.ptr(l1), N.ptr(l2)))
        return mu1, mu2, l1, l2

    def treeplex(self, player):
        from .solver import Treeplex
        nodes = self.dec1 if player == 0 else self.dec2
        acts = self.actions1 if player == 0 else self.actions2
        parent = np.zeros(nodes, np.int32)
        aptr = np.zeros(nodes + 1, np.int32)
        aseq = np.zeros(max(acts, 1), np.int32)
        _check(host().krh_instance_treeplex(self._h, player, N.ptr(parent), N.ptr(aptr), N.ptr(aseq)))
        return Treeplex(self.n1 if player == 0 else self.n2, parent, aptr, aseq[:acts])

    def kron_view(self):
        """kr_kron_board for kr_engine_create_kron (valid while self lives)."""
        v = N.kr_kron_board()
        _check(host().krh_instance_kron_view(self._h, C.byref(v)))
        return v

    def sparsify_device(self, device=0):
        """Technique B with postprocessing built on the device
        (kr_factors_build_device), bit-exact against sparsify("b", True)."""
        return DeviceFactors(self, device)

    def dense_nnz(self):
        """densePayoffNonzeros (kron.hpp:198-207)."""
        return int(host().krh_dense_nnz(self._h))

    def sparsify(self, technique="b", post=True, peel_iters=1000):
        """techniqueA / techniqueB (sparsify.hpp:165-312), optionally postprocessed."""
        out = C.c_void_p()
        _check(host().krh_sparsify(self._h, 0 if technique.lower() == "a" else 1, int(post), peel_iters,
                                   C.byref(out)))
        return Factors(out.value)


class Factors:
    """Sparsification (sparsify.hpp:110-121): Ahat CSR, U CSR, M CSC, V CSC."""

    NAMES = ("ahat", "u", "m", "v")

    def __init__(self, handle):
        self._h = C.c_void_p(handle)
        d = np.zeros(9, np.int64)
        _check(host().krh_factors_dims(self._h, N.ptr(d)))
        self.rows, self.cols, self.k = int(d[0]), int(d[1]), int(d[2])
        self.nnz = {"ahat": int(d[3]), "u": int(d[4]), "m": int(d[5]), "v": int(d[6])}
        self.technique = "a" if d[7] == 0 else "b"
        self.postprocessed = bool(d[8])

    def __del__(self):
        if _HOST is not None and getattr(self, "_h", None) and self._h.value:
            _HOST.krh_factors_free(self._h)
            self._h = C.c_void_p()

    def size(self):
        """SizeReport::total (sparsify.hpp:123-130): nnz including M's diagonal."""
        return sum(self.nnz.values())

    def view(self):
        """kr_factors pointing into this object's storage (for kr_engine_create)."""
        v = N.kr_factors()
        _check(host().krh_factors_view(self._h, C.byref(v)))
        return v

    def factors(self):
        """name -> (outer, inner, val) numpy copies in the reference storage order."""
        v = self.view()
        out = {}
        for name in self.NAMES:
            c = getattr(v, name)
            no = c.outer_size
            outer = np.ctypeslib.as_array(C.cast(c.outer, C.POINTER(C.c_int64)), (no + 1,)).copy()
            nnz = int(outer[-1])
            if nnz:
                inner = np.ctypeslib.as_array(C.cast(c.inner, C.POINTER(C.c_int32)), (nnz,)).copy()
                val = np.ctypeslib.as_array(C.cast(c.val, C.POINTER(C.c_double)), (nnz,)).copy()
            else:
                inner, val = np.zeros(0, np.int32), np.zeros(0)
            out[name] = (outer, inner, val)
        out["n1"], out["n2"] = int(v.n1), int(v.n2)
        return out

    def validate(self):
        _check(host().krh_factors_validate(self._h))

    def postprocess(self):
        out = C.c_void_p()
        _check(host().krh_postprocess(self._h, C.byref(out)))
        return Factors(out.value)

    def write_bundle(self, directory):
        _check(host().krh_bundle_write(self._h, os.fsencode(directory)))

    @classmethod
    def read_bundle(cls, directory):
        out = C.c_void_p()
        _check(host().krh_bundle_read(os.fsencode(directory), C.byref(out)))
        return cls(out.value)

    @classmethod
    def from_arrays(cls, rows, cols, k, f, technique="b", postprocessed=True, n1=0, n2=0):
        keep = []
        kf = N.kr_factors(rows, cols, k, *(N.compressed(*f[n], keep) for n in cls.NAMES), n1, n2)
        out = C.c_void_p()
        _check(host().krh_factors_from_arrays(C.byref(kf), 0 if technique == "a" else 1, int(postprocessed),
                                              C.byref(out)))
        return cls(out.value)


class DeviceFactors:
    """Factors built on the device (kr_factors_build_device), held as host
    copies; the same interface as Factors for engines and comparisons."""

    NAMES = Factors.NAMES

    def __init__(self, inst, device=0):
        v = inst.kron_view()
        out = C.c_void_p()
        N.check(N.cuda().kr_factors_build_device(C.byref(v), device, C.byref(out)))
        self._h = out
        fv = N.kr_factors()
        N.check(N.cuda().kr_devfactors_view(self._h, C.byref(fv)))
        self._v = fv
        self.rows, self.cols, self.k = int(fv.rows), int(fv.cols), int(fv.k)
        self.seconds = N.cuda().kr_devfactors_seconds(self._h)
        self.nnz = {}
        for n in self.NAMES:
            c = getattr(fv, n)
            self.nnz[n] = int(np.ctypeslib.as_array(C.cast(c.outer, C.POINTER(C.c_int64)), (c.outer_size + 1,))[-1])

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            N.cuda().kr_devfactors_free(self._h)
            self._h = C.c_void_p()

    def size(self):
        return sum(self.nnz.values())

    def view(self):
        return self._v

    factors = Factors.factors


def builtin(name, seed=1, hands=0, shared=0, board="", deck=52, tree=1):
    out = C.c_void_p()
    _check(host().krh_instance_builtin(name.encode(), seed, hands, shared, board.encode(), deck, tree, C.byref(out)))
    return Instance(out.value)


def custom_instance(board, deck, cards1, w1, cards2, w2, stack, pot, menu, all_in=True, raise_cap=-1):
    """krh_instance_custom: a river instance from explicit pieces.  board: 5
    card ids; cards*: (m, 2) uint8 card ids; w*: belief weights; menu: pot
    fractions used in every betting context by both players."""
    b = np.ascontiguousarray(board, np.int32)
    c1 = np.ascontiguousarray(cards1, np.uint8).reshape(-1, 2)
    c2 = np.ascontiguousarray(cards2, np.uint8).reshape(-1, 2)
    w1 = np.ascontiguousarray(w1, np.float64)
    w2 = np.ascontiguousarray(w2, np.float64)
    mn = np.ascontiguousarray(menu, np.float64)
    out = C.c_void_p()
    _check(host().krh_instance_custom(N.ptr(b), deck, N.ptr(c1), N.ptr(w1), len(c1), N.ptr(c2), N.ptr(w2), len(c2),
                                      float(stack), float(pot), N.ptr(mn), len(mn), int(all_in), int(raise_cap),
                                      C.byref(out)))
    return Instance(out.value)


def read_instance(path):
    """readInstance (instance_io.hpp:237-247)."""
    out = C.c_void_p()
    _check(host().krh_instance_from_json(os.fsencode(path), C.byref(out)))
    return Instance(out.value)


def turn_boards(turn="Ks7d4c2h", nboards=48, tree=3, seed_base=1000):
    """Config 3: the river boards under a turn, one full-range
    river per card, beliefs seeded with seed_base + card id."""
    ranks, suits = "23456789TJQKA", "cdhs"
    used = {turn[i:i + 2] for i in range(0, len(turn), 2)}
    cards = [r + s for r in ranks for s in suits if r + s not in used][:nboards]
    return [(c, seed_base + ranks.index(c[0]) * 4 + suits.index(c[1])) for c in cards]


def turn_instances(turn="Ks7d4c2h", nboards=48, tree=3, threads=None, indices=None, factors=True):
    """Build the turn's river instances (and B-post factors) in parallel threads
    (libkrhost releases the GIL inside each ctypes call).  `indices` selects a
    subset of the boards (a rank's shard)."""
    from concurrent.futures import ThreadPoolExecutor
    specs = turn_boards(turn, nboards, tree)
    if indices is not None:
        specs = [specs[i] for i in indices]

    def one(spec):
        card, seed = spec
        inst = builtin("river_full", seed=seed, board=turn + card, tree=tree)
        return inst, (inst.sparsify("b", True) if factors else None)

    with ThreadPoolExecutor(max_workers=threads or min(16, os.cpu_count() or 1)) as ex:
        return list(ex.map(one, specs))
