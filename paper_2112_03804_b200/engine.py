"""CudaEngine: the reference's GradientEngine boundary on the B200.

Mirrors kronriver::FactoredEngine (solver.hpp:30-40):
    Ax(x2)  -> A x2     (matvec, engine.hpp:58-93)
    ATx(x1) -> A^T x1   (matvecTranspose, engine.hpp:96-133)
    flops() -> cumulative multiply-adds (engine.hpp:16-17)
through the C ABI of libkrcuda.so.  Errors carry the reference codes
(InvalidInputError for size mismatches, ContractError for a bad M).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N


def _factor_struct(sp, keep):
    f = sp.factors() if hasattr(sp, "factors") else sp
    get = (lambda k: f[k]) if isinstance(f, dict) else (lambda k: getattr(f, k))
    rows, cols, k = int(getattr(sp, "rows", None) or get("rows")), int(getattr(sp, "cols", None) or get("cols")), \
        int(getattr(sp, "k", None) if getattr(sp, "k", None) is not None else get("k"))
    n1 = int(getattr(sp, "n1", 0) or (f.get("n1", 0) if isinstance(f, dict) else 0))
    n2 = int(getattr(sp, "n2", 0) or (f.get("n2", 0) if isinstance(f, dict) else 0))
    parts = [N.compressed(*get(name), keep) for name in ("ahat", "u", "m", "v")]
    return N.kr_factors(rows, cols, k, *parts, n1, n2)


class CudaEngine:
    """GradientEngine whose products run as sm_100a kernels in HBM.

    `factors` is one Sparsification-like object (attributes rows/cols/k and a
    factors() mapping name -> (outer, inner, val) in the reference storage
    order), or a list of them for a block-diagonal multi-board engine.
    """

    def __init__(self, factors, device=0, flags=0):
        L = N.cuda()
        keep = []
        boards = factors if isinstance(factors, (list, tuple)) else [factors]
        arr = (N.kr_factors * len(boards))(*[_factor_struct(b, keep) for b in boards])
        h = C.c_void_p()
        N.check(L.kr_engine_create_boards(arr, len(boards), device, flags, C.byref(h)))
        self._attach(h, device, len(boards))

    @classmethod
    def kron(cls, instances, device=0, flags=0):
        """Implicit Kronecker engine (kr_engine_create_kron): the same products
        computed from each board's F, S, strength keys, cards and lambdas with
        nothing materialised.  `instances` is one
        host.Instance or a list of them sharing one betting tree."""
        insts = instances if isinstance(instances, (list, tuple)) else [instances]
        return cls.from_kron_boards([i.kron_view() for i in insts], device, flags)

    @classmethod
    def from_kron_boards(cls, boards, device=0, flags=0, kind="implicit"):
        """Engine from kr_kron_board structs (the caller keeps the arrays they
        point to alive until this returns: the engine copies): the implicit
        engine (K7), or kind="kfactored" the Kronecker-factored one."""
        L = N.cuda()
        arr = (N.kr_kron_board * len(boards))(*boards)
        h = C.c_void_p()
        create = L.kr_engine_create_kfactored if kind == "kfactored" else L.kr_engine_create_kron
        N.check(create(arr, len(boards), device, flags, C.byref(h)))
        self = cls.__new__(cls)
        self._attach(h, device, len(boards))
        self.implicit = kind != "kfactored"
        self.kfactored_mode = kind == "kfactored"
        return self

    @classmethod
    def device_built(cls, instances, device=0, flags=0):
        """The factored engine (Technique B post) built entirely on the device
        from the instances' KronPayoff pieces (kr_engine_create_device_b):
        bitwise the products of CudaEngine([inst.sparsify("b", True) ...])."""
        L = N.cuda()
        insts = instances if isinstance(instances, (list, tuple)) else [instances]
        arr = (N.kr_kron_board * len(insts))(*[i.kron_view() for i in insts])
        h = C.c_void_p()
        N.check(L.kr_engine_create_device_b(arr, len(insts), device, flags, C.byref(h)))
        self = cls.__new__(cls)
        self._attach(h, device, len(insts))
        return self

    @classmethod
    def kfactored(cls, instances, device=0, flags=0):
        """Kronecker-factored engine (kr_engine_create_kfactored): Technique B
        post kept as its hand-space factors and the tree's F and S, every
        Kronecker product expanded on the fly; products bitwise those of
        CudaEngine([inst.sparsify("b", True) ...])."""
        L = N.cuda()
        insts = instances if isinstance(instances, (list, tuple)) else [instances]
        arr = (N.kr_kron_board * len(insts))(*[i.kron_view() for i in insts])
        h = C.c_void_p()
        N.check(L.kr_engine_create_kfactored(arr, len(insts), device, flags, C.byref(h)))
        self = cls.__new__(cls)
        self._attach(h, device, len(insts))
        self.kfactored_mode = True
        return self

    implicit = False
    kfactored_mode = False

    # -- SelfCheckEngine (solver.hpp:67-99) on the device -------------------
    def set_selfcheck(self, reference, every=500, tol=1e-8):
        """Replay every `every`-th product through `reference` (an engine over
        the same boards, typically CudaEngine.kron: the block formula) and
        compare on the device; a deviation above tol (1 + max|expect|) makes
        the next host call raise ContractError.  reference=None: off."""
        N.check(N.cuda().kr_engine_set_selfcheck(self._h, reference.handle if reference else None, int(every),
                                                 float(tol)))
        self._sc_ref = reference  # keep the reference engine alive

    def selfcheck_status(self):
        """(checks made, worst err / (tol (1 + max|expect|))); raises
        ContractError if a check failed."""
        n, w = C.c_int64(), C.c_double()
        N.check(N.cuda().kr_engine_selfcheck_status(self._h, C.byref(n), C.byref(w)))
        return n.value, w.value

    def _attach(self, h, device, nboards):
        self._h = h
        dims = np.zeros(8, np.int64)
        N.check(N.cuda().kr_engine_dims(self._h, N.ptr(dims)))
        self.rows, self.cols, self.k = int(dims[0]), int(dims[1]), int(dims[2])
        self.nnz = {"ahat": int(dims[3]), "u": int(dims[4]), "m": int(dims[5]), "v": int(dims[6])}
        self.m_identity = bool(dims[7])
        self.device = device
        self.nboards = nboards

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            N.cuda().kr_engine_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    # -- GradientEngine (solver.hpp:21-27) --------------------------------
    def Ax(self, x2):
        x = np.ascontiguousarray(x2, np.float64)
        y = np.empty(self.rows)
        N.check(N.cuda().kr_engine_ax(self._h, N.ptr(x), len(x), N.ptr(y), len(y)))
        return y

    def pair(self, x2, x1, out=None):
        """(A x2, Aᵀ x1) through kr_engine_pair: both directions' host<->device
        copies and kernels in flight together (bitwise Ax then ATx).  `out`:
        optional (ax, atx) host arrays to fill (pinned ones replay a graph)."""
        x = np.ascontiguousarray(x2, np.float64)
        y = np.ascontiguousarray(x1, np.float64)
        ax, atx = out if out is not None else (np.empty(self.rows), np.empty(self.cols))
        N.check(N.cuda().kr_engine_pair(self._h, N.ptr(x), len(x), N.ptr(ax), len(ax), N.ptr(y), len(y), N.ptr(atx),
                                        len(atx)))
        return ax, atx

    def pair_queue(self, xs, ys, out=None):
        """A queue of independent pairs through kr_engine_pair_queue: returns
        ([A x for x in xs], [Aᵀ y for y in ys]), each the bits of `pair`.  The
        input copies of the next pair and the output copies of the previous
        one overlap each pair's kernels.  `out`: optional (axs, atxs) lists
        of host arrays to fill (pinned ones keep the bus at its duplex rate)."""
        if len(xs) != len(ys):
            raise ValueError("xs and ys must have the same length")
        xs = [np.ascontiguousarray(x, np.float64) for x in xs]
        ys = [np.ascontiguousarray(y, np.float64) for y in ys]
        axs, atxs = out if out is not None else ([np.empty(self.rows) for _ in xs], [np.empty(self.cols) for _ in ys])
        P = C.c_void_p * max(len(xs), 1)
        px, py = P(*[N.ptr(a) for a in xs]), P(*[N.ptr(a) for a in ys])
        pax, patx = P(*[N.ptr(a) for a in axs]), P(*[N.ptr(a) for a in atxs])
        nx = len(xs[0]) if xs else self.cols
        ny = len(ys[0]) if ys else self.rows
        if any(len(a) != nx for a in xs) or any(len(a) != ny for a in ys):
            raise N.InvalidInputError("queued inputs must all have the same length")
        N.check(N.cuda().kr_engine_pair_queue(self._h, len(xs), px, nx, pax, len(axs[0]) if axs else self.rows, py, ny,
                                              patx, len(atxs[0]) if atxs else self.cols))
        return axs, atxs

    def ATx(self, x1):
        y = np.ascontiguousarray(x1, np.float64)
        x = np.empty(self.cols)
        N.check(N.cuda().kr_engine_atx(self._h, N.ptr(y), len(y), N.ptr(x), len(x)))
        return x

    def flops(self):
        return int(N.cuda().kr_engine_flops(self._h))

    def last_flops(self):
        return int(N.cuda().kr_engine_last_flops(self._h))

    def launches(self):
        return int(N.cuda().kr_engine_launches(self._h))

    def flops_per_product(self):
        nz = self.nnz
        return nz["v"] + nz["u"] + nz["ahat"] + (0 if self.m_identity else nz["m"] - self.k)

    def bytes_per_product(self):
        """Algorithmic HBM bytes of one product (BASELINE.md §2 formula):
        fp64 values + int32 indices + int32 outer pointers of Ahat, U, V (and
        M's off-diagonals when M != I), plus reading x and writing y.  The
        implicit engine materialises nothing: reading x and writing y."""
        if self.implicit:
            return 8 * (self.rows + self.cols)
        nz = self.nnz
        b = 12 * nz["ahat"] + 4 * (self.rows + 1) + 12 * nz["u"] + 4 * (self.rows + 1) \
            + 12 * nz["v"] + 4 * (self.k + 1) + 8 * (self.rows + self.cols)
        if not self.m_identity:
            b += 12 * (nz["m"] - self.k) + 4 * (self.k + 1)
        return b

    # -- per-kernel event timing (kr_engine_set_timing) -------------------
    KERNELS = ("VT", "UA", "UT", "AV")  # V^T x | [U|Ahat][z;x] | U^T y | [Ahat^T|V][y;z]

    def set_timing(self, enabled=True, only=None):
        """Bracket SpMV launches with events; only: names from KERNELS (all if None)."""
        mask = 0xF if only is None else sum(1 << self.KERNELS.index(k) for k in only)
        N.check(N.cuda().kr_engine_set_timing_mask(self._h, mask))
        N.check(N.cuda().kr_engine_set_timing(self._h, int(enabled)))

    def kernel_times(self):
        """Per SpMV matrix since the last call: launches, total ms, algorithmic
        bytes of one launch."""
        n = np.zeros(4, np.int64)
        ms, by = np.zeros(4), np.zeros(4)
        N.check(N.cuda().kr_engine_kernel_times(self._h, N.ptr(n), N.ptr(ms), N.ptr(by)))
        return {k: {"launches": int(n[i]), "ms": float(ms[i]), "bytes_per_launch": float(by[i])}
                for i, k in enumerate(self.KERNELS)}

    # -- device-pointer variants (torch tensors on the engine's device) ----
    @property
    def stream(self):
        return N.cuda().kr_engine_stream(self._h)

    def ax_device(self, x_ptr, y_ptr, stream=None):
        N.check(N.cuda().kr_engine_ax_device(self._h, C.c_void_p(x_ptr), C.c_void_p(y_ptr),
                                             C.c_void_p(stream) if stream else None))

    def atx_device(self, y_ptr, x_ptr, stream=None):
        N.check(N.cuda().kr_engine_atx_device(self._h, C.c_void_p(y_ptr), C.c_void_p(x_ptr),
                                              C.c_void_p(stream) if stream else None))

    def pair_device(self, x_ptr, ax_ptr, y_ptr, atx_ptr, stream=None):
        """A x and A^T y in flight together (kr_engine_pair_device)."""
        N.check(N.cuda().kr_engine_pair_device(self._h, C.c_void_p(x_ptr), C.c_void_p(ax_ptr), C.c_void_p(y_ptr),
                                               C.c_void_p(atx_ptr), C.c_void_p(stream) if stream else None))
