"""ctypes bindings of the product's native libraries.

libkrcuda.so exports the kr_* C ABI declared in include/kr_engine.h.  There
is no CPU fallback anywhere below this module: if the CUDA library cannot be
loaded, or no device is present, every product entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import build as _build

KR_STATUS = {0: "OK", 1: "INVALID_INPUT", 2: "PARSE", 3: "IO", 4: "GUARD_EXCEEDED", 5: "DEGENERATE_BELIEFS",
             6: "CONTRACT", 7: "CUDA", 8: "NO_DEVICE"}

_CUDA = None


class KrError(RuntimeError):
    """Library error carrying the reference's stable code (errors.hpp:11-20)."""

    def __init__(self, code, msg):
        self.status = code
        self.code = KR_STATUS.get(code, str(code))
        super().__init__(f"{self.code}: {msg}")


class InvalidInputError(KrError):
    pass


class ContractError(KrError):
    pass


class GuardError(KrError):
    pass


class ParseError(KrError):
    pass


class DegenerateBeliefsError(KrError):
    pass


class NoDeviceError(KrError):
    pass


_ERR_CLASS = {1: InvalidInputError, 2: ParseError, 4: GuardError, 5: DegenerateBeliefsError, 6: ContractError,
              8: NoDeviceError}


class kr_compressed(C.Structure):
    _fields_ = [("outer_size", C.c_int64), ("outer", C.c_void_p), ("inner", C.c_void_p), ("val", C.c_void_p)]


class kr_factors(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("k", C.c_int64), ("ahat", kr_compressed),
                ("u", kr_compressed), ("m", kr_compressed), ("v", kr_compressed), ("n1", C.c_int32),
                ("n2", C.c_int32)]


class kr_kron_board(C.Structure):
    _fields_ = [("m1", C.c_int32), ("m2", C.c_int32), ("n1", C.c_int32), ("n2", C.c_int32), ("key1", C.c_void_p),
                ("key2", C.c_void_p), ("cards1", C.c_void_p), ("cards2", C.c_void_p), ("lambda1", C.c_void_p),
                ("lambda2", C.c_void_p), ("F", kr_compressed), ("S", kr_compressed)]


class kr_treeplex(C.Structure):
    _fields_ = [("n_seq", C.c_int32), ("n_nodes", C.c_int32), ("node_parent_seq", C.c_void_p),
                ("node_action_ptr", C.c_void_p), ("action_seq", C.c_void_p)]


class kr_dcfr_params(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta", C.c_double), ("gamma", C.c_double), ("max_iters", C.c_int32),
                ("target_exploitability", C.c_double), ("checkpoint_every", C.c_int32), ("rule", C.c_int32)]


class kr_dcfr_result(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("exploitability", C.c_double), ("gradient_flops", C.c_int64),
                ("trace_len", C.c_int32), ("trace_cap", C.c_int32), ("trace_iter", C.c_void_p),
                ("trace_expl", C.c_void_p), ("trace_br1", C.c_void_p), ("trace_br2", C.c_void_p),
                ("trace_board_br1", C.c_void_p), ("trace_board_br2", C.c_void_p), ("avg1", C.c_void_p),
                ("avg2", C.c_void_p), ("seconds", C.c_double)]


# Every symbol include/kr_engine.h declares (checked by the CPU test suite).
CUDA_SYMBOLS = [
    "kr_engine_create", "kr_engine_create_boards", "kr_engine_destroy", "kr_engine_dims", "kr_engine_ax",
    "kr_engine_atx", "kr_engine_ax_device", "kr_engine_atx_device", "kr_engine_pair_device", "kr_engine_flops", "kr_engine_last_flops",
    "kr_engine_stream", "kr_engine_device", "kr_engine_launches", "kr_host_alloc", "kr_host_free", "kr_last_error",
    "kr_device_count", "kr_solver_create", "kr_solver_destroy", "kr_solver_run", "kr_solver_best_response",
    "kr_solver_launches", "kr_solver_begin", "kr_solver_iterate", "kr_solver_checkpoint", "kr_solver_averages",
    "kr_solver_iteration", "kr_engine_set_timing", "kr_engine_set_timing_mask", "kr_engine_kernel_times", "kr_engine_create_kron",
    "kr_solver_set_rule", "kr_turn_solver_create", "kr_turn_solver_run", "kr_turn_solver_destroy",
    "kr_turn_solver_launches", "kr_turn_solver_set_exchange", "kr_turn_solver_sizes",
    "kr_factors_build_device", "kr_devfactors_view", "kr_devfactors_seconds", "kr_devfactors_free",
    "kr_engine_create_device_b", "kr_engine_create_kfactored", "kr_engine_pair", "kr_engine_pair_queue", "kr_checked_verify", "kr_checked_selftest", "kr_solver_step_kind", "kr_jit_step_source",
    "kr_comm_unique_id", "kr_comm_init_rank", "kr_comm_init_all", "kr_comm_destroy", "kr_comm_rank", "kr_comm_size",
    "kr_solver_set_comm", "kr_turn_solver_set_comm", "kr_engine_set_selfcheck", "kr_engine_selfcheck_status",
]


def cuda_lib_path():
    # KR_CUDA_LIB_VARIANT=name loads lib/libkrcuda_<name>.so (A/B kernel timing)
    v = os.environ.get("KR_CUDA_LIB_VARIANT")
    return os.path.join(_build.LIBDIR, f"libkrcuda_{v}.so" if v else "libkrcuda.so")


def _torch_nccl():
    """PyTorch's bundled NCCL (the copy libtorch binds), if the wheel is here."""
    try:
        import nvidia.nccl as m
        for d in getattr(m, "__path__", []):
            p = os.path.join(d, "lib", "libnccl.so.2")
            if os.path.exists(p):
                return p
    except ImportError:
        pass
    return None


def cuda():
    """Load libkrcuda.so (building it in-tree if missing)."""
    global _CUDA
    if _CUDA is None:
        nccl = _torch_nccl()
        if nccl:  # kr_comm dlopens NCCL on first use: share PyTorch's copy
            os.environ.setdefault("KR_NCCL_LIB", nccl)
        path = cuda_lib_path()
        if os.environ.get("KR_CUDA_LIB_VARIANT") == "checked":
            _build.build_cuda_variant("checked", ["KR_CHECKED"])   # no-op when current
        elif not os.path.exists(path):
            _build.build_cuda()
        L = C.CDLL(path)
        L.kr_last_error.restype = C.c_char_p
        L.kr_last_error.argtypes = [C.POINTER(C.c_int)]
        L.kr_engine_flops.restype = C.c_int64
        L.kr_engine_last_flops.restype = C.c_int64
        L.kr_engine_launches.restype = C.c_int64
        L.kr_engine_stream.restype = C.c_void_p
        L.kr_host_alloc.restype = C.c_void_p
        L.kr_host_alloc.argtypes = [C.c_int64]
        L.kr_host_free.argtypes = [C.c_void_p]
        for name in ("kr_engine_flops", "kr_engine_last_flops", "kr_engine_launches", "kr_engine_stream",
                     "kr_engine_device", "kr_engine_destroy"):
            getattr(L, name).argtypes = [C.c_void_p]
        L.kr_engine_ax.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64]
        L.kr_engine_atx.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64]
        L.kr_engine_ax_device.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.kr_engine_atx_device.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.kr_engine_pair_device.argtypes = [C.c_void_p] * 6
        L.kr_engine_pair.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                     C.c_void_p, C.c_int64]
        L.kr_jit_step_source.restype = C.c_int64
        L.kr_jit_step_source.argtypes = [C.POINTER(kr_treeplex), C.c_int, C.c_char_p, C.c_int64]
        L.kr_solver_step_kind.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_char_p)]
        L.kr_checked_verify.restype = C.c_int64
        L.kr_checked_verify.argtypes = []
        L.kr_checked_selftest.restype = C.c_int64
        L.kr_checked_selftest.argtypes = [C.c_int]
        L.kr_engine_pair_queue.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                           C.c_void_p, C.c_int64, C.c_void_p, C.c_int64]
        L.kr_engine_dims.argtypes = [C.c_void_p, C.c_void_p]
        L.kr_engine_create.argtypes = [C.POINTER(kr_factors), C.c_int, C.c_uint32, C.POINTER(C.c_void_p)]
        L.kr_engine_create_boards.argtypes = [C.POINTER(kr_factors), C.c_int, C.c_int, C.c_uint32,
                                              C.POINTER(C.c_void_p)]
        L.kr_engine_create_kron.argtypes = [C.POINTER(kr_kron_board), C.c_int, C.c_int, C.c_uint32,
                                            C.POINTER(C.c_void_p)]
        if hasattr(L, "kr_solver_create"):
            L.kr_solver_create.argtypes = [C.c_void_p, C.POINTER(kr_treeplex), C.POINTER(kr_treeplex), C.c_int,
                                           C.c_void_p, C.c_void_p, C.c_double, C.POINTER(C.c_void_p)]
            L.kr_solver_destroy.argtypes = [C.c_void_p]
            L.kr_solver_run.argtypes = [C.c_void_p, C.POINTER(kr_dcfr_params), C.POINTER(kr_dcfr_result)]
            L.kr_solver_best_response.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64,
                                                  C.POINTER(C.c_double), C.c_void_p]
            L.kr_solver_launches.restype = C.c_int64
            L.kr_solver_launches.argtypes = [C.c_void_p]
            L.kr_solver_begin.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_double]
            L.kr_solver_set_rule.argtypes = [C.c_void_p, C.c_int]
            L.kr_solver_iterate.argtypes = [C.c_void_p, C.c_int]
            L.kr_solver_checkpoint.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
            L.kr_solver_averages.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
            L.kr_solver_iteration.argtypes = [C.c_void_p]
        L.kr_turn_solver_create.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.POINTER(kr_treeplex),
                                            C.POINTER(kr_treeplex), C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                            C.c_void_p, C.c_double, C.POINTER(C.c_void_p)]
        L.kr_turn_solver_run.argtypes = [C.c_void_p, C.POINTER(kr_dcfr_params), C.POINTER(kr_dcfr_result)]
        L.kr_turn_solver_destroy.argtypes = [C.c_void_p]
        L.kr_turn_solver_launches.restype = C.c_int64
        L.kr_turn_solver_launches.argtypes = [C.c_void_p]
        L.kr_turn_solver_set_exchange.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p,
                                                  C.c_void_p, C.c_void_p]
        L.kr_turn_solver_set_comm.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.kr_solver_set_comm.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.kr_comm_unique_id.argtypes = [C.c_void_p]
        L.kr_comm_init_rank.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.kr_comm_init_all.argtypes = [C.c_int, C.c_void_p, C.c_void_p]
        L.kr_comm_destroy.argtypes = [C.c_void_p]
        L.kr_comm_rank.argtypes = [C.c_void_p]
        L.kr_comm_size.argtypes = [C.c_void_p]
        L.kr_engine_set_selfcheck.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_double]
        L.kr_engine_selfcheck_status.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.kr_turn_solver_sizes.argtypes = [C.c_void_p, C.c_void_p]
        L.kr_engine_create_device_b.argtypes = [C.POINTER(kr_kron_board), C.c_int, C.c_int, C.c_uint32,
                                                C.POINTER(C.c_void_p)]
        L.kr_engine_create_kfactored.argtypes = [C.POINTER(kr_kron_board), C.c_int, C.c_int, C.c_uint32,
                                                 C.POINTER(C.c_void_p)]
        L.kr_factors_build_device.argtypes = [C.POINTER(kr_kron_board), C.c_int, C.POINTER(C.c_void_p)]
        L.kr_devfactors_view.argtypes = [C.c_void_p, C.POINTER(kr_factors)]
        L.kr_devfactors_seconds.restype = C.c_double
        L.kr_devfactors_seconds.argtypes = [C.c_void_p]
        L.kr_devfactors_free.argtypes = [C.c_void_p]
        L.kr_engine_set_timing.argtypes = [C.c_void_p, C.c_int]
        L.kr_engine_set_timing_mask.argtypes = [C.c_void_p, C.c_int]
        L.kr_engine_kernel_times.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        _CUDA = L
    return _CUDA


def check(rc):
    if rc != 0:
        code = C.c_int()
        msg = cuda().kr_last_error(C.byref(code)).decode()
        raise _ERR_CLASS.get(rc, KrError)(rc, msg)


def device_count():
    return int(cuda().kr_device_count())


def ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def compressed(outer, inner, val, keep):
    outer = np.ascontiguousarray(outer, np.int64)
    inner = np.ascontiguousarray(inner, np.int32)
    val = np.ascontiguousarray(val, np.float64)
    keep += [outer, inner, val]
    return kr_compressed(len(outer) - 1, ptr(outer), ptr(inner), ptr(val))
