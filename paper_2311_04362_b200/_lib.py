"""ctypes binding of libitsk_b200.so (include/itsk_b200.h).

The product path has no CPU fallback: if the library is missing or no sm_100
device is present, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libitsk_b200.so")

ITSK_OK, ITSK_EINVAL, ITSK_ESINGULAR, ITSK_ECUDA, ITSK_ENODEV = range(5)
STOP_REASONS = {0: "max_iters", 1: "stopped_by_rule", 2: "diverged"}

c_i64 = ctypes.c_int64
c_dp = ctypes.c_void_p


class SingularMatrixError(ValueError):
    """A triangular factor has an exactly-zero diagonal entry
    (mirrors itsketch.linalg.SingularMatrixError, linalg.py:17-18)."""


class ItskCudaError(RuntimeError):
    pass


class LoopParams(ctypes.Structure):
    """itsk_loop_params (include/itsk_b200.h)."""

    _fields_ = [
        ("m", c_i64), ("n", c_i64), ("lda", c_i64),
        ("max_iters", c_i64), ("extra_iters", c_i64),
        ("variant", ctypes.c_int32), ("r_slots", ctypes.c_int32),
        ("alpha", ctypes.c_double), ("beta", ctypes.c_double),
        ("u", ctypes.c_double), ("gamma", ctypes.c_double), ("rho", ctypes.c_double),
        ("truth_beta", ctypes.c_double),
        ("has_truth", ctypes.c_int32),
        ("A", c_dp), ("b", c_dp), ("R", c_dp), ("Rp", c_dp), ("x_true", c_dp), ("r_true", c_dp),
        ("normest", c_dp), ("condest", c_dp),
        ("xs", c_dp), ("rs", c_dp), ("trace", c_dp), ("cs", c_dp),
        ("ws", c_dp), ("ws_bytes", c_i64),
        ("csr", c_dp),
        ("est_ready", c_dp),
        ("peer", c_dp),
        ("opts", ctypes.c_uint32),
    ]


MAX_PEERS = 8  # include/itsk_b200.h ITSK_MAX_PEERS


class PeerParams(ctypes.Structure):
    """itsk_peer_params (include/itsk_b200.h)."""

    _fields_ = [
        ("rank", ctypes.c_int32), ("size", ctypes.c_int32), ("epoch_base", c_i64),
        ("recv", c_dp * MAX_PEERS), ("flags", c_dp * MAX_PEERS),
    ]


class LoopResult(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int32), ("stop_reason", ctypes.c_int32),
        ("done", ctypes.c_int32), ("sol_slot", ctypes.c_int32),
        ("bnorm2", ctypes.c_double), ("pad", ctypes.c_double * 3),
    ]


_SIGS = {
    "itsk_last_error": (ctypes.c_char_p, []),
    "itsk_version": (ctypes.c_int, []),
    "itsk_device_check": (ctypes.c_int, [ctypes.c_int]),
    "itsk_launch_count": (c_i64, []),
    "itsk_pattern_workspace": (ctypes.c_int, [c_i64, c_i64, c_i64, ctypes.POINTER(c_i64)]),
    "itsk_sparse_sign_pattern": (ctypes.c_int, [c_i64, c_i64, c_i64, ctypes.POINTER(ctypes.c_uint64),
                                                ctypes.c_int, ctypes.c_uint32, c_dp, c_dp, c_dp, c_dp,
                                                c_dp, c_i64, c_dp]),
    "itsk_pattern_csr": (ctypes.c_int, [c_dp, c_dp, c_i64, c_i64, c_i64, c_dp, c_dp, c_dp, c_i64, c_dp]),
    "itsk_sketch": (ctypes.c_int, [c_dp, c_i64, c_i64, c_i64, c_dp, c_dp, c_dp, c_i64, c_i64, c_dp,
                                   c_i64, c_dp]),
    "itsk_sketch_rows": (ctypes.c_int, [c_dp, c_i64, c_i64, c_i64, c_dp, c_dp, c_dp, c_i64, c_i64, c_dp,
                                        c_i64, c_i64, c_i64, ctypes.c_int, c_dp]),
    "itsk_qr_workspace": (ctypes.c_int, [c_i64, c_i64, ctypes.POINTER(c_i64)]),
    "itsk_qr_row_blocks": (ctypes.c_int, [c_i64, c_i64, ctypes.POINTER(c_i64)]),
    "itsk_qr_aug": (ctypes.c_int, [c_dp, c_i64, c_i64, c_i64, c_dp, c_dp, c_dp, c_i64, c_dp]),
    "itsk_qr_aug_async": (ctypes.c_int, [c_dp, c_i64, c_i64, c_i64, c_dp, c_dp, c_dp, c_i64, c_dp, c_dp]),
    "itsk_trsv": (ctypes.c_int, [c_dp, c_i64, c_dp, c_dp, ctypes.c_int, c_dp]),
    "itsk_trsv_rp": (ctypes.c_int, [c_dp, c_dp, c_i64, c_dp, c_dp, ctypes.c_int, c_dp]),
    "itsk_trsv_pair_cl": (ctypes.c_int, [c_dp, c_dp, c_i64, c_dp, c_dp, c_dp]),
    "itsk_trsv_pair": (ctypes.c_int, [c_dp, c_i64, c_dp, c_dp, c_dp, c_dp]),
    "itsk_normest": (ctypes.c_int, [c_dp, c_i64, c_dp, c_i64, c_dp, c_dp, c_dp]),
    "itsk_pack_upper_doubles": (ctypes.c_int, [c_i64, ctypes.POINTER(c_i64)]),
    "itsk_pack_upper": (ctypes.c_int, [c_dp, c_i64, c_dp, c_dp]),
    "itsk_condest_workspace": (ctypes.c_int, [c_i64, ctypes.POINTER(c_i64)]),
    "itsk_condest": (ctypes.c_int, [c_dp, c_i64, c_dp, c_dp, c_dp, c_dp]),
    "itsk_condest_ws": (ctypes.c_int, [c_dp, c_i64, c_dp, c_dp, c_dp, c_dp, c_i64, c_dp]),
    "itsk_pass_workspace": (ctypes.c_int, [c_i64, c_i64, ctypes.POINTER(c_i64)]),
    "itsk_fused_pass": (ctypes.c_int, [c_dp, c_i64, c_i64, c_i64, c_dp, c_dp, c_dp, c_dp, c_dp, c_dp,
                                       c_dp, c_i64, c_dp]),
    "itsk_fused_pass_scaled": (ctypes.c_int, [c_dp, c_i64, c_i64, c_i64, c_dp, ctypes.c_double, c_dp, c_dp,
                                              c_dp, c_dp, c_dp, c_dp, c_i64, c_dp]),
    "itsk_pass_workspace_init": (ctypes.c_int, [c_dp, c_i64, c_i64, c_dp]),
    "itsk_fused_pass_ex": (ctypes.c_int, [c_dp, c_i64, c_i64, c_i64, c_dp, ctypes.c_double, c_dp, c_dp,
                                          c_dp, c_dp, c_dp, c_dp, c_i64, ctypes.c_uint, c_dp]),
    "itsk_csr_plan_create": (ctypes.c_int, [c_dp, c_dp, c_dp, c_i64, c_i64, c_i64, c_dp, ctypes.POINTER(c_dp)]),
    "itsk_csr_plan_destroy": (None, [c_dp]),
    "itsk_csr_shape": (ctypes.c_int, [c_dp, ctypes.POINTER(c_i64), ctypes.POINTER(c_i64), ctypes.POINTER(c_i64)]),
    "itsk_csr_sketch": (ctypes.c_int, [c_dp, c_dp, c_dp, c_dp, c_i64, c_i64, c_dp, c_i64, c_dp]),
    "itsk_csr_pass": (ctypes.c_int, [c_dp, c_dp, ctypes.c_double, c_dp, c_dp, c_dp, c_dp, c_dp, c_dp]),
    "itsk_loop_workspace": (ctypes.c_int, [c_i64, c_i64, ctypes.POINTER(c_i64)]),
    "itsk_loop_begin": (ctypes.c_int, [ctypes.POINTER(LoopParams), c_dp]),
    "itsk_loop_begin_local": (ctypes.c_int, [ctypes.POINTER(LoopParams), c_dp]),
    "itsk_loop_begin_finish": (ctypes.c_int, [ctypes.POINTER(LoopParams), c_dp]),
    "itsk_loop_step_pre": (ctypes.c_int, [ctypes.POINTER(LoopParams), c_dp]),
    "itsk_loop_step_post": (ctypes.c_int, [ctypes.POINTER(LoopParams), c_dp]),
    "itsk_loop_graph_create": (ctypes.c_int, [ctypes.POINTER(LoopParams), c_dp, ctypes.POINTER(c_dp)]),
    "itsk_loop_graph_launch": (ctypes.c_int, [c_dp, c_dp]),
    "itsk_loop_graph_destroy": (None, [c_dp]),
    "itsk_struct_size": (c_i64, [ctypes.c_int]),
    "itsk_loop_finish": (ctypes.c_int, [ctypes.POINTER(LoopParams), c_dp]),
    "itsk_flag_store": (ctypes.c_int, [c_dp, ctypes.c_uint64, c_dp]),
    "itsk_loop_result_ptr": (ctypes.c_int, [ctypes.POINTER(LoopParams), ctypes.POINTER(c_dp)]),
}

PASS_WS_READY = 1  # include/itsk_b200.h ITSK_PASS_WS_READY
LOOP_TAIL_SUMS = 1  # include/itsk_b200.h ITSK_LOOP_TAIL_SUMS

_lock = threading.Lock()
_lib = None


def load(path: str = LIB_PATH):
    """Load the shared library (no device needed) and bind every symbol."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ImportError(
                f"{path} is missing: build it with `python -m paper_2311_04362_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


_dev_checked: set[int] = set()


def lib_for_device(dev: int):
    lib = load()
    if dev not in _dev_checked:
        check(lib.itsk_device_check(dev))
        _dev_checked.add(dev)
    return lib


def check(status: int) -> None:
    if status == ITSK_OK:
        return
    msg = (_lib.itsk_last_error() or b"").decode(errors="replace") if _lib else ""
    if status == ITSK_EINVAL:
        raise ValueError(msg)
    if status == ITSK_ESINGULAR:
        raise SingularMatrixError(msg or "zero diagonal entry in triangular factor")
    if status == ITSK_ENODEV:
        raise RuntimeError(f"no sm_100 B200 device: {msg}")
    raise ItskCudaError(msg)


def exported_symbols() -> list[str]:
    return list(_SIGS)
