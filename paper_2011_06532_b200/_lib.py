"""ctypes binding of the C ABI declared in include/ttb.h (library _ttb.so).

The product path has no CPU fallback: if the shared library or a CUDA device
is missing, every compute entry point raises (CapabilityError / OSError).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import (CapabilityError, CapacityError, ContractError, DeadlockError, NumericError,
                     ShapeError, TTError)

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("TTB_LIB") or os.path.join(_HERE, "_ttb.so")

TTB_OK = 0
_ERRMAP = {
    1: ShapeError,
    2: ContractError,
    3: NumericError,
    4: CapacityError,
    5: TTError,        # CUDA runtime failure
    6: TTError,        # NCCL failure
    7: CapabilityError,
    8: DeadlockError,
}

_P = C.c_void_p
_I64 = C.c_int64
_PI64 = C.POINTER(C.c_int64)
_PD = C.POINTER(C.c_double)
_PP = C.POINTER(C.c_void_p)

# name -> (restype, argtypes); every symbol include/ttb.h declares
SIGNATURES = {
    "ttb_last_error": (C.c_char_p, []),
    "ttb_abi_version": (C.c_int, []),
    "ttb_launch_counter": (C.c_longlong, []),
    "ttb_comm_stats": (C.c_int, [C.POINTER(C.c_longlong)]),
    "ttb_ctx_create": (C.c_int, [C.c_int, _P, _PP]),
    "ttb_ctx_destroy": (C.c_int, [_P]),
    "ttb_ctx_set_stream": (C.c_int, [_P, _P]),
    "ttb_ctx_trim": (C.c_int, [_P]),
    "ttb_comm_unique_id": (C.c_int, [_P]),
    "ttb_ctx_init_comm": (C.c_int, [_P, C.c_int, C.c_int, _P]),
    "ttb_group_create": (C.c_int, [C.c_int, _PP]),
    "ttb_group_destroy": (C.c_int, [_P]),
    "ttb_group_abort": (C.c_int, [_P]),
    "ttb_ctx_join_group": (C.c_int, [_P, _P, C.c_int]),
    "ttb_scale": (C.c_int, [_P, _I64, _P, C.c_double, _P]),
    "ttb_add": (C.c_int, [_P, C.c_int, C.c_int, _PI64, _PI64, _PP, _PD, _PP]),
    "ttb_hadamard": (C.c_int, [_P, C.c_int, _PI64, _PI64, _PI64, _PP, _PP, _PP]),
    "ttb_fill_random": (C.c_int, [_P, C.POINTER(C.c_uint32), C.c_int, C.c_int, _PI64, _PI64, _PI64, _PI64,
                                  _PI64, _PP]),
    "ttb_inner": (C.c_int, [_P, C.c_int, _PI64, _PI64, _PI64, _PP, _PP, _PD]),
    "ttb_sumsq": (C.c_int, [_P, _I64, _P, _PD]),
    "ttb_norm_sym": (C.c_int, [_P, C.c_int, _PI64, _PI64, _PP, _PD, C.POINTER(C.c_int)]),
    "ttb_pivoted_cholesky": (C.c_int, [_P, C.c_int, _P, _P, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                       C.POINTER(C.c_int)]),
    "ttb_orthonormalize": (C.c_int, [_P, C.c_int, C.c_int, _PI64, _PI64, _PP, _PP]),
    "ttb_norm_ortho": (C.c_int, [_P, C.c_int, _PI64, _PI64, _PP, _PD]),
    "ttb_round": (C.c_int, [_P, C.c_int, C.c_double, _I64, C.c_int, _PI64, _PI64, _PP, _PP, _PI64, _PD]),
    "ttb_round_hadamard": (C.c_int, [_P, C.c_int, C.c_double, _I64, C.c_int, _PI64, _PI64, _PI64, _PP, _PP, _PP,
                                     _PI64, _PD]),
    "ttb_round_host": (C.c_int, [_P, C.c_int, C.c_double, _I64, C.c_int, _PI64, _PI64, _PP, _PP, _PI64, _PD]),
    "ttb_tsqr_factor": (C.c_int, [_P, _I64, _I64, _I64, C.c_int, _P, _PP, _P]),
    "ttb_tsqr_apply": (C.c_int, [_P, _P, _I64, _P, _P]),
    "ttb_tsqr_free": (C.c_int, [_P, _P]),
    "ttb_truncated_svd": (C.c_int, [_P, _I64, _I64, _P, C.c_double, _I64, _P, _P, _P, _PI64, _PD,
                                    C.POINTER(C.c_int)]),
    "ttb_mode2_spmm": (C.c_int, [_P, _I64, _I64, _I64, _P, _P, _P, _I64, _P, _P, _P, _I64, _I64, _I64, _I64]),
    "ttb_mode2_spmm_sum": (C.c_int, [_P, C.c_int, C.c_int, _I64, _I64, _I64, _PP, _PP, _PP, _I64, _P, _PP, _P]),
    "ttb_gather_slices": (C.c_int, [_P, _I64, _I64, _I64, _P, _I64, _P, _P]),
    "ttb_exchange": (C.c_int, [_P, C.c_int, C.POINTER(C.c_int), _PP, _PI64, _PP, _PI64]),
    "ttb_read_slabs": (C.c_int, [_P, C.c_char_p, _I64, C.c_int, _PI64, _PI64, _PI64, _PI64, _PP]),
    "ttb_write_slabs": (C.c_int, [_P, C.c_char_p, _I64, C.c_int, _PI64, _PI64, _PI64, _PI64, _PP]),
    "ttb_fp64_peak": (C.c_int, [_P, _PD, _PD]),
    "ttb_prof_enable": (C.c_int, [C.c_int]),
    "ttb_prof_dump": (C.c_int, [C.c_char_p, C.c_longlong]),
}

_lib = None
_lock = threading.Lock()


def load():
    """Load _ttb.so (raises if it has not been built)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(SO_PATH):
            raise CapabilityError(
                f"CUDA library {SO_PATH} is missing; build it with "
                "`python -m paper_2011_06532_b200.build` (there is no CPU fallback)")
        lib = C.CDLL(SO_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc):
    if rc != TTB_OK:
        msg = load().ttb_last_error().decode(errors="replace")
        raise _ERRMAP.get(rc, TTError)(msg)


def i64_array(vals):
    vals = [int(v) for v in vals]
    return (C.c_int64 * max(1, len(vals)))(*vals)


def ptr_array(ptrs):
    ptrs = [int(p) for p in ptrs]
    return (C.c_void_p * max(1, len(ptrs)))(*ptrs)


def launch_counter():
    return int(load().ttb_launch_counter())


def comm_stats():
    """(allgathers, allgather doubles, allreduces + p2p transfers, their doubles)."""
    buf = (C.c_longlong * 4)()
    check(load().ttb_comm_stats(buf))
    return tuple(int(v) for v in buf)


def prof_enable(on=True):
    check(load().ttb_prof_enable(1 if on else 0))


def prof_dump():
    """{kernel class: (launches, total_ms)} recorded since the last dump."""
    buf = C.create_string_buffer(1 << 16)
    check(load().ttb_prof_dump(buf, len(buf)))
    out = {}
    for line in buf.value.decode().splitlines():
        name, cnt, ms = line.split()
        out[name] = (int(cnt), float(ms))
    return out


def fp64_peak(stream=0):
    a, b = C.c_double(), C.c_double()
    check(load().ttb_fp64_peak(C.c_void_p(stream), C.byref(a), C.byref(b)))
    return float(a.value), float(b.value)
