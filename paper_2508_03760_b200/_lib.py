"""ctypes binding of the C ABI in include/fc2.h (libfc2.so, built for sm_100a).

This is the binding a maintainer of the reference would add:
plain pointers, sizes and int status codes.  There is no CPU fallback: if the
library or a CUDA device is missing, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import CodeRangeError, ConfigError, DataError, DecodeFormatError, NotApplicableError

_HERE = os.path.dirname(os.path.abspath(__file__))
# FC2_LIB: alternate build of the same library (kernel-variant experiments)
LIB_PATH = os.environ.get("FC2_LIB") or os.path.join(_HERE, "libfc2.so")

FC2_OK = 0
FC2_ECONFIG = -1
FC2_EDATA = -2
FC2_EFORMAT = -3
FC2_ENOTAPPLICABLE = -4
FC2_ECUDA = -5

ERR_NONFINITE = 1
ERR_SPIKE_INDEX = 2
ERR_LOG2_TIE = 4
ERR_TIMEOUT = 8
ERR_CODE_RANGE = 16
ERR_NEGATIVE = 32
ERR_EXPERT_RANGE = 64

BF16, F32, F64 = 0, 1, 2


class Config(ctypes.Structure):
    _fields_ = [
        ("bitwidth", ctypes.c_int32),
        ("group_size", ctypes.c_int32),
        ("scheme", ctypes.c_int32),
        ("scale_encoding", ctypes.c_int32),
        ("theta", ctypes.c_int32),
    ]


_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_PP = ctypes.POINTER(ctypes.c_void_p)
_PI64 = ctypes.POINTER(ctypes.c_int64)
_PCFG = ctypes.POINTER(Config)

# name -> (restype, argtypes); the exported surface of include/fc2.h
SIGNATURES = {
    "fc2_check_config": (_I32, [_PCFG]),
    "fc2_footprint": (_I32, [_PCFG, _I64, _PI64]),
    "fc2_plane_offset": (_I64, [_PCFG, _I64, _I32]),
    "fc2_meta_offset": (_I64, [_PCFG, _I64]),
    "fc2_set_intlog_table": (_I32, [_I32, ctypes.POINTER(ctypes.c_double)]),
    "fc2_encode": (_I32, [_PCFG, _P, _I32, _I64, _I64, _P, _P, _P]),
    "fc2_encode_batch": (_I32, [_PCFG, _I32, _I32, _PP, _PI64, _PI64, _PP, _P, _P]),
    "fc2_decode": (_I32, [_PCFG, _P, _I64, _P, _I32, _I64, _P, _P]),
    "fc2_decode_batch": (_I32, [_PCFG, _I32, _I32, _PP, _PI64, _PP, _PI64, _P, _P]),
    "fc2_encode_host": (_I32, [_PCFG, _P, _I32, _I64, _P, _P, _P, _I64, _P, _P]),
    "fc2_decode_host": (_I32, [_PCFG, _P, _I64, _P, _P, _I32, _P, _I64, _P, _P]),
    "fc2_roundtrip_host": (_I32, [_PCFG, _P, _I32, _I64, _P, _P, _P, _I32, _P, _P, _I64, _P, _P]),
    "fc2_reduce_requant": (_I32, [_PCFG, _I32, _PP, _I64, _I32, _PP, _P, _P]),
    "fc2_reduce_requant_batch": (_I32, [_PCFG, _I32, _PP, _I64, _I32, _I64, _I32, _PP, _I64, _P, _P]),
    "fc2_allreduce_oneshot": (_I32, [_P, _PCFG, _P, _I32, _P, _I32, _I64, _I64, _I64, _P, ctypes.c_double, _P]),
    "fc2_allreduce_fused": (_I32, [_P, _PCFG, _P, _I32, _P, _I32, _I64, _I64, _I64, _P, ctypes.c_double, _P]),
    "fc2_gather_decode": (_I32, [_PCFG, _I32, _PP, _I64, _P, _I32, _I64, _P, _P]),
    "fc2_pack_codes": (_I32, [_P, _I64, _I32, _P, _P, _P]),
    "fc2_unpack_codes": (_I32, [_P, _I64, _I32, _P, _P]),
    "fc2_f32_to_bf16_bits": (_I32, [_P, _I64, _P, _P]),
    "fc2_bf16_bits_to_f32": (_I32, [_P, _I64, _P, _P]),
    "fc2_group_encode_raw": (_I32, [_P, _I64, _I32, _I32, _P, _P, _P, _P, _P]),
    "fc2_group_decode_raw": (_I32, [_P, _I64, ctypes.c_double, ctypes.c_double, _P, _P]),
    "fc2_scale_to_int": (_I32, [_P, _I64, _I32, _P, _P, _P]),
    "fc2_int_to_scale": (_I32, [_P, _I64, _I32, _P, _P]),
    "fc2_comm_handle_bytes": (_I32, []),
    "fc2_comm_create": (_I32, [_I32, _I32, _I64, ctypes.POINTER(ctypes.c_void_p), _P]),
    "fc2_comm_open_peers": (_I32, [_P, _P]),
    "fc2_comm_destroy": (_I32, [_P]),
    "fc2_comm_buffer": (_P, [_P, _I32]),
    "fc2_comm_barrier": (_I32, [_P, _P, ctypes.c_double, _P]),
    "fc2_allreduce_2step": (_I32, [_P, _PCFG, _P, _I32, _P, _I32, _I64, _I64, _P, ctypes.c_double, _P]),
    "fc2_allreduce_2step_pipe": (_I32, [_P, _PCFG, _P, _I32, _P, _I32, _I64, _I32, _I64, _I64, _I64, _P,
                                        ctypes.c_double, _P]),
    "fc2_a2a_q": (_I32, [_P, _PCFG, _P, _I32, _PI64, _P, _I32, _I64, _I64, _P, ctypes.c_double, _P]),
    "fc2_copy_check": (_I32, [_P, _I32, _P, _I32, _I64, _P, _P]),
    "fc2_copy_bytes": (_I32, [_P, _P, _I64, _I32, _P]),
    "fc2_encode_batch_rows": (_I32, [_PCFG, _I32, _I32, _P, _PP, _I64, _PI64, _PI64, _PP, _P, _P]),
    "fc2_moe_route": (_I32, [_P, _I32, _I64, _I32, _I32, _I32, _P, _P, _P, _P, _P]),
    "fc2_gather_rows_check": (_I32, [_P, _I32, _P, _I64, _I64, _P, _I32, _P, _P]),
    "fc2_moe_combine_sum": (_I32, [_I32, _PP, _P, _P, _P, _I64, _I64, _P, _I32, _P, _P]),
    "fc2_moe_combine_q": (_I32, [_PCFG, _I32, _I32, _PP, _PI64, _P, _I32, _P, _I64, _I64, _P, _I32, _P, _P]),
    "fc2_comm_allgather_i32": (_I32, [_P, _P, _I32, _P, _P, ctypes.c_double, _P]),
    "fc2_moe_dispatch": (_I32, [_P, _PCFG, _P, _I32, _I64, _I64, _P, _PI64, _P, _I32, _I64, _I64, _P,
                                ctypes.c_double, _P]),
    "fc2_moe_combine": (_I32, [_P, _PCFG, _P, _I32, _I64, _I64, _PI64, _P, _P, _P, _I32, _I64, _I64, _P,
                               ctypes.c_double, _P]),
    "fc2_last_error": (ctypes.c_char_p, []),
    "fc2_launch_count": (_I64, []),
    "fc2_version": (_I32, []),
}

_lock = threading.Lock()
_lib = None


def load(path: str = LIB_PATH):
    """Load libfc2.so (no CUDA calls happen at load time)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(
                f"{path} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback"
            )
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def lib():
    return _lib if _lib is not None else load()


def check(rc: int) -> None:
    """Map a C status code onto the reference's exception types (errors.py:4-21)."""
    if rc == FC2_OK:
        return
    msg = lib().fc2_last_error().decode(errors="replace")
    if rc == FC2_ECONFIG:
        raise ConfigError(msg)
    if rc == FC2_EDATA:
        raise DataError(msg)
    if rc == FC2_EFORMAT:
        raise DecodeFormatError(msg)
    if rc == FC2_ENOTAPPLICABLE:
        raise NotApplicableError(msg)
    raise RuntimeError(f"fc2 CUDA failure: {msg}")


def raise_dev_err(bits: int, what: str = "") -> None:
    """Raise for a device error word (dev_err) the way the reference would."""
    if bits & ERR_NONFINITE:
        raise DataError(f"{what}input contains non-finite values")
    if bits & ERR_NEGATIVE:
        raise DataError(f"{what}scale must be non-negative")
    if bits & ERR_CODE_RANGE:
        raise CodeRangeError(f"{what}codes out of range")
    if bits & ERR_SPIKE_INDEX:
        raise DecodeFormatError(f"{what}spike index out of range for group size")
    if bits & ERR_EXPERT_RANGE:
        raise ConfigError(f"{what}expert id out of range")
    if bits & ERR_TIMEOUT:
        raise RuntimeError(f"{what}cross-rank wait timed out")


def ptr_array(ptrs):
    arr = (ctypes.c_void_p * max(1, len(ptrs)))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr


def i64_array(vals):
    arr = (ctypes.c_int64 * max(1, len(vals)))()
    for i, v in enumerate(vals):
        arr[i] = int(v)
    return arr
