"""ctypes binding of libpfw.so (include/pfw.h).

This is the only door to the CUDA path.  There is no CPU fallback: if the
library is missing or no CUDA device is visible, every classification entry
point raises ``NativeUnavailable`` loudly.
"""

from __future__ import annotations

import ctypes
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PFW_LIB") or os.path.join(PKG, "libpfw.so")  # PFW_LIB: experiment builds

NO_MATCH = 0x7FFFFFFF  # PFW_NO_MATCH
HOST_FIRST_MINUS1 = 1  # PFW_HOST_FIRST_MINUS1
PFW_OK, PFW_ERR_INVALID, PFW_ERR_CUDA, PFW_ERR_NOMEM, PFW_ERR_GENERATION = range(5)


class NativeUnavailable(RuntimeError):
    """libpfw.so is not built or no CUDA device is visible."""


class NativeError(RuntimeError):
    """A CUDA / library failure reported through the C-ABI."""


_lib = None
_lock = threading.Lock()

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int
_U64 = ctypes.c_uint64
_U32 = ctypes.c_uint32

_SIGS = {
    "pfw_last_error": (ctypes.c_char_p, []),
    "pfw_version": (ctypes.c_char_p, []),
    "pfw_device_count": (_I32, []),
    "pfw_ruleset_create": (_I32, [_I32, _I64] + [_P] * 10 + [ctypes.POINTER(_P)]),
    "pfw_ruleset_destroy": (_I32, [_P]),
    "pfw_ruleset_size": (_I64, [_P]),
    "pfw_ruleset_matchset_bytes": (_I64, [_P]),
    "pfw_ruleset_set_shard": (_I32, [_P, _I64, _I64]),
    "pfw_ruleset_info": (_I32, [_P, ctypes.c_char_p, ctypes.POINTER(_I64)]),
    "pfw_ruleset_device": (_I32, [_P]),
    "pfw_pack_packets_host": (_I32, [_I64, _P, _P, _P, _P, _P, _P]),
    "pfw_scan_range": (_I32, [_P, _I64, _I64, _P, _I64, _P, _P, _P, _P, _P]),
    "pfw_scan_range_columns": (_I32, [_P, _I64, _I64, _P, _P, _P, _P, _P, _I64, _P, _P, _P, _P, _P]),
    "pfw_scan_partition_accumulate": (_I32, [_P, _I64, _I64, _P, _I64, _P, _P, _P, _P]),
    "pfw_accumulator_init": (_I32, [_I64, _P, _P, _P]),
    "pfw_scan_partitions": (_I32, [_P, _I64, _P, _I64, _P, _P, _P, _P]),
    "pfw_scan_fused_min": (_I32, [_P, _I64, _I64, _P, _I64, _P, _P, _P, _I32, _I32, _P, _P]),
    "pfw_peer_enable": (_I32, [_I32, _I32]),
    "pfw_ipc_handle_size": (_I32, []),
    "pfw_ipc_get_handle": (_I32, [_P, _P, ctypes.POINTER(_U64)]),
    "pfw_ipc_open": (_I32, [_I32, _P, ctypes.POINTER(_P)]),
    "pfw_ipc_close": (_I32, [_I32, _P]),
    "pfw_verdicts": (_I32, [_P, _P, _I64, _P, _P]),
    "pfw_combine_min": (_I32, [_P, _I64, _I64, _P, _P]),
    "pfw_classify_host": (_I32, [_P, _P, _I64, _P, _P, _P, _I64]),
    "pfw_classify_host_columns": (_I32, [_P, _P, _P, _P, _P, _P, _I64, _P, _P, _P, _I64]),
    "pfw_classify_host_ex": (_I32, [_P, _P, _P, _P, _P, _P, _P, _I64, _P, _P, _P, _I64, _U32]),
    "pfw_classify_host_partitions": (_I32, [_P, _I64, _P, _P, _P, _P, _P, _P, _I64, _P, _P, _P, _P, _I64, _U32]),
    "pfw_generate_traffic": (_I32, [_I32, _U64, _I64, _I32, _U32, _I32, _U32, _I32, _I32, _I32,
                                    _I32, _I32, _P, _P]),
    "pfw_generate_traffic_at": (_I32, [_I32, _U64, _I64, _I64, _I32, _U32, _I32, _U32, _I32, _I32, _I32,
                                       _I32, _I32, _P, _P]),
    "pfw_io_last_error": (ctypes.c_char_p, []),
    "pfw_parse_rules": (_I32, [_P, _I64, _I64] + [_P] * 10 + [ctypes.POINTER(_I64)]),
    "pfw_parse_traffic": (_I32, [_P, _I64, _I64, _P, _P, ctypes.POINTER(_I64)]),
    "pfw_format_results": (_I32, [_P, _P, _P, _I64, _P, _I64, ctypes.POINTER(_I64)]),
    "pfw_launch_count": (_I64, []),
    "pfw_probe_l2_lines": (_I32, [_P, _I64, _I32, _I32, _I32, _P]),
    "pfw_read_counter": (_I32, [ctypes.c_char_p, ctypes.POINTER(_I64)]),
    "pfw_set_tuning": (_I32, [ctypes.c_char_p, _I64]),
}

EXPORTS = tuple(_SIGS)


def load(path: str = LIB_PATH):
    """Load libpfw.so (does not require a GPU)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise NativeUnavailable(
                    f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
            lib = ctypes.CDLL(path)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def lib():
    return load()


def last_error() -> str:
    return (lib().pfw_last_error() or b"").decode(errors="replace")


def check(rc: int, what: str) -> None:
    if rc == PFW_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == PFW_ERR_INVALID:
        raise ValueError(msg)
    raise NativeError(msg)


def device_count() -> int:
    return int(lib().pfw_device_count())


def require_device() -> None:
    if device_count() < 1:
        raise NativeUnavailable("no CUDA device visible: the packet-filter path runs only on the GPU "
                                "(there is no CPU fallback)")


def launch_count() -> int:
    return int(lib().pfw_launch_count())


def ruleset_info(handle, key: str) -> int:
    """pfw_ruleset_info: matchset_bytes / compressed / summaries / index_base."""
    v = ctypes.c_int64(0)
    check(lib().pfw_ruleset_info(handle, key.encode(), ctypes.byref(v)), f"pfw_ruleset_info({key})")
    return int(v.value)


def read_counter(name: str) -> int:
    """Read and reset an instrumentation counter (pfw_read_counter)."""
    v = ctypes.c_int64(0)
    check(lib().pfw_read_counter(name.encode(), ctypes.byref(v)), f"pfw_read_counter({name})")
    return int(v.value)


def set_tuning(key: str, value: int) -> None:
    check(lib().pfw_set_tuning(key.encode(), int(value)), f"pfw_set_tuning({key})")


def version() -> str:
    return lib().pfw_version().decode()
