"""ctypes binding of the C-ABI in include/hg_b200.h (libhg_b200.so).

The library is built in-tree (`make`, or `__graft_entry__.build()`). There is
no CPU fallback: if the shared library is missing, or no sm_100 device is
present, every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
# HG_B200_LIB: an alternate build of the same C-ABI (A/B tuning runs only)
LIB_PATH = os.environ.get("HG_B200_LIB") or os.path.join(HERE, "libhg_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "hg_b200.h")

HG_OK, HG_EINVAL, HG_ERANGE, HG_EOVERFLOW, HG_ENOMEM, HG_ECUDA, HG_ENCCL, HG_EUNSUPPORTED, HG_EIO = range(9)
HASH_MIX64, HASH_IDENTITY = 0, 1
BUILD_SIMPLE, BUILD_BINNED = 1, 2


class hg_build_config(C.Structure):
    _fields_ = [
        ("load_factor", C.c_double),
        ("bin_count", C.c_uint64),
        ("hash_seed", C.c_uint64),
        ("vertex_count", C.c_uint64),
        ("variant", C.c_int32),
        ("hash_kind", C.c_int32),
        ("stable", C.c_int32),
        ("aggregate", C.c_int32),
        ("partition_vertices", C.c_uint64),
        ("global_vertices", C.c_uint64),
        ("vertex_base", C.c_uint64),
    ]


class hg_table_info(C.Structure):
    _fields_ = [
        ("num_vertices", C.c_uint64),
        ("num_edges", C.c_uint64),
        ("hash_seed", C.c_uint64),
        ("load_factor", C.c_double),
        ("key_width", C.c_int32),
        ("val_width", C.c_int32),
        ("off_width", C.c_int32),
        ("hash_kind", C.c_int32),
    ]


class hg_probe_options(C.Structure):
    _fields_ = [
        ("materialize", C.c_int32),
        ("pair_width", C.c_int32),
        ("pair_cap", C.c_uint64),
        ("pairs", C.c_void_p),
        ("counts", C.c_void_p),
        ("device_result", C.c_void_p),
        ("method", C.c_int32),
        ("flags", C.c_int32),
        ("hash_seed", C.c_uint64),
        ("hash_kind", C.c_int32),
        ("reserved", C.c_int32),
    ]


class hg_probe_result(C.Structure):
    _fields_ = [
        ("match_count", C.c_uint64),
        ("key_comparisons", C.c_uint64),
        ("pairs_written", C.c_uint64),
        ("truncated", C.c_int32),
    ]


class hg_kernel_time(C.Structure):
    _fields_ = [("name", C.c_char * 48), ("launches", C.c_uint64), ("total_ms", C.c_double)]


class HashGraphError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[hg status {status}] {msg}")
        self.status = status


_vp = C.c_void_p
_u64 = C.c_uint64
_i32 = C.c_int32

# name -> (restype, argtypes); must cover every function declared in hg_b200.h
SIGNATURES = {
    "hg_abi_version": (_i32, []),
    "hg_last_error": (C.c_char_p, []),
    "hg_build_config_init": (None, [C.POINTER(hg_build_config)]),
    "hg_probe_options_init": (None, [C.POINTER(hg_probe_options)]),
    "hg_derived_vertex_count": (_i32, [_u64, C.c_double, C.POINTER(_u64)]),
    "hg_hash_to_vertex": (_u64, [_u64, _u64, _u64]),
    "hg_build": (_i32, [_vp, _i32, _vp, _i32, _u64, C.POINTER(hg_build_config), _vp,
                        C.POINTER(_vp)]),
    "hg_table_get_info": (_i32, [_vp, C.POINTER(hg_table_info)]),
    "hg_table_device_arrays": (_i32, [_vp, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp)]),
    "hg_table_export": (_i32, [_vp, _vp, _vp, _vp, _vp]),
    "hg_table_destroy": (_i32, [_vp, _vp]),
    "hg_table_import": (_i32, [_vp, _vp, _vp, _u64, _u64, _u64, C.c_double, _i32, _vp,
                               C.POINTER(_vp)]),
    "hg_probe": (_i32, [_vp, _vp, _i32, _u64, C.POINTER(hg_probe_options),
                        C.POINTER(hg_probe_result), _vp]),
    "hg_probe_new_prepared": (_i32, [_vp, _vp, C.POINTER(hg_probe_options),
                                     C.POINTER(hg_probe_result), _vp]),
    "hg_probe_new": (_i32, [_vp, _u64, _vp, _u64, _i32, C.POINTER(hg_build_config),
                            C.POINTER(hg_probe_options), C.POINTER(hg_probe_result), _vp]),
    "hg_count_instances": (_i32, [_vp, _u64, C.POINTER(_u64), _vp]),
    "hg_validate": (_i32, [_vp, _vp, _u64, C.POINTER(_i32), _vp]),
    "hg_route_records": (_i32, [_vp, _i32, _vp, _i32, _u64, _u64, _u64, _i32, _u64, C.c_uint32,
                                _vp, _vp, _vp]),
    "hg_route_pairs": (_i32, [_vp, _vp, _i32, _u64, _u64, C.c_uint32, _vp, _vp, _vp]),
    "hg_build_records": (_i32, [_vp, _i32, _i32, _u64, C.POINTER(hg_build_config), _vp,
                                C.POINTER(_vp)]),
    "hg_count_instances_hasher": (_i32, [_vp, _u64, _i32, _u64, C.POINTER(_u64), _vp]),
    "hg_validate_hasher": (_i32, [_vp, _vp, _u64, _i32, _u64, C.POINTER(_i32), _vp]),
    "hg_generate": (_i32, [_vp, _i32, _u64, _i32, _u64, _u64, C.c_double, _vp, _u64, _vp]),
    "hg_shard_range": (_i32, [_u64, C.c_uint32, C.c_uint32, C.POINTER(_u64), C.POINTER(_u64)]),
    "hg_route": (_i32, [_vp, _i32, _vp, _i32, _u64, _u64, _u64, _i32, _u64, C.c_uint32, _vp, _vp,
                        _vp, _vp]),
    "hg_keys_file_count": (_i32, [C.c_char_p, C.POINTER(_u64)]),
    "hg_keys_read": (_i32, [C.c_char_p, _vp, _i32, _u64, C.POINTER(_u64), _vp]),
    "hg_keys_write": (_i32, [C.c_char_p, _vp, _i32, _u64, _vp]),
    "hg_profiler_enable": (None, [_i32]),
    "hg_profiler_collect": (_i32, [C.POINTER(hg_kernel_time), _i32]),
}

_LIB = None


def header_functions() -> list[str]:
    """Every function name declared in include/hg_b200.h."""
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hg_[a-z0-9_]+)\s*\(", text)) - {"hg_status"})


def lib():
    """Loads libhg_b200.so (fails loudly when it has not been built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(`make` or `python -c 'import __graft_entry__ as g; g.build()'`). "
                "There is no CPU fallback.")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def check(status: int) -> None:
    if status != HG_OK:
        msg = lib().hg_last_error().decode(errors="replace")
        raise HashGraphError(status, msg)


def profiler_enable(on: bool) -> None:
    lib().hg_profiler_enable(1 if on else 0)


def profiler_collect() -> dict:
    """{kernel name: (launches, total_ms)} for launches since the last collect."""
    buf = (hg_kernel_time * 64)()
    n = lib().hg_profiler_collect(buf, 64)
    return {buf[i].name.decode(): (int(buf[i].launches), float(buf[i].total_ms))
            for i in range(min(n, 64))}
