"""ctypes binding of the C-ABI in include/fsb_b200.h (libfsb_b200.so).

This is the Python-side counterpart of the binding a maintainer would add on
the reference side.  The library is built in-tree by
_build.py; there is no fallback -- if it cannot be loaded the import fails.
"""
from __future__ import annotations

import ctypes
import os

from . import _build

FSB_OK = 0
FSB_ERR_INVALID_CONFIG = 1
FSB_ERR_INVALID_ARGUMENT = 2
FSB_ERR_CUDA = 3
FSB_ERR_NCCL = 4
FSB_ERR_OUT_OF_MEMORY = 5
FSB_ERR_UNSUPPORTED = 6

STRATEGY_AUTO = 0
STRATEGY_STREAM = 1
STRATEGY_PERSISTENT = 2
STRATEGY_GRID = 3

FLAG_NO_ALTERNATE = 0x1
FLAG_FORCE_NCCL = 0x2
FLAG_NO_BULK = 0x4
FLAG_FORCE_BULK = 0x8
FLAG_NO_PDL = 0x10
FLAG_PEER_EXCHANGE = 0x20
FLAG_CHECKED = 0x40
FLAG_STATIC_TILES = 0x80
FLAG_DYNAMIC_TILES = 0x100
FLAG_FLAT_GRID = 0x200
FLAG_HOST_EXCHANGE = 0x400
FLAG_L2_GRID = 0x800
FLAG_WS_TILES = 0x1000
FLAG_LAST_CTA_FOLD = 0x2000


class fsb_sim_config(ctypes.Structure):
    _fields_ = [
        ("num_fish", ctypes.c_uint64),
        ("pond_size", ctypes.c_double),
        ("weight_scale", ctypes.c_double),
        ("num_steps", ctypes.c_uint64),
        ("seed", ctypes.c_uint64),
        ("step_base", ctypes.c_double),
    ]


class fsb_timing(ctypes.Structure):
    _fields_ = [
        ("seconds_total", ctypes.c_double),
        ("seconds_move", ctypes.c_double),
        ("seconds_eat", ctypes.c_double),
        ("seconds_loop", ctypes.c_double),
    ]


class fsb_engine_options(ctypes.Structure):
    _fields_ = [
        ("device", ctypes.c_int),
        ("rank", ctypes.c_int),
        ("world_size", ctypes.c_int),
        ("nccl_unique_id", ctypes.c_void_p),
        ("strategy", ctypes.c_int),
        ("flags", ctypes.c_uint),
    ]


# (name, restype, argtypes) for every symbol include/fsb_b200.h declares.
_vp, _u64, _int, _dbl, _sz = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_double, ctypes.c_size_t
_P = ctypes.POINTER
SIGNATURES = [
    ("fsb_abi_version", _int, []),
    ("fsb_last_error", ctypes.c_char_p, []),
    ("fsb_config_validate", _int, [_P(fsb_sim_config)]),
    ("fsb_shard_range", _int, [_u64, _int, _int, _P(_u64), _P(_u64)]),
    ("fsb_checksum_update", _u64, [_u64, _vp, _u64]),
    ("fsb_device_count", _int, [_P(_int)]),
    ("fsb_host_alloc", _int, [_P(_vp), _sz]),
    ("fsb_host_free", _int, [_vp]),
    ("fsb_nccl_unique_id", _int, [_vp, _sz]),
    ("fsb_engine_create", _int, [_P(fsb_sim_config), _P(fsb_engine_options), _P(_vp)]),
    ("fsb_engine_destroy", _int, [_vp]),
    ("fsb_engine_shard", _int, [_vp, _P(_u64), _P(_u64)]),
    ("fsb_engine_init", _int, [_vp]),
    ("fsb_engine_upload", _int, [_vp, _vp, _u64]),
    ("fsb_engine_download", _int, [_vp, _vp, _u64]),
    ("fsb_engine_move", _int, [_vp, _u64, _P(_dbl)]),
    ("fsb_engine_eat", _int, [_vp, _P(_dbl), _P(_dbl)]),
    ("fsb_engine_run", _int, [_vp, _u64, _u64, _vp, _vp, _P(fsb_timing)]),
    ("fsb_engine_simulate", _int, [_vp, _vp, _vp, _P(fsb_timing)]),
    ("fsb_engine_barycentre", _int, [_vp, _vp, _vp]),
    ("fsb_engine_gather", _int, [_vp, _vp, _u64, _vp]),
    ("fsb_engine_checksum", _int, [_vp, _u64, _P(_u64)]),
    ("fsb_engine_synchronize", _int, [_vp]),
    ("fsb_engine_stream", _int, [_vp, _P(_vp)]),
    ("fsb_engine_time_step_kernels", _int, [_vp, _u64, _u64, _vp]),
    ("fsb_engine_last_launches", _int, [_vp, _P(_u64)]),
    ("fsb_engine_last_strategy", _int, [_vp, _P(_int), _P(ctypes.c_char_p)]),
    ("fsb_engine_set_grid", _int, [_vp, _int]),
    ("fsb_engine_set_tile_groups", _int, [_vp, _int]),
    ("fsb_engine_grid", _int, [_vp, _P(_int), _P(_int)]),
    ("fsb_engine_partial", _int, [_vp, _vp]),
    ("fsb_engine_set_partials", _int, [_vp, _vp, _sz]),
    ("fsb_engine_peer_handle", _int, [_vp, _vp, _sz]),
    ("fsb_engine_peer_connect", _int, [_vp, _vp, _sz]),
    ("fsb_engine_peer_connect_local", _int, [_vp, _vp, ctypes.c_int]),
    ("fsb_selftest_fast_math", _int, [_int, _u64, _u64, _vp]),
]


ABI_VERSION = 2  # FSB_B200_ABI_VERSION


class FsbError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[fsb status {code}] {msg}")
        self.code = code


_lib = None


def _pin_nccl() -> None:
    """Point FSB_NCCL_LIB at the NCCL that torch links (the nvidia-nccl wheel),
    unless the caller chose one: the engine dlopens NCCL lazily, and a different
    libnccl.so.2 loaded first would shadow torch's by soname."""
    if os.environ.get("FSB_NCCL_LIB"):
        return
    try:
        import importlib.util

        spec = importlib.util.find_spec("nvidia.nccl")
        for d in (spec.submodule_search_locations if spec else None) or []:
            cand = os.path.join(d, "lib", "libnccl.so.2")
            if os.path.exists(cand):
                os.environ["FSB_NCCL_LIB"] = cand
                return
    except Exception:
        pass


def lib() -> ctypes.CDLL:
    """Load (building first if stale) libfsb_b200.so.  FSB_LIB may name a
    prebuilt variant of the same library (tools/variants.py A/B builds)."""
    global _lib
    if _lib is None:
        _pin_nccl()
        path = os.environ.get("FSB_LIB") or _build.build()
        L = ctypes.CDLL(path)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.fsb_abi_version() != ABI_VERSION:
            raise ImportError("libfsb_b200.so ABI mismatch")
        _lib = L
    return _lib


def lib_path() -> str:
    return os.path.abspath(os.environ.get("FSB_LIB") or _build.LIB)


def check(rc: int) -> None:
    if rc != FSB_OK:
        msg = lib().fsb_last_error().decode(errors="replace")
        if rc == FSB_ERR_INVALID_CONFIG:
            raise ValueError(msg)  # mirrors std::invalid_argument (sim.hpp:45-48)
        raise FsbError(rc, msg)
