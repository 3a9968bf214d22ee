"""ctypes binding of ``libsnpb200.so`` (C ABI declared in ``include/snpb200.h``).

The library is built in-tree by ``__graft_entry__.build()`` (or
``python -m paper_2408_04343_b200.build``).  Loading it never falls back to
anything: if the ``.so`` is missing or no CUDA device is visible, the engine
raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

LIB_NAME = "libsnpb200.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME

SNP_OK, SNP_ERR_NEGATIVE, SNP_ERR_BAD_ARG, SNP_ERR_CUDA, SNP_ERR_CAPACITY = range(5)
SNP_FMT_SPARSE, SNP_FMT_ELL, SNP_FMT_COMPRESSED = range(3)
SNP_VARIANT_AUTO, SNP_VARIANT_PULL, SNP_VARIANT_PUSH, SNP_VARIANT_TILED, SNP_VARIANT_TILED2, SNP_VARIANT_SMALL = range(6)
SNP_REC_CONFIGS, SNP_REC_DELAYS, SNP_REC_SPIKING, SNP_REC_DIGEST = 1, 2, 4, 8
SNP_RUNNING, SNP_HALT_STEP_LIMIT, SNP_HALT_NO_APPLICABLE, SNP_HALT_NEGATIVE, SNP_HALT_EXCHANGE = range(5)
SNP_IPC_HANDLE_BYTES = 64
STAT_NAMES = ("steps", "scanned", "fired", "sending", "edges", "rows", "open")

_i64p = ctypes.POINTER(ctypes.c_int64)
_u8p = ctypes.POINTER(ctypes.c_uint8)


class SystemDesc(ctypes.Structure):
    _fields_ = [
        ("format", ctypes.c_int32), ("variant", ctypes.c_int32),
        ("q", ctypes.c_int64), ("m", ctypes.c_int64),
        ("initial", _i64p), ("offsets", _i64p), ("threshold", _i64p), ("is_exact", _u8p),
        ("consumed", _i64p), ("produced", _i64p), ("delay", _i64p),
        ("adj_offsets", _i64p), ("adj_targets", _i64p),
        ("syn_target", _i64p), ("syn_rows", ctypes.c_int64),
        ("ell_target", _i64p), ("ell_amount", _i64p), ("ell_rows", ctypes.c_int64),
        ("sparse_data", _i64p),
        ("device", ctypes.c_int32), ("world", ctypes.c_int32), ("rank", ctypes.c_int32),
        ("x_pbits", ctypes.c_int32), ("x_pmax", ctypes.c_int64),
    ]


class RunOpts(ctypes.Structure):
    _fields_ = [
        ("max_steps", ctypes.c_int64), ("policy", ctypes.c_int32), ("record", ctypes.c_int32),
        ("seed", ctypes.c_uint64), ("chunk", ctypes.c_int64), ("use_graph", ctypes.c_int32),
        ("collect_stats", ctypes.c_int32),
    ]


class TraceOut(ctypes.Structure):
    _fields_ = [
        ("configs", _i64p), ("delays", _i64p), ("spiking", _i64p), ("cap", ctypes.c_int64),
        ("first_row_step", ctypes.c_int64), ("config_rows", ctypes.c_int64),
        ("spiking_rows", ctypes.c_int64),
        ("config_digests", ctypes.c_void_p), ("delay_digests", ctypes.c_void_p),
        ("spiking_digests", ctypes.c_void_p),
    ]


class Result(ctypes.Structure):
    _fields_ = [
        ("steps", ctypes.c_int64), ("halt", ctypes.c_int32), ("error", ctypes.c_int32),
        ("negative_neuron", ctypes.c_int64), ("negative_value", ctypes.c_int64),
        ("stats", ctypes.c_uint64 * 7), ("kernel_launches", ctypes.c_int64),
    ]

    def stats_dict(self) -> dict:
        return {name: int(self.stats[i]) for i, name in enumerate(STAT_NAMES)}


PUSH_KERNELS = {0: "none", 1: "unfused", 2: "atomic", 3: "binned"}


class EngineInfo(ctypes.Structure):
    _fields_ = [
        ("q", ctypes.c_int64), ("m", ctypes.c_int64), ("z", ctypes.c_int64),
        ("device_bytes", ctypes.c_int64), ("format", ctypes.c_int32), ("variant", ctypes.c_int32),
        ("p_mode", ctypes.c_int32), ("heavy_neurons", ctypes.c_int32),
        ("in_edges", ctypes.c_int64), ("p_common", ctypes.c_int64),
        ("tile", ctypes.c_int64), ("n_tiles", ctypes.c_int64),
        ("ring_stages", ctypes.c_int32), ("counter_bits", ctypes.c_int32), ("stage_bytes", ctypes.c_int64),
        ("push_kernel", ctypes.c_int32), ("push_tiles", ctypes.c_int32),
    ]


class Exchange(ctypes.Structure):
    _fields_ = [
        ("slot", ctypes.c_void_p * 3), ("slot_bytes", ctypes.c_int64), ("chunk_offset_bytes", ctypes.c_int64),
        ("chunk_bytes", ctypes.c_int64), ("lo", ctypes.c_int64), ("hi", ctypes.c_int64),
        ("neurons_per_rank", ctypes.c_int64), ("world", ctypes.c_int32), ("rank", ctypes.c_int32),
    ]


# (name, restype, argtypes) -- every symbol include/snpb200.h declares
_EngineP = ctypes.c_void_p
SIGNATURES = [
    ("snp_abi_version", ctypes.c_int, []),
    ("snp_last_error", ctypes.c_char_p, []),
    ("snp_device_count", ctypes.c_int, []),
    ("snp_engine_create", ctypes.c_int, [ctypes.POINTER(SystemDesc), ctypes.POINTER(ctypes.c_void_p)]),
    ("snp_engine_destroy", None, [_EngineP]),
    ("snp_engine_get_info", ctypes.c_int, [_EngineP, ctypes.POINTER(EngineInfo)]),
    ("snp_begin", ctypes.c_int, [_EngineP, ctypes.c_void_p]),
    ("snp_advance", ctypes.c_int, [_EngineP, ctypes.POINTER(RunOpts), ctypes.c_int64,
                                   ctypes.POINTER(TraceOut), ctypes.POINTER(Result)]),
    ("snp_read_state", ctypes.c_int, [_EngineP, ctypes.c_void_p, ctypes.c_void_p]),
    ("snp_run", ctypes.c_int, [_EngineP, ctypes.c_void_p, ctypes.POINTER(RunOpts), ctypes.c_void_p,
                               ctypes.c_void_p, ctypes.POINTER(Result)]),
    ("snp_last_device_ms", ctypes.c_double, [_EngineP]),
    ("snp_sv_calc", ctypes.c_int, [_EngineP, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
                                   ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p]),
    ("snp_step", ctypes.c_int, [_EngineP, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_void_p, ctypes.c_void_p]),
    ("snp_update_delays", ctypes.c_int, [_EngineP, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    ("snp_exchange_info", ctypes.c_int, [_EngineP, ctypes.POINTER(Exchange)]),
    ("snp_set_stream", ctypes.c_int, [_EngineP, ctypes.c_void_p]),
    ("snp_configure", ctypes.c_int, [_EngineP, ctypes.POINTER(RunOpts)]),
    ("snp_launch_step", ctypes.c_int, [_EngineP]),
    ("snp_read_trace", ctypes.c_int, [_EngineP, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_void_p]),
    ("snp_poll", ctypes.c_int, [_EngineP, ctypes.POINTER(Result)]),
    ("snp_engine_layout_digest", ctypes.c_int, [_EngineP, ctypes.c_void_p]),
    ("snp_exchange_ipc_handle", ctypes.c_int, [_EngineP, ctypes.c_void_p]),
    ("snp_exchange_connect", ctypes.c_int, [_EngineP, ctypes.c_void_p, ctypes.c_int]),
    ("snp_exchange_connect_local", ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int]),
    ("snp_time_steps", ctypes.c_int, [_EngineP, ctypes.POINTER(RunOpts), ctypes.c_int64,
                                      ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                      ctypes.POINTER(Result)]),
]

_lib = None


class NativeError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


def load() -> ctypes.CDLL:
    """Load the in-tree library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("SNPB200_LIB", LIB_PATH))
    if not path.exists():
        raise ImportError(
            f"{path} not found: build the CUDA engine first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    lib = ctypes.CDLL(str(path))
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc != SNP_OK:
        msg = load().snp_last_error().decode(errors="replace")
        raise NativeError(rc, msg)


def ptr(a: np.ndarray | None):
    """Raw pointer of a C-contiguous array (None -> NULL)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    return ctypes.c_void_p(a.ctypes.data)


def i64p(a: np.ndarray | None):
    if a is None:
        return None
    return a.ctypes.data_as(_i64p)


def u8p(a: np.ndarray | None):
    if a is None:
        return None
    return a.ctypes.data_as(_u8p)
