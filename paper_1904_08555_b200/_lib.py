"""ctypes declarations for libjitmat.so (mirrors include/jit_mat.h)."""
from __future__ import annotations

import ctypes
import os

lib_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libjitmat.so")
if not os.path.exists(lib_path):
    raise ImportError(
        f"{lib_path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is no CPU fallback)")

lib = ctypes.CDLL(lib_path)

JM_F32, JM_F64 = 0, 1
JM_ADDEND_ONES, JM_ADDEND_IDENTITY = 0, 1
JM_KIND_SPECIALIZED, JM_KIND_GENERIC, JM_KIND_AOT_SPECIALIZED = 0, 1, 2
JM_OK = 0
JM_E_INVALID, JM_E_UNSUPPORTED, JM_E_NOT_INITIALIZED = -1, -2, -3
JM_E_ARCH, JM_E_COMPILE, JM_E_CUDA, JM_E_ALIGN = -4, -5, -6, -7
JM_FLAG_SYNC, JM_FLAG_HOST_BUFFERS, JM_FLAG_RESIDENT, JM_FLAG_STREAMING = 1, 2, 4, 8
JM_FLAG_BATCH_COMPILE = 16
JM_FLAG_LATENCY = 32
JM_TILE_NAMES = {0: "generic", 1: "tpm", 2: "warp_dmma", 3: "cta_dmma", 4: "warp_f32",
                 5: "cta_f32", 6: "rows", 7: "matmul", 8: "tpm2", 9: "tpms", 10: "f32_rows", 11: "f64_reg", 12: "lat", 13: "f32_tc"}
JM_OP_MATMUL = 2
JM_OP_MASS = 3
JM_OP_STREAM = 4
JM_OP_LAT = 5


class JitMatError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class jm_run_desc(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int), ("dtype", ctypes.c_int), ("addend", ctypes.c_int),
                ("kind", ctypes.c_int), ("batch", ctypes.c_int64), ("repeat", ctypes.c_int64),
                ("in_", ctypes.c_void_p), ("out", ctypes.c_void_p), ("stream", ctypes.c_void_p),
                ("flags", ctypes.c_uint)]


class jm_stats(ctypes.Structure):
    _fields_ = [("compilations", ctypes.c_int64), ("hits", ctypes.c_int64),
                ("misses", ctypes.c_int64), ("launches", ctypes.c_int64),
                ("compile_ms_total", ctypes.c_double), ("keys_ready", ctypes.c_int32),
                ("keys_failed", ctypes.c_int32), ("imports", ctypes.c_int64), ("programs", ctypes.c_int64)]


class jm_key_info(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("dtype", ctypes.c_int32), ("addend", ctypes.c_int32),
                ("kind", ctypes.c_int32), ("state", ctypes.c_int32), ("regs", ctypes.c_int32),
                ("local_bytes", ctypes.c_int32), ("smem_bytes", ctypes.c_int32),
                ("threads", ctypes.c_int32), ("tile", ctypes.c_int32),
                ("cubin_bytes", ctypes.c_int64), ("compile_ms", ctypes.c_double),
                ("op", ctypes.c_int32), ("variant", ctypes.c_int32)]


_I, _I64, _P, _U64 = ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_uint64
_SIGS = {
    "jit_mat_init": (_I, [_I]),
    "jit_mat_run": (_I, [_I, _I, _I64, _I64, _P, _P]),
    "jit_mat_shutdown": (_I, []),
    "jit_mat_run_ex": (_I, [ctypes.POINTER(jm_run_desc)]),
    "jit_mat_run_host": (_I, [_I, _I, _I64, _I64, _P, _P]),
    "jit_mat_run_many": (_I, [ctypes.POINTER(jm_run_desc), _I, _P, ctypes.c_uint]),
    "jit_mat_cache_export": (_I, [_I, _I, _I, _P, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
    "jit_mat_cache_import": (_I, [_P, ctypes.c_size_t]),
    "jit_mat_set_stream": (_I, [_P]),
    "jit_mat_prepare": (_I, [_I, _I, _I, _I]),
    "jit_mat_prepare_for": (_I, [_I, _I, _I, _I, _I64, ctypes.c_uint, ctypes.POINTER(_I)]),
    "jit_mat_dtype_from_name": (_I, [ctypes.c_char_p]),
    "jit_mat_last_error": (ctypes.c_char_p, []),
    "jit_mat_stats": (_I, [ctypes.POINTER(jm_stats)]),
    "jit_mat_key_info": (_I, [ctypes.POINTER(jm_key_info), _I]),
    "jit_mat_reset_stats": (_I, []),
    "jit_mat_fill": (_I, [_I, _I, _I, _U64, _I64, _I64, _P]),
    "jit_mat_checksum": (_I, [_I, _I, _I64, _I64, _P, ctypes.POINTER(_U64),
                              ctypes.POINTER(ctypes.c_double)]),
    "jit_mat_device_info": (_I, [ctypes.POINTER(_I)] * 3),
    "jit_mat_version": (ctypes.c_char_p, []),
    "jit_mat_compile_check": (_I, [_I, _I, _I, ctypes.POINTER(ctypes.c_longlong)]),
    "jit_mat_matmul": (_I, [_I, _I, _I, _I64, _P, _P, _P, _P]),
    "jit_mat_mass": (_I, [_I, _I, _I, _I64, _P, _P, _P, _P, _P]),
    "jit_mat_time_lookup": (_I, [_I, _I, _I, _I, _I64, ctypes.POINTER(ctypes.c_double)]),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTS = tuple(_SIGS)
