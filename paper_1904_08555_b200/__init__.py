"""paper_1904_08555_b200 — JIT-specialized batched small-matrix update on B200.

A thin ctypes binding over ``libjitmat.so`` (C ABI: ``include/jit_mat.h``).
Every name below mirrors the C entry point of the same name; the functions do
argument marshalling only — all work (NVRTC specialization, caching, every
kernel) happens inside the library.  There is no CPU fallback: if the library
is missing the import fails, and without a B200 ``jit_mat_init`` returns
``JM_E_ARCH`` / ``JM_E_CUDA``.

The operation is the Eigen benchmark update of ClangJIT (arXiv 1904.08555,
PAPER.md:362, Listings 4/5 lines 364-414): ``M <- Ones + T(0.00005)*(M + M*M)``
repeated ``repeat`` times on each of ``batch`` independent N x N matrices.
"""
from __future__ import annotations

import ctypes
import os

from ._lib import (  # noqa: F401  (re-exported C ABI)
    JM_ADDEND_IDENTITY, JM_ADDEND_ONES, JM_E_ALIGN, JM_E_ARCH, JM_E_COMPILE, JM_E_CUDA,
    JM_E_INVALID, JM_E_NOT_INITIALIZED, JM_E_UNSUPPORTED, JM_F32, JM_F64, JM_FLAG_HOST_BUFFERS,
    JM_FLAG_RESIDENT, JM_FLAG_STREAMING, JM_FLAG_SYNC, JM_FLAG_BATCH_COMPILE, JM_FLAG_LATENCY, JM_KIND_AOT_SPECIALIZED, JM_KIND_GENERIC, JM_KIND_SPECIALIZED, JM_OK, JM_OP_MATMUL,
    JM_OP_LAT, JM_OP_STREAM, JM_TILE_NAMES, JitMatError,
    jm_key_info, jm_run_desc, jm_stats, lib, lib_path,
)

__all__ = [
    "jit_mat_init", "jit_mat_run", "jit_mat_shutdown", "jit_mat_run_ex", "jit_mat_run_host",
    "jit_mat_run_many", "jit_mat_cache_export", "jit_mat_cache_import", "jit_mat_matmul",
    "jit_mat_time_lookup", "matmul", "jit_mat_mass", "mass",
    "jit_mat_set_stream", "jit_mat_prepare", "jit_mat_prepare_for", "jit_mat_dtype_from_name", "jit_mat_last_error",
    "jit_mat_stats", "jit_mat_key_info", "jit_mat_reset_stats", "jit_mat_fill",
    "jit_mat_checksum", "jit_mat_device_info", "jit_mat_version", "jit_mat_compile_check",
    "run", "JitMatError",
]

_DTYPES = {"float": JM_F32, "f32": JM_F32, "float32": JM_F32,
           "double": JM_F64, "f64": JM_F64, "float64": JM_F64}
_ADDENDS = {"ones": JM_ADDEND_ONES, "identity": JM_ADDEND_IDENTITY}
_KINDS = {"specialized": JM_KIND_SPECIALIZED, "generic": JM_KIND_GENERIC,
          "aot_specialized": JM_KIND_AOT_SPECIALIZED}


def _check(rc: int, what: str) -> int:
    if rc < 0:
        raise JitMatError(rc, f"{what}: {jit_mat_last_error()}")
    return rc


def _enum(table: dict, x, what: str) -> int:
    """Name or integer -> the C enum value; an unknown name is an error, never 0."""
    if isinstance(x, int):
        return x
    if x in table:
        return table[x]
    raise ValueError(f"unknown {what} {x!r} (one of {sorted(table)} or its integer value)")


def _ad(addend) -> int:
    return _enum(_ADDENDS, addend, "addend")


def _kd(kind) -> int:
    return _enum(_KINDS, kind, "kind")


def _dt(dtype) -> int:
    if isinstance(dtype, int):
        return dtype
    name = getattr(dtype, "__name__", None) or str(dtype).replace("torch.", "")
    if name in _DTYPES:
        return _DTYPES[name]
    return _check(lib.jit_mat_dtype_from_name(str(dtype).encode()), "dtype")


# ---------------------------------------------------------------- C ABI mirror
def jit_mat_init(device: int = -1) -> None:
    _check(lib.jit_mat_init(int(device)), "jit_mat_init")


def jit_mat_shutdown() -> None:
    _check(lib.jit_mat_shutdown(), "jit_mat_shutdown")


def jit_mat_run(n: int, dtype, batch: int, repeat: int, in_ptr: int, out_ptr: int) -> None:
    _check(lib.jit_mat_run(int(n), _dt(dtype), int(batch), int(repeat), ctypes.c_void_p(in_ptr),
                           ctypes.c_void_p(out_ptr)), "jit_mat_run")


def jit_mat_run_ex(n: int, dtype, batch: int, repeat: int, in_ptr: int, out_ptr: int, *,
                   addend="ones", kind="specialized", stream: int | None = None,
                   flags: int = 0) -> None:
    d = jm_run_desc(int(n), _dt(dtype), _ad(addend), _kd(kind),
                    int(batch), int(repeat), ctypes.c_void_p(in_ptr), ctypes.c_void_p(out_ptr),
                    ctypes.c_void_p(stream or 0), int(flags))
    _check(lib.jit_mat_run_ex(ctypes.byref(d)), "jit_mat_run_ex")


def jit_mat_run_host(n: int, dtype, batch: int, repeat: int, in_ptr: int, out_ptr: int) -> None:
    _check(lib.jit_mat_run_host(int(n), _dt(dtype), int(batch), int(repeat),
                                ctypes.c_void_p(in_ptr), ctypes.c_void_p(out_ptr)),
           "jit_mat_run_host")


def jit_mat_run_many(groups, stream: int | None = None, sync: bool = False,
                     batch_compile: bool = False) -> None:
    """Mixed-N batch: ``groups`` is a sequence of dicts with keys n, dtype, batch,
    repeat, in_ptr, out_ptr and optional addend / kind (C: jit_mat_run_many);
    ``batch_compile`` compiles the cold keys as a few multi-expression NVRTC
    programs (JM_FLAG_BATCH_COMPILE)."""
    arr = (jm_run_desc * max(1, len(groups)))()
    for i, g in enumerate(groups):
        arr[i] = jm_run_desc(int(g["n"]), _dt(g["dtype"]), _ad(g.get("addend", "ones")),
                             _kd(g.get("kind", "specialized")), int(g["batch"]),
                             int(g["repeat"]), ctypes.c_void_p(g["in_ptr"]),
                             ctypes.c_void_p(g["out_ptr"]), None, 0)
    _check(lib.jit_mat_run_many(arr, len(groups), ctypes.c_void_p(stream or 0),
                                (JM_FLAG_SYNC if sync else 0) | (JM_FLAG_BATCH_COMPILE if batch_compile else 0)),
           "jit_mat_run_many")


def jit_mat_cache_export(n: int, dtype, addend="ones") -> bytes:
    """Blob (key + symbol + sm_100a cubin) of a compiled specialization."""
    ln = ctypes.c_size_t(0)
    a = _ad(addend)
    _check(lib.jit_mat_cache_export(int(n), _dt(dtype), a, None, 0, ctypes.byref(ln)),
           "jit_mat_cache_export")
    buf = ctypes.create_string_buffer(ln.value)
    _check(lib.jit_mat_cache_export(int(n), _dt(dtype), a, buf, ln.value, ctypes.byref(ln)),
           "jit_mat_cache_export")
    return buf.raw[:ln.value]


def jit_mat_cache_import(blob: bytes) -> None:
    """Install a blob from jit_mat_cache_export without running NVRTC."""
    _check(lib.jit_mat_cache_import(blob, len(blob)), "jit_mat_cache_import")


def jit_mat_matmul(n: int, dtype, batch: int, a_ptr: int, b_ptr: int, c_ptr: int, *,
                   kind="specialized", stream: int | None = None) -> None:
    """c[b] += a[b] @ b[b] (Listing 8; C: jit_mat_matmul)."""
    _check(lib.jit_mat_matmul(int(n), _dt(dtype), _kd(kind), int(batch),
                              ctypes.c_void_p(a_ptr), ctypes.c_void_p(b_ptr), ctypes.c_void_p(c_ptr),
                              ctypes.c_void_p(stream or 0)), "jit_mat_matmul")


def jit_mat_mass(dofs: int, quads: int, elements: int, B_ptr: int, op_ptr: int, x_ptr: int,
                 y_ptr: int, *, kind="specialized", stream: int | None = None) -> None:
    """Laghos 2D mass action y_e += B^T((B x_e B^T) .* op_e) B (C: jit_mat_mass)."""
    _check(lib.jit_mat_mass(int(dofs), int(quads), _kd(kind), int(elements),
                            ctypes.c_void_p(B_ptr), ctypes.c_void_p(op_ptr), ctypes.c_void_p(x_ptr),
                            ctypes.c_void_p(y_ptr), ctypes.c_void_p(stream or 0)), "jit_mat_mass")


def mass(B, op, x, y, *, kind: str = "specialized", stream=None, sync: bool = False):
    """y += mass action of x for float64 CUDA tensors B (Q,D), op (E,Q,Q), x/y (E,D,D)."""
    import torch

    Q, D = B.shape
    E = x.shape[0]
    for t, shp in ((B, (Q, D)), (op, (E, Q, Q)), (x, (E, D, D)), (y, (E, D, D))):
        if tuple(t.shape) != shp or t.dtype != torch.float64 or not t.is_cuda or not t.is_contiguous():
            raise ValueError("expected contiguous float64 CUDA tensors B (Q,D), op (E,Q,Q), x/y (E,D,D)")
    st = stream if stream is not None else torch.cuda.current_stream(x.device)
    jit_mat_mass(D, Q, E, B.data_ptr(), op.data_ptr(), x.data_ptr(), y.data_ptr(), kind=kind,
                 stream=st.cuda_stream)
    if sync:
        st.synchronize()
    return y


def jit_mat_time_lookup(n: int, dtype, addend="ones", kind="specialized", iters: int = 1_000_000) -> float:
    """Average ns per cache-hit lookup, timed inside the library (row a1)."""
    ns = ctypes.c_double(0.0)
    _check(lib.jit_mat_time_lookup(int(n), _dt(dtype), _ad(addend),
                                   _kd(kind), int(iters), ctypes.byref(ns)),
           "jit_mat_time_lookup")
    return float(ns.value)


def matmul(a, b, c, *, kind: str = "specialized", stream=None, sync: bool = False):
    """c += a @ b for CUDA tensors of shape (batch, n, n); returns c."""
    import torch

    for t in (a, b, c):
        if t.dim() != 3 or t.shape != a.shape or t.dtype != a.dtype or not t.is_cuda or not t.is_contiguous():
            raise ValueError("a, b, c must be contiguous CUDA tensors of one (batch, n, n) shape and dtype")
    st = stream if stream is not None else torch.cuda.current_stream(a.device)
    jit_mat_matmul(a.shape[1], str(a.dtype), a.shape[0], a.data_ptr(), b.data_ptr(), c.data_ptr(),
                   kind=kind, stream=st.cuda_stream)
    if sync:
        st.synchronize()
    return c


def jit_mat_set_stream(stream: int | None) -> None:
    _check(lib.jit_mat_set_stream(ctypes.c_void_p(stream or 0)), "jit_mat_set_stream")


def jit_mat_prepare(n: int, dtype, addend="ones", kind="specialized") -> None:
    _check(lib.jit_mat_prepare(int(n), _dt(dtype), _ad(addend),
                               _kd(kind)), "jit_mat_prepare")


def jit_mat_prepare_for(n: int, dtype, repeat: int, addend="ones", kind="specialized",
                        flags: int = 0) -> int:
    """Prepare the kernel a run with this repeat count (and flags) launches;
    returns its variant (0 resident, 1 streaming)."""
    v = ctypes.c_int(-1)
    _check(lib.jit_mat_prepare_for(int(n), _dt(dtype), _ad(addend),
                                   _kd(kind), int(repeat), int(flags), ctypes.byref(v)),
           "jit_mat_prepare_for")
    return int(v.value)


def jit_mat_dtype_from_name(name: str) -> int:
    return lib.jit_mat_dtype_from_name(name.encode())


def jit_mat_last_error() -> str:
    return lib.jit_mat_last_error().decode(errors="replace")


def jit_mat_stats() -> dict:
    s = jm_stats()
    _check(lib.jit_mat_stats(ctypes.byref(s)), "jit_mat_stats")
    return {f: getattr(s, f) for f, _ in jm_stats._fields_}


def jit_mat_key_info() -> list[dict]:
    cnt = lib.jit_mat_key_info(None, 0)
    arr = (jm_key_info * max(cnt, 1))()
    cnt = lib.jit_mat_key_info(arr, cnt)
    out = []
    for i in range(cnt):
        d = {f: getattr(arr[i], f) for f, _ in jm_key_info._fields_}
        d["tile_name"] = JM_TILE_NAMES.get(d["tile"], "?")
        out.append(d)
    return out


def jit_mat_reset_stats() -> None:
    _check(lib.jit_mat_reset_stats(), "jit_mat_reset_stats")


def jit_mat_fill(n: int, dtype, dist: int, seed: int, global_first: int, batch: int,
                 out_ptr: int) -> None:
    _check(lib.jit_mat_fill(int(n), _dt(dtype), int(dist), ctypes.c_uint64(seed),
                            int(global_first), int(batch), ctypes.c_void_p(out_ptr)),
           "jit_mat_fill")


def jit_mat_checksum(n: int, dtype, global_first: int, batch: int, x_ptr: int) -> tuple[int, float]:
    u = ctypes.c_uint64(0)
    f = ctypes.c_double(0.0)
    _check(lib.jit_mat_checksum(int(n), _dt(dtype), int(global_first), int(batch),
                                ctypes.c_void_p(x_ptr), ctypes.byref(u), ctypes.byref(f)),
           "jit_mat_checksum")
    return int(u.value), float(f.value)


def jit_mat_device_info() -> dict:
    sm, ma, mi = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    _check(lib.jit_mat_device_info(ctypes.byref(sm), ctypes.byref(ma), ctypes.byref(mi)),
           "jit_mat_device_info")
    return {"sm_count": sm.value, "cc": (ma.value, mi.value)}


def jit_mat_version() -> str:
    return lib.jit_mat_version().decode()


def jit_mat_compile_check(n: int, dtype, addend="ones") -> int:
    """NVRTC-compile a key without a GPU; addend="matmul" selects k_matmul,
    addend="stream" the streaming variant of k_update, and addend="mass"
    selects k_mass<n, dtype> (dtype = quads, an int)."""
    cb = ctypes.c_longlong(0)
    if addend == "mass":
        _check(lib.jit_mat_compile_check(int(n), int(dtype), 3, ctypes.byref(cb)), "jit_mat_compile_check")
        return int(cb.value)
    ops = {"matmul": JM_OP_MATMUL, "stream": JM_OP_STREAM, "lat": JM_OP_LAT}
    a = ops[addend] if addend in ops else _ad(addend)
    _check(lib.jit_mat_compile_check(int(n), _dt(dtype), a, ctypes.byref(cb)), "jit_mat_compile_check")
    return int(cb.value)


# ---------------------------------------------------------------- convenience
def run(x, repeat: int, out=None, *, addend: str = "ones", kind: str = "specialized",
        stream=None, sync: bool = False, variant: str | None = None):
    """Apply the update to a CUDA tensor ``x`` of shape (batch, n, n) (float32/float64).

    Marshals the tensor pointers into :func:`jit_mat_run_ex`; ``out`` may be ``x``
    (in place).  Runs on ``stream`` (default: torch's current stream).
    ``variant`` = "resident" / "streaming" / "latency" forces the kernel variant
    (default: the library picks by repeat count and batch, see jit_mat.h VARIANT).
    """
    import torch

    if x.dim() != 3 or x.shape[1] != x.shape[2]:
        raise ValueError("expected a (batch, n, n) tensor")
    if not x.is_cuda or not x.is_contiguous():
        raise ValueError("expected a contiguous CUDA tensor")
    if out is None:
        out = torch.empty_like(x)
    if out.shape != x.shape or out.dtype != x.dtype or not out.is_contiguous():
        raise ValueError("out must match x")
    st = stream if stream is not None else torch.cuda.current_stream(x.device)
    jit_mat_run_ex(x.shape[1], str(x.dtype), x.shape[0], repeat, x.data_ptr(), out.data_ptr(),
                   addend=addend, kind=kind, stream=st.cuda_stream,
                   flags=(JM_FLAG_SYNC if sync else 0) | _VARIANTS[variant])
    return out


_VARIANTS = {None: 0, "auto": 0, "resident": JM_FLAG_RESIDENT, "streaming": JM_FLAG_STREAMING,
             "latency": JM_FLAG_LATENCY}


def _selftest_loaded() -> str:
    return os.path.abspath(lib_path)
