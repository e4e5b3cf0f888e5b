"""CPU oracle for the batched Eigen-benchmark update — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
and ``--impl reference`` legs may import this package.  The product package
``paper_1904_08555_b200`` never imports it (tests/test_boundary.py checks).

The arithmetic lives in ``jm_oracle.c`` (plain C triple loop, compiled with
``-O2 -ffp-contract=off``; see its header for the paper passages and the
readings R1-R9).  This module only builds/loads it and marshals numpy arrays.

Pinned by tests/test_oracle_pins.py (O1-O12 of SURVEY.md §8(c)); no function
here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "jm_oracle.c")
_LIB = os.path.join(_HERE, "libjm_oracle.so")
_lock = threading.Lock()
_lib = None

ONES = 0
IDENTITY = 1
ADDENDS = {"ones": ONES, "identity": IDENTITY}


def build(force: bool = False) -> str:
    """Compile jm_oracle.c -> libjm_oracle.so (gcc, no fast-math, no FMA contraction)."""
    if (not force and os.path.exists(_LIB)
            and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC)):
        return _LIB
    tmp = _LIB + f".tmp{os.getpid()}"
    cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-fPIC",
           "-shared", "-pthread", "-o", tmp, _SRC]
    subprocess.run(cmd, check=True)
    os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            lib.jm_oracle_run.restype = ctypes.c_int
            lib.jm_oracle_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_int64, ctypes.c_int64,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
            lib.jm_oracle_matmul.restype = ctypes.c_int
            lib.jm_oracle_matmul.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                             ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.c_int]
            lib.jm_oracle_mass.restype = ctypes.c_int
            lib.jm_oracle_mass.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_int]
            _lib = lib
    return _lib


def mass_apply(y: np.ndarray, B: np.ndarray, op: np.ndarray, x: np.ndarray,
               threads: int | None = None) -> np.ndarray:
    """Return y + (Laghos 2D mass action on x) per element (reading R18; float64).

    Shapes: B (Q, D) = dofToQuad, op (E, Q, Q), x and y (E, D, D).  Follows
    jm_oracle.c's rMassMultAdd2D loop order; inputs are not modified.
    """
    lib = _load()
    B = np.ascontiguousarray(B, dtype=np.float64)
    op = np.ascontiguousarray(op, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.array(y, dtype=np.float64, copy=True, order="C")
    Q, D = B.shape
    E = x.shape[0]
    if x.shape != (E, D, D) or out.shape != (E, D, D) or op.shape != (E, Q, Q):
        raise ValueError("shapes: B (Q,D), op (E,Q,Q), x/y (E,D,D)")
    th = default_threads() if threads is None else int(threads)
    rc = lib.jm_oracle_mass(D, Q, E, B.ctypes.data_as(ctypes.c_void_p),
                            op.ctypes.data_as(ctypes.c_void_p), x.ctypes.data_as(ctypes.c_void_p),
                            out.ctypes.data_as(ctypes.c_void_p), th)
    if rc != 0:
        raise ValueError(f"jm_oracle_mass rejected arguments (rc={rc})")
    return out


def matmul_acc(c: np.ndarray, a: np.ndarray, b: np.ndarray, threads: int | None = None) -> np.ndarray:
    """Return c + a @ b per batch entry (Listing 8, batch reading R16).

    Computed in the arrays' dtype by jm_oracle.c (ascending k, separate
    multiply and add); the inputs are not modified.
    """
    lib = _load()
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    out = np.array(c, copy=True, order="C")
    if not (a.shape == b.shape == out.shape and a.dtype == b.dtype == out.dtype):
        raise ValueError("a, b, c must share shape (batch, n, n) and dtype")
    if a.ndim != 3 or a.shape[1] != a.shape[2]:
        raise ValueError("expected (batch, n, n)")
    dt = {np.dtype(np.float32): 0, np.dtype(np.float64): 1}.get(a.dtype)
    if dt is None:
        raise ValueError("oracle supports float32/float64")
    th = default_threads() if threads is None else int(threads)
    rc = lib.jm_oracle_matmul(a.shape[1], dt, a.shape[0], a.ctypes.data_as(ctypes.c_void_p),
                              b.ctypes.data_as(ctypes.c_void_p),
                              out.ctypes.data_as(ctypes.c_void_p), th)
    if rc != 0:
        raise ValueError(f"jm_oracle_matmul rejected arguments (rc={rc})")
    return out


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def run(x: np.ndarray, repeat: int, addend: str | int = "ones",
        threads: int | None = None) -> np.ndarray:
    """Return f^repeat applied to every matrix of ``x`` (shape (batch, n, n)).

    ``x`` must be float32 or float64; the update is computed in that type
    (the element type is the template argument T).
    """
    lib = _load()
    x = np.ascontiguousarray(x)
    if x.ndim != 3 or x.shape[1] != x.shape[2]:
        raise ValueError("expected (batch, n, n)")
    if x.dtype == np.float32:
        dt = 0
    elif x.dtype == np.float64:
        dt = 1
    else:
        raise ValueError("oracle supports float32/float64")
    a = ADDENDS[addend] if isinstance(addend, str) else int(addend)
    batch, n, _ = x.shape
    out = np.empty_like(x)
    th = default_threads() if threads is None else int(threads)
    rc = lib.jm_oracle_run(n, dt, a, batch, int(repeat),
                           x.ctypes.data_as(ctypes.c_void_p),
                           out.ctypes.data_as(ctypes.c_void_p), th)
    if rc != 0:
        raise ValueError(f"jm_oracle_run rejected arguments (rc={rc})")
    return out
