"""CPU tier: the C-ABI library loads, exports every symbol include/jit_mat.h
declares, rejects bad calls without a GPU, NVRTC-compiles every
specialization for sm_100a, and the product path is independent of the oracle.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def jm():
    import paper_1904_08555_b200 as jm
    return jm


def _header_symbols():
    with open(os.path.join(ROOT, "include", "jit_mat.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"^JM_API\s+[\w\s\*]*?\b(jit_mat_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_declared_symbol(jm):
    syms = _header_symbols()
    assert len(syms) >= 17
    for s in syms:
        assert hasattr(jm.lib, s), s
    assert set(syms) == set(jm._lib.EXPORTS)


def test_library_exports_only_the_abi(jm):
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", jm.lib_path], capture_output=True,
                         text=True, check=True).stdout
    funcs = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert funcs == set(_header_symbols())


def test_calls_fail_cleanly_without_init(jm):
    lib = jm.lib
    if lib.jit_mat_init(0) == 0:   # a GPU box: this test is about the uninitialised state
        pytest.skip("device present")
    assert lib.jit_mat_run(4, 1, 1, 1, None, None) in (jm.JM_E_NOT_INITIALIZED, jm.JM_E_INVALID)
    assert lib.jit_mat_run(4, 1, 0, 1, None, None) == jm.JM_E_NOT_INITIALIZED
    assert lib.jit_mat_prepare(4, 1, 0, 0) == jm.JM_E_NOT_INITIALIZED
    assert lib.jit_mat_prepare_for(16, 1, 0, 0, 1, 0, None) == jm.JM_E_NOT_INITIALIZED
    assert lib.jit_mat_shutdown() == jm.JM_E_NOT_INITIALIZED
    rc = lib.jit_mat_init(0)
    assert rc in (jm.JM_E_CUDA, jm.JM_E_ARCH)
    assert jm.jit_mat_last_error()


def test_argument_validation_precedes_init(jm):
    lib = jm.lib
    assert lib.jit_mat_prepare(0, 1, 0, 0) == jm.JM_E_INVALID
    assert lib.jit_mat_prepare(65, 1, 0, 0) == jm.JM_E_UNSUPPORTED
    assert lib.jit_mat_prepare(4, 7, 0, 0) == jm.JM_E_UNSUPPORTED
    assert lib.jit_mat_prepare(4, 1, 3, 0) == jm.JM_E_INVALID
    assert lib.jit_mat_prepare(4, 1, 0, 9) == jm.JM_E_INVALID


def test_dtype_names(jm):
    # Listing 4's type switch: float, double, long double
    assert jm.jit_mat_dtype_from_name("float") == jm.JM_F32
    assert jm.jit_mat_dtype_from_name("double") == jm.JM_F64
    assert jm.jit_mat_dtype_from_name("long double") == jm.JM_E_UNSUPPORTED
    assert jm.jit_mat_dtype_from_name("int") == jm.JM_E_UNSUPPORTED


def test_version(jm):
    assert "sm_100a" in jm.jit_mat_version()


@pytest.mark.parametrize("dtype", ["double", "float"])
def test_every_specialization_compiles_for_sm100a(jm, dtype):
    """NVRTC instantiates k_update<N, T, Ones> for every N in [1, 64] (no GPU)."""
    with cf.ThreadPoolExecutor(min(8, os.cpu_count() or 1)) as ex:
        sizes = list(ex.map(lambda n: jm.jit_mat_compile_check(n, dtype), range(1, 65)))
    assert all(s > 1000 for s in sizes)


@pytest.mark.parametrize("dtype", ["double", "float"])
def test_every_streaming_variant_compiles_for_sm100a(jm, dtype):
    """The low-repeat variant k_update_stream<N, T, Ones> for every N: the
    bulk-copy ring behind the DMMA / FP32 tile kinds, the double-buffered
    stage behind the thread-per-matrix kind."""
    with cf.ThreadPoolExecutor(min(8, os.cpu_count() or 1)) as ex:
        sizes = list(ex.map(lambda n: jm.jit_mat_compile_check(n, dtype, "stream"), range(1, 65)))
    assert all(s > 1000 for s in sizes)


@pytest.mark.parametrize("dtype", ["double", "float"])
def test_every_latency_variant_compiles_for_sm100a(jm, dtype):
    """k_update_lat<N, T, Ones> (a warp per matrix) for every N with N*N <= 32;
    larger N has no latency variant."""
    assert all(jm.jit_mat_compile_check(n, dtype, "lat") > 1000 for n in range(1, 6))
    with pytest.raises(jm.JitMatError):
        jm.jit_mat_compile_check(6, dtype, "lat")


@pytest.mark.parametrize("n", [1, 5, 8, 13, 33, 64])
def test_identity_specializations_compile(jm, n):
    assert jm.jit_mat_compile_check(n, "double", "identity") > 0
    assert jm.jit_mat_compile_check(n, "float", "identity") > 0


def test_compile_check_rejects_bad_keys(jm):
    from paper_1904_08555_b200 import JitMatError
    with pytest.raises(JitMatError):
        jm.jit_mat_compile_check(0, "double")
    with pytest.raises(JitMatError):
        jm.jit_mat_compile_check(65, "float")


def test_nvrtc_source_has_no_includes():
    from paper_1904_08555_b200 import _build
    src = _build.kernel_source()
    assert not re.search(r"^\s*#\s*include", src, flags=re.M)
    assert "k_update" in src


def test_product_never_touches_the_oracle():
    pkg = os.path.join(ROOT, "paper_1904_08555_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cpp", ".cu", ".cuh", ".h")):
                with open(os.path.join(dirpath, fn)) as f:
                    txt = f.read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, flags=re.M), fn
                assert "jm_oracle" not in txt, fn
    # and the oracle shares nothing with the product
    with open(os.path.join(ROOT, "oracle", "jm_oracle.c")) as f:
        src = f.read()
    assert "#include \"" not in src


def test_oracle_is_not_linked_into_the_library(jm):
    import subprocess
    out = subprocess.run(["nm", "-D", jm.lib_path], capture_output=True, text=True).stdout
    assert "jm_oracle" not in out


def test_binding_rejects_unknown_enum_names():
    """a misspelled addend/kind name must raise, never become 0
    (Ones / specialized); integers pass through unchanged."""
    import paper_1904_08555_b200 as jm
    assert jm._ad("identity") == jm.JM_ADDEND_IDENTITY and jm._ad(jm.JM_ADDEND_IDENTITY) == 1
    assert jm._kd("generic") == jm.JM_KIND_GENERIC and jm._kd(jm.JM_KIND_GENERIC) == 1
    with pytest.raises(ValueError):
        jm._ad("Identity")
    with pytest.raises(ValueError):
        jm._kd("specialised")
    with pytest.raises(ValueError):   # run_many marshals every group before calling the library
        jm.jit_mat_run_many([{"n": 4, "dtype": "f64", "batch": 1, "repeat": 1, "in_ptr": 0, "out_ptr": 0,
                              "addend": "Identity"}])


def test_every_mass_specialization_compiles_for_sm100a(jm):
    """k_mass<D, Q> (Listing 12, reading R18) for every D, Q in 1..8:
    the thread-per-element kernel and the r02 DMMA kernel (jm_plan.h mass_dmma)."""
    pairs = [(d, q) for d in range(1, 9) for q in range(1, 9)]
    with cf.ThreadPoolExecutor(min(8, os.cpu_count() or 1)) as ex:
        sizes = list(ex.map(lambda p: jm.jit_mat_compile_check(p[0], p[1], "mass"), pairs))
    assert all(s > 1000 for s in sizes)
    with pytest.raises(jm.JitMatError):
        jm.jit_mat_compile_check(9, 4, "mass")
