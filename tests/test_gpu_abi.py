"""C ABI behaviour on the GPU: cache laws, error codes, concurrency, key info.

Cache-law ideas follow SPEC.md:644 (1000 calls over 10 keys -> 10
compilations) and SPEC.md:561 (concurrent lookup, mutually exclusive
insertion); the paper's program-global cache is PAPER.md:306 / Algorithm 1
lines 319 and 347.
"""
from __future__ import annotations

import os
import threading

import numpy as np
import pytest

import jm_synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture()
def jm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1904_08555_b200 as jm
    torch.cuda.init()
    jm.jit_mat_init(0)
    yield jm


def _fresh(jm):
    jm.jit_mat_shutdown()
    jm.jit_mat_init(0)
    jm.jit_mat_reset_stats()


def test_single_compilation_law(jm):
    _fresh(jm)
    rng = np.random.default_rng(1904)
    keys = [(n, dt) for n, dt in zip([2, 3, 5, 8, 11, 16, 21, 32, 40, 64],
                                     ["f64", "f32"] * 5)]
    bufs = {}
    for n, dt in keys:
        tdt = torch.float64 if dt == "f64" else torch.float32
        bufs[(n, dt)] = torch.zeros(4, n, n, dtype=tdt, device="cuda")
    trace = rng.integers(0, len(keys), 1000)
    for i in trace:
        n, dt = keys[i]
        x = bufs[(n, dt)]
        jm.jit_mat_run(n, dt, 4, 1, x.data_ptr(), x.data_ptr())
    torch.cuda.synchronize()
    st = jm.jit_mat_stats()
    assert st["compilations"] == 10
    assert st["misses"] == 10
    assert st["hits"] == 990
    assert st["launches"] == 1000
    assert st["keys_ready"] == 10


def test_concurrent_cold_key_compiles_once(jm):
    _fresh(jm)
    errs = []

    def worker():
        try:
            jm.jit_mat_prepare(24, "double")
        except Exception as e:  # pragma: no cover
            errs.append(e)

    ts = [threading.Thread(target=worker) for _ in range(16)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs
    st = jm.jit_mat_stats()
    assert st["compilations"] == 1
    assert st["hits"] + st["misses"] == 16


def test_distinct_keys_compile_in_parallel_threads(jm):
    _fresh(jm)
    keys = [(n, dt) for n in (6, 9, 14, 27) for dt in ("double", "float")]
    ts = [threading.Thread(target=jm.jit_mat_prepare, args=k) for k in keys]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert jm.jit_mat_stats()["compilations"] == len(keys)


def test_generic_is_preseeded(jm):
    _fresh(jm)
    for n in (1, 7, 64):
        jm.jit_mat_prepare(n, "double", kind="generic")
    assert jm.jit_mat_stats()["compilations"] == 0


def test_key_info_reports_registers(jm):
    _fresh(jm)
    for n, dt in ((4, "double"), (16, "double"), (15, "float"), (16, "float"), (32, "float"), (64, "double")):
        jm.jit_mat_prepare(n, dt)
    info = {(k["n"], k["dtype"], k["kind"]): k for k in jm.jit_mat_key_info()}
    k16 = info[(16, 1, 0)]
    assert k16["state"] == 2 and k16["regs"] > 0 and k16["cubin_bytes"] > 0
    assert k16["tile_name"] == "warp_dmma"
    assert info[(64, 1, 0)]["tile_name"] == "cta_dmma"
    assert info[(4, 1, 0)]["tile_name"] == "tpm"
    assert info[(15, 0, 0)]["tile_name"] == "f32_rows"
    assert info[(16, 0, 0)]["tile_name"] == "warp_f32"
    assert info[(32, 0, 0)]["tile_name"] == "f32_tc"        # FP32 on the tensor cores (3xTF32)
    for k in info.values():
        assert k["local_bytes"] == 0, f"spill in {k}"


def test_error_codes(jm):
    x = torch.zeros(8, 4, 4, dtype=torch.float64, device="cuda")
    p = x.data_ptr()
    lib = jm.lib
    assert lib.jit_mat_run(0, 1, 8, 1, p, p) == jm.JM_E_INVALID
    assert lib.jit_mat_run(65, 1, 8, 1, p, p) == jm.JM_E_UNSUPPORTED
    assert lib.jit_mat_run(4, 2, 8, 1, p, p) == jm.JM_E_UNSUPPORTED
    assert lib.jit_mat_run(4, 1, -1, 1, p, p) == jm.JM_E_INVALID
    assert lib.jit_mat_run(4, 1, 8, -1, p, p) == jm.JM_E_INVALID
    assert lib.jit_mat_run(4, 1, 8, 1 << 31, p, p) == jm.JM_E_INVALID
    assert lib.jit_mat_run(4, 1, 4, 1, p + 8, p + 8) == jm.JM_E_ALIGN
    assert lib.jit_mat_run(4, 1, 4, 1, p, p + 128) == jm.JM_E_INVALID   # partial overlap
    assert lib.jit_mat_run(4, 1, 4, 1, None, p) == jm.JM_E_INVALID
    assert lib.jit_mat_run(4, 1, 0, 1, None, None) == jm.JM_OK            # empty batch
    assert lib.jit_mat_dtype_from_name(b"long double") == jm.JM_E_UNSUPPORTED
    assert "long double" in jm.jit_mat_last_error()
    assert lib.jit_mat_dtype_from_name(b"double") == jm.JM_F64
    assert lib.jit_mat_dtype_from_name(b"float") == jm.JM_F32
    assert lib.jit_mat_init(1 if torch.cuda.device_count() == 1 else 0) in (jm.JM_E_INVALID, jm.JM_OK)


def test_shutdown_then_not_initialized(jm):
    x = torch.zeros(2, 3, 3, dtype=torch.float32, device="cuda")
    jm.jit_mat_shutdown()
    assert jm.lib.jit_mat_run(3, 0, 2, 1, x.data_ptr(), x.data_ptr()) == jm.JM_E_NOT_INITIALIZED
    assert jm.lib.jit_mat_prepare(3, 0, 0, 0) == jm.JM_E_NOT_INITIALIZED
    jm.jit_mat_init(0)
    y = jm.run(x, 1, sync=True)
    assert torch.all(y == 1.0)   # O1: zero input, one repeat -> all ones


def test_device_info(jm):
    info = jm.jit_mat_device_info()
    assert info["cc"][0] == 10
    assert info["sm_count"] == torch.cuda.get_device_properties(0).multi_processor_count


def test_set_stream_is_honoured(jm):
    s = torch.cuda.Stream()
    x = jm_synth.generate(16, "f64", "bench", 1, 0, 4096)
    xd = torch.from_numpy(x).cuda()
    out = torch.empty_like(xd)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        jm.jit_mat_set_stream(s.cuda_stream)
        jm.jit_mat_run(16, "f64", 4096, 10, xd.data_ptr(), out.data_ptr())
        ev = torch.cuda.Event()
        ev.record(s)
    ev.synchronize()
    ref = torch.empty_like(xd)
    jm.run(xd, 10, ref, sync=True)
    assert torch.equal(out, ref)
    jm.jit_mat_set_stream(torch.cuda.current_stream().cuda_stream)


def test_aot_specializations_preseeded_and_identical(jm):
    """F3's three-way comparison: JIT (NVRTC) vs AoT specialization (nvcc) vs generic.

    The AoT specializations are the same template body compiled ahead of time, so
    their outputs must equal the NVRTC ones bit for bit; they never compile
    (explicit specializations are used instead of JIT-compiling).
    """
    _fresh(jm)
    for n in (3, 7, 16):
        jm.jit_mat_prepare(n, "double", kind="aot_specialized")
    assert jm.jit_mat_stats()["compilations"] == 0
    for n in (3, 7, 16):
        for addend in ("ones", "identity"):
            x = torch.from_numpy(jm_synth.generate(n, "f64", "hard", 9, 0, 999)).cuda()
            a = jm.run(x, 5, addend=addend, kind="aot_specialized", sync=True)
            b = jm.run(x, 5, addend=addend, kind="specialized", sync=True)
            assert torch.equal(a, b), (n, addend)
    with pytest.raises(jm.JitMatError) as e:
        jm.jit_mat_prepare(8, "double", kind="aot_specialized")
    assert e.value.code == jm.JM_E_UNSUPPORTED
    with pytest.raises(jm.JitMatError):
        jm.jit_mat_prepare(16, "float", kind="aot_specialized")


def test_cache_export_import_skips_nvrtc(jm):
    """f2: one process compiles, another installs the blob (NVRTC not run)."""
    _fresh(jm)
    x = torch.from_numpy(jm_synth.generate(13, "f64", "hard", 2, 0, 77)).cuda()
    ref = jm.run(x, 3, sync=True)
    ref100 = jm.run(x, 100, sync=True)     # R = 3 runs the streaming variant, R = 100 the resident one
    blob = jm.jit_mat_cache_export(13, "double")
    assert blob[:4] == b"JMC3" and len(blob) > 2000
    _fresh(jm)
    jm.jit_mat_cache_import(blob)
    jm.jit_mat_cache_import(blob)          # second import: no-op
    got = jm.run(x, 3, sync=True)
    got100 = jm.run(x, 100, sync=True)
    st = jm.jit_mat_stats()
    assert st["compilations"] == 0 and st["imports"] == 2
    assert torch.equal(got, ref) and torch.equal(got100, ref100)
    with pytest.raises(jm.JitMatError):
        jm.jit_mat_cache_import(blob[:40])
    with pytest.raises(jm.JitMatError):
        jm.jit_mat_cache_import(b"JMC1" + blob[4:])
    # another build: digest mismatch
    bad = bytearray(blob)
    bad[4] = ord("0") if bad[4] != ord("0") else ord("1")
    with pytest.raises(jm.JitMatError, match="another library build"):
        jm.jit_mat_cache_import(bytes(bad))
    # the same cubins relabelled as another key: name expression mismatch
    import struct
    other = bytearray(blob)
    struct.pack_into("<i", other, 4 + 64, 21)
    with pytest.raises(jm.JitMatError, match="does not match"):
        jm.jit_mat_cache_import(bytes(other))
    with pytest.raises(jm.JitMatError):
        jm.jit_mat_cache_export(14, "double")


def test_non_sm100_device_is_rejected_without_fallback():
    """A device that is not compute capability 10.x (simulated with the
    JIT_MAT_FAKE_CC_MAJOR test hook) gets JM_E_ARCH at init and every run then
    fails with JM_E_NOT_INITIALIZED: there is no CPU fallback."""
    import subprocess
    import sys
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import paper_1904_08555_b200 as jm\n"
        "rc = jm.lib.jit_mat_init(0)\n"
        "assert rc == jm.JM_E_ARCH, rc\n"
        "assert 'compute capability 9' in jm.jit_mat_last_error()\n"
        "assert jm.lib.jit_mat_run(4, 1, 0, 1, None, None) == jm.JM_E_NOT_INITIALIZED\n"
        "print('ok')\n" % ROOT)
    env = dict(os.environ, JIT_MAT_FAKE_CC_MAJOR="9")
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0 and p.stdout.strip() == "ok", p.stderr[-2000:]


@pytest.mark.parametrize("groups", ["1", "3"])
def test_run_many_batched_compile(jm, groups, monkeypatch):
    """f2: the cold keys of a mixed-N call compiled as multi-expression NVRTC
    programs (JM_FLAG_BATCH_COMPILE) give the same bits as the per-key path."""
    monkeypatch.setenv("JIT_MAT_COMPILE_GROUPS", groups)
    cases = [(5, "f64", 3), (12, "f64", 1), (17, "f64", 100), (24, "f32", 2), (33, "f32", 100), (40, "f64", 3)]
    xs = [torch.from_numpy(jm_synth.generate(n, dt, "shard", 77 + n, 0, 41)).cuda() for n, dt, _ in cases]
    _fresh(jm)
    want = [jm.run(x, r, sync=True) for x, (n, dt, r) in zip(xs, cases)]
    _fresh(jm)
    outs = [torch.empty_like(x) for x in xs]
    jm.jit_mat_run_many([dict(n=n, dtype=dt, batch=41, repeat=r, in_ptr=x.data_ptr(), out_ptr=y.data_ptr())
                         for x, y, (n, dt, r) in zip(xs, outs, cases)], sync=True, batch_compile=True)
    st = jm.jit_mat_stats()
    assert st["compilations"] == len(cases) and st["programs"] == min(int(groups), len(cases))
    for w, g, c in zip(want, outs, cases):
        assert torch.equal(w, g), f"batched compile differs at {c}"
    info = [k for k in jm.jit_mat_key_info() if k["kind"] == 0]
    assert len(info) == len(cases) and all(k["state"] == 2 and k["regs"] > 0 for k in info)
