"""JIT isolation ("no file-system access" at JIT
time, PAPER.md:351 the in-memory source): specializing a key must not open
any source, header or compiled-kernel file.  An LD_PRELOAD shim
(tests/support/open_spy.c, test-only) logs every open/openat/fopen path while
JM_OPEN_SPY_LOG is set; NVRTC compiles for sm_100a without a GPU, so this runs
on the CPU tier.
"""
from __future__ import annotations

import os
import subprocess
import sys
import textwrap

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUSPECT = (".h", ".hpp", ".cuh", ".cu", ".cubin", ".ptx", ".fatbin", ".cpp", ".c")


@pytest.fixture(scope="module")
def spy_lib(tmp_path_factory):
    out = tmp_path_factory.mktemp("spy") / "open_spy.so"
    subprocess.run(["gcc", "-O2", "-shared", "-fPIC", "-o", str(out),
                    os.path.join(ROOT, "tests", "support", "open_spy.c"), "-ldl"], check=True)
    return str(out)


def _spy_run(spy_lib, log, body):
    code = textwrap.dedent(f"""
        import os, sys
        sys.path.insert(0, {ROOT!r})
        import paper_1904_08555_b200 as jm
        os.environ["JM_OPEN_SPY_LOG"] = {str(log)!r}
        {body}
        del os.environ["JM_OPEN_SPY_LOG"]
    """)
    env = dict(os.environ, LD_PRELOAD=spy_lib)
    subprocess.run([sys.executable, "-c", code], check=True, env=env, timeout=600)
    return open(log).read().split() if os.path.exists(log) else []


def test_spy_sees_file_opens(spy_lib, tmp_path):
    # the shim works: an explicit read of a header is logged
    paths = _spy_run(spy_lib, tmp_path / "log", f"open({os.path.join(ROOT, 'include', 'jit_mat.h')!r}).read()")
    assert any(p.endswith("jit_mat.h") for p in paths)


@pytest.mark.parametrize("args", [(16, "double", "ones"), (5, "float", "identity"), (40, "double", "stream"),
                                  (8, "float", "matmul")])
def test_specialization_opens_no_source_or_kernel_files(spy_lib, tmp_path, args):
    n, dt, what = args
    paths = _spy_run(spy_lib, tmp_path / "log", f"assert jm.jit_mat_compile_check({n}, {dt!r}, {what!r}) > 0")
    bad = [p for p in paths if p.endswith(SUSPECT) or "/include" in p or "csrc" in p]
    assert not bad, f"NVRTC specialization opened files: {bad}"
