"""The C ABI library loads without a GPU and exports every symbol include/a2a_exec.h declares."""
from __future__ import annotations

import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_every_declared_symbol_is_exported():
    from paper_2309_13541_b200 import _native
    hdr = open(os.path.join(ROOT, "include", "a2a_exec.h")).read()
    names = set(re.findall(r"^\s*(?:int|const char\*)\s+(a2a_\w+)\s*\(", hdr, re.M))
    assert len(names) >= 20
    lib = ctypes.CDLL(_native.LIB_PATH)
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    assert b"sm_100a" in _native.lib.a2a_version()


def test_sm100a_cubin_embedded():
    """The executor .so carries sm_100a SASS (no PTX-only / other-arch fallback)."""
    import shutil
    import subprocess
    from paper_2309_13541_b200 import _native
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([exe, "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_bind_without_gpu_fails_loudly():
    import pytest
    from paper_2309_13541_b200.artifacts import load_artifact
    from paper_2309_13541_b200.executor import ExecutorError, Plan
    a = load_artifact("torus2x4")
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with Plan(a.g, a.sched, m=64) as p:
        with pytest.raises((ExecutorError, ValueError)):
            p.bind(0)
