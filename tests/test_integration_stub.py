"""The ctypes stub shown in INTEGRATION.md works as written (extracted and run)."""
from __future__ import annotations

import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_integration_stub_runs(artifacts, golden):
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    code = re.search(r"```python\n(# a2aflow/evaluate\.py.*?)```", text, re.S).group(1)
    from paper_2309_13541_b200 import _native
    from paper_2309_13541_b200.executor import EvalError
    code = code.replace('"paper_2309_13541_b200/_a2a_exec.so"', repr(_native.LIB_PATH))
    ns = {"EvalError": EvalError}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    import ctypes as C
    ns["_lib"].a2a_last_error.restype = C.c_char_p
    a = artifacts("gk8_2")
    for (m, b, sync), want in zip(golden["params"], golden["configs"]["gk8_2"]["replay"]):
        T, ok = ns["replay_timestep_schedule"](a.g, a.sched, m, b, sync)
        assert ok and repr(T) == want["T"]
