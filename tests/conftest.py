"""Shared fixtures.  GPU tests are marked ``gpu``; everything else runs on CPU."""
from __future__ import annotations

import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def artifacts():
    from paper_2309_13541_b200.artifacts import load_artifact
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = load_artifact(name)
        return cache[name]
    return get


def apply_edit(sched, edit):
    """Rebuild a corrupted schedule from a golden edit record."""
    import copy
    from paper_2309_13541_b200.schedule import Instruction
    s = copy.deepcopy(sched)
    drop = set(edit.get("drop", []))
    s.instructions = [x for i, x in enumerate(s.instructions) if i not in drop]
    for a in edit.get("append", []):
        s.instructions.append(Instruction(*a))
    return s
