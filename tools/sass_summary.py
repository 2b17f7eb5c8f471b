"""Opcode histogram of every kernel in _a2a_exec.so (cuobjdump -sass), the SASS
evidence for the copy engines: UBLKCP.* (TMA bulk copies) and SYNCS.* (mbarrier)
in the TMA kernels, LDG/STG .128 in the LSU kernels, STRONG.SYS / MEMBAR.*.SYS
for cross-GPU flags.  Usage: python tools/sass_summary.py > profiles/r01_sass_summary.txt"""
from __future__ import annotations

import collections
import datetime
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2309_13541_b200", "_a2a_exec.so")
KEEP = re.compile(r"^(UBLKCP|SYNCS|LDG|STG|LDS|STS|ATOMG|RED|MEMBAR|FENCE|CCTL|BAR|ELECT|UTMA|LD\.|ST\.|ATOM)")


def main():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    hist, fn = collections.OrderedDict(), None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            fn = m.group(1)
            hist.setdefault(fn, collections.Counter())
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
        if fn and m and KEEP.match(m.group(1)):
            hist[fn][m.group(1)] += 1
    sym = subprocess.run(["c++filt"], input="\n".join(hist), capture_output=True, text=True).stdout.split("\n")
    print(f"# SASS evidence for _a2a_exec.so (cuobjdump -sass), {datetime.date.today()}, sm_100a")
    print("# kernels:")
    for f, d in zip(hist, sym):
        print(f"#   {f}  ({d})")
    print("\n# instruction histogram per kernel (memory / sync opcodes)")
    for f, c in hist.items():
        for op, n in sorted(c.items()):
            print(f"{f} {op} {n}")
    tma = [f for f, c in hist.items() if any(k.startswith("UBLKCP") for k in c)]
    print(f"\n# kernels with TMA bulk copies (UBLKCP): {len(tma)}")


if __name__ == "__main__":
    sys.exit(main())
