"""SASS guard for the bench tile (CPU: inspects the built libswdb.so).

The pass kernel's speed hangs on its instruction stream: the
biased 16x2 arithmetic issues exactly 3 VIADDMNMX + 1 VIMNMX3 per pair of cells
plus the S maximum, and the 16x29 bench tile must not touch local memory.  A
source change that perturbs the main loop (register allocation, spills, a
different cell form) shows here before any GPU time is spent on it.
"""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1702_07195_b200", "libswdb.so")
KERNEL = "sw16_pass_kernelILi29ELi16ELb0ELi0ELi512ELi4ELb0E"   # R=29, G=16, no boundary input, QPM 0


def _sass():
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    if not os.path.exists(LIB):
        from paper_1702_07195_b200 import build
        build.build()
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    for f in out.split("Function : ")[1:]:
        if KERNEL in f.split("\n", 1)[0]:
            return f
    pytest.fail(f"{KERNEL} not found in {LIB}")


def _main_loop(sass):
    ins = []
    for ln in sass.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", ln)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    best = None
    for a, t in ins:
        m = re.search(r"BRA (?:\S+ )?0x([0-9a-f]+)", t)
        if m:
            tgt = int(m.group(1), 16)
            if tgt < a and (best is None or a - tgt > best[1] - best[0]):
                best = (tgt, a)
    lo, hi = best
    body = [t for a, t in ins if lo <= a <= hi]
    # the unrolled column block starts after the claim code's VOTE.ALL (exit test)
    k = next(i for i, t in enumerate(body) if "VOTE.ALL" in t)
    return body[k:]


def test_bench_tile_instruction_stream():
    body = _main_loop(_sass())
    ops = [re.sub(r"^@!?U?P\w+\s+", "", t).split()[0] for t in body]
    U, R = 4, 29
    # per column: R rows x (hg, E, F) + the S reset max; R rows of Eq. 1 + (R-1)/2 S maxima
    assert ops.count("VIADDMNMX.U16x2") == U * (3 * R + 1)
    assert ops.count("VIMNMX3.U16x2") == U * (R + (R - 1) // 2)
    assert not any(o.startswith(("LDL", "STL")) for o in ops), "local memory (spills) in the main loop"
    # 245 issue slots per column in round 2: a regression shows as growth
    assert len(body) <= U * 250, len(body)
