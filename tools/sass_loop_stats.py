"""Instruction mix of the pass kernel's column loop, from SASS (dev tool, CPU only).

Compiles csrc/kernels.cu to a cubin with extra -D flags, finds the column
loop of one sw16_pass_kernel instantiation (the largest backward branch's
body, minus the item-claim block the loop skips) and prints instructions per
column by class: ALU-pipe (VIMNMX3, VIADDMNMX, ...), FMA-pipe (IMAD incl.
IMAD.MOV), LDS, SHFL, other.

    python tools/sass_loop_stats.py [--R 29 --G 16 --bin 0] [-D SW_UNROLL=2 ...]
"""
import argparse
import collections
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1702_07195_b200 import build as B  # noqa: E402

ALU = ("VIMNMX3", "VIADDMNMX", "VIMNMX", "VIADD", "LOP3", "ISETP", "SEL", "IADD3", "SHF", "LEA", "POPC", "FLO", "VOTE")
FMA = ("IMAD",)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--R", type=int, default=29)
    ap.add_argument("--G", type=int, default=16)
    ap.add_argument("--bin", type=int, default=0)
    ap.add_argument("--U", type=int, default=0, help="unroll U of the instantiation (0: SW_UNROLL or 4)")
    ap.add_argument("-D", action="append", default=[])
    ap.add_argument("--xptxas", action="append", default=[], help="extra ptxas option, e.g. --register-usage-level=8")
    args = ap.parse_args()
    U = args.U or int(next((d.split("=")[1] for d in args.D if d.startswith("SW_UNROLL=")), 4))
    with tempfile.TemporaryDirectory() as td:
        cub = os.path.join(td, "k.cubin")
        cmd = [B._nvcc()] + B.NVCC_FLAGS + ["-D" + d for d in args.D] + [f"-Xptxas={x}" for x in args.xptxas] + ["-cubin", "-o", cub,
                                                                          os.path.join(B.CSRC, "kernels.cu")]
        subprocess.run(cmd, check=True)
        sass = subprocess.run(["cuobjdump", "-sass", cub], check=True, capture_output=True, text=True).stdout
    # sw16_pass_kernel<R, G, BIN, QPM = 0, NT = 512, U, WAVE = false, DA, RA>: the
    # non-wavefront instantiation of the tile, whatever its DA / RA forms
    name = f"16sw16_pass_kernelILi{args.R}ELi{args.G}ELb{args.bin}ELi0ELi512ELi{U}ELb0ELb"
    lines = sass.split("\n")
    st = next((i for i, l in enumerate(lines) if "Function :" in l and name in l), None)
    if st is None:
        sys.exit(f"no instantiation matching {name}* in the cubin")
    en = next((i for i in range(st + 1, len(lines)) if "Function :" in lines[i]), len(lines))
    ins = []
    for l in lines[st:en]:
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)(.*?);", l)
        if m:
            ins.append((int(m.group(1), 16), m.group(3), m.group(4)))
    # the column loop: the innermost backward branch whose body holds the rows
    # (at least U*R VIMNMX3)
    best = None
    for a, op, rest in ins:
        if op.startswith("BRA"):
            t = re.search(r"0x([0-9a-f]+)", rest)
            if not t or int(t.group(1), 16) >= a:
                continue
            lo = int(t.group(1), 16)
            nmx = sum(1 for x in ins if lo <= x[0] <= a and x[1].startswith("VIMNMX3"))
            if nmx >= U * args.R and (best is None or a - lo < best[1] - best[0]):
                best = (lo, a)
    body = [x for x in ins if best[0] <= x[0] <= best[1]]
    print(f"loop {best[0]:#x}..{best[1]:#x}", file=sys.stderr)
    # skip the item-claim block: from the first forward branch at the top to its target
    a0, op0, rest0 = body[1]
    if op0.startswith("BRA"):
        skip_to = int(re.search(r"0x([0-9a-f]+)", rest0).group(1), 16)
        body = body[:2] + [x for x in body if x[0] >= skip_to]
        print(f"skip to {skip_to:#x}", file=sys.stderr)
    c = collections.Counter()
    movs = 0
    for _, op, _ in body:
        base = op.split(".")[0]
        if op.startswith("IMAD.MOV") or base == "MOV":
            movs += 1
        if base in ALU:
            c["alu"] += 1
        elif base.startswith(FMA):
            c["fma"] += 1
        elif base in ("LDS",):
            c["lds"] += 1
        elif base == "SHFL":
            c["shfl"] += 1
        else:
            c["other"] += 1
    n = len(body)
    print(f"tile {args.G}x{args.R} bin={args.bin} U={U} {' '.join(args.D + args.xptxas)}: {n} instructions / {U} columns = "
          f"{n / U:.1f} per column; " + ", ".join(f"{k} {v / U:.1f}" for k, v in sorted(c.items())) +
          f"; moves {movs / U:.1f}; ALU-pipe cycles {2 * c['alu'] / U:.1f} vs issue {n / U:.1f} per column")


if __name__ == "__main__":
    main()
