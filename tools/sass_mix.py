"""Opcode / pipe mix of a SASS region (dev tool).
usage: python tools/sass_mix.py file.sass [start_addr_hex end_addr_hex]"""
import re, sys, collections
ALU = {"VIADDMNMX", "VIMNMX", "VIMNMX3", "PRMT", "LOP3", "IADD3", "ISETP", "SEL", "SHF", "LEA", "IABS", "VIADD",
       "FMNMX", "PLOP3", "MOV", "LOP", "CSET", "ICMP", "IMNMX", "BMSK", "SGXT", "FSEL", "P2R", "R2P", "POPC", "FLO", "BREV"}
FMA = {"IMAD", "FFMA", "FMUL", "FADD", "IDP", "IMUL"}
LSU = {"LDS", "STS", "LDG", "STG", "LDL", "STL", "SHFL", "ATOMG", "ATOMS", "RED", "LD", "ST", "LDC", "ATOM"}
txt = open(sys.argv[1]).read().splitlines()
lo = int(sys.argv[2], 16) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else 1 << 60
cnt = collections.Counter(); pipe = collections.Counter()
for ln in txt:
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.x]+)?", ln)
    if not m: continue
    a = int(m.group(1), 16)
    if not (lo <= a < hi): continue
    op = m.group(3); full = op + (m.group(4) or "")
    cnt[full] += 1
    if op == "VIADD": p = "alu?"
    elif op in ALU: p = "alu"
    elif op in FMA: p = "fma"
    elif op in LSU: p = "lsu/mio"
    else: p = "other"
    pipe[p] += 1
for k, v in cnt.most_common(40): print(f"{v:6d} {k}")
print(dict(pipe))
