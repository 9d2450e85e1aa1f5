"""Print the main loop (largest backward branch) of a SASS dump, optionally only
some opcodes (dev tool): python tools/sass_loop.py file.sass [--mix]"""
import re, sys, subprocess, os
lines = open(sys.argv[1]).read().splitlines()
ins = []
for ln in lines:
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", ln)
    if m: ins.append((int(m.group(1), 16), m.group(2).strip()))
best = None
for a, t in ins:
    m = re.search(r"BRA (?:\S+ )?0x([0-9a-f]+)", t)
    if m:
        tgt = int(m.group(1), 16)
        if tgt < a and (best is None or a - tgt > best[1] - best[0]): best = (tgt, a)
lo, hi = best
print(f"loop 0x{lo:x}..0x{hi:x}: {(hi - lo) // 16 + 1} instructions")
if "--mix" in sys.argv:
    here = os.path.dirname(os.path.abspath(__file__))
    subprocess.run([sys.executable, os.path.join(here, "sass_mix.py"), sys.argv[1], f"{lo:x}", f"{hi + 16:x}"])
else:
    for a, t in ins:
        if lo <= a <= hi: print(f"{a:05x} {t}")
