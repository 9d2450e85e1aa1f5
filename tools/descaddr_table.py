"""From the two calibrations (SW_DESCADDR=0 / =1 builds of tools/calibrate_tiles.py),
pick per (tile, pass kind) the faster descriptor-address form (>= 0.5% faster) and
write the kDescFromQp table and the chosen variants' efficiencies into kernels.cu;
the merged record goes to profiles/r02b_descaddr_calibration.jsonl (dev tool).

    python tools/descaddr_table.py gpurun_out/calib_da0.jsonl gpurun_out/calib_da1.jsonl
"""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
K = os.path.join(ROOT, "paper_1702_07195_b200", "csrc", "kernels.cu")
MIN_GAIN = 1.005


def load(p):
    return {(d["G"], d["R"]): d for d in (json.loads(l) for l in open(p) if l.startswith("{"))}


def main():
    a, b = load(sys.argv[1]), load(sys.argv[2])
    picks, eff, rec = [], {}, []
    for key in sorted(a):
        if key not in b:
            continue
        G, R = key
        e0 = b[key]["eff0"] >= a[key]["eff0"] * MIN_GAIN
        e1 = b[key]["eff1"] >= a[key]["eff1"] * MIN_GAIN
        if e0:
            picks.append((G, R, False))
        if e1:
            picks.append((G, R, True))
        eff[key] = (b[key]["eff0"] if e0 else a[key]["eff0"], b[key]["eff1"] if e1 else a[key]["eff1"])
        rec.append({"G": G, "R": R, "eff0_base": a[key]["eff0"], "eff0_qp": b[key]["eff0"], "pick0": int(e0),
                    "eff1_base": a[key]["eff1"], "eff1_qp": b[key]["eff1"], "pick1": int(e1)})
    with open(os.path.join(ROOT, "profiles", "r02b_descaddr_calibration.jsonl"), "w") as f:
        for r in rec:
            f.write(json.dumps(r) + "\n")
    s = open(K).read()
    body = "".join("    {%d, %d, %s},\n" % (G, R, "true" if bn else "false") for G, R, bn in picks) or \
        "    {0, 0, false},\n"
    s = re.sub(r"(constexpr DescPick kDescFromQp\[\] = \{\n)(.*?)(\};)", lambda m: m.group(1) + body + m.group(3),
               s, flags=re.S)
    def row(m):
        G, R = int(m.group(1)), int(m.group(2))
        if (G, R) not in eff:
            return m.group(0)
        return "{%d, %d, %.1ff, %.1ff}" % (G, R, eff[(G, R)][0], eff[(G, R)][1])
    i = s.index("const TileEff kTileEff[] = {")
    j = s.index("};", i)
    s = s[:i] + re.sub(r"\{(\d+), (\d+), ([\d.]+)f, ([\d.]+)f\}", row, s[i:j]) + s[j:]
    open(K, "w").write(s)
    print(f"{len(picks)} instantiations take the s_qp form")
    for r in rec:
        print(r)


if __name__ == "__main__":
    main()
