"""Summarise an ncu launch list (gpu__time_duration.sum CSV) per kernel (dev tool).

    python tools/launch_summary.py launches.csv "header comment" > profiles/rNN_launches_summary.tsv
"""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
ix = {n: j for j, n in enumerate(rows[i])}
agg = collections.OrderedDict()
scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
for r in rows[i + 1:]:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    v = float(r[ix["Metric Value"]].replace(",", "")) * scale.get(r[ix["Metric Unit"]], 1.0)
    a = agg.setdefault(r[ix["Kernel Name"]], [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(v[1] for v in agg.values())
print(f"# {sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]}")
print("# cold-cache and serialised: compare SHARES, not absolute times")
print("kernel\tlaunches\ttotal_ms\tshare")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:80]}\t{n}\t{t:.3f}\t{t / tot:.4f}")
