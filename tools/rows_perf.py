"""Rows mode (long database sequences along the rows) against the ordinary
path: whole-search time on databases with long sequences (dev/report tool).

    python tools/rows_perf.py > profiles/r02_rows_mode.jsonl
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1702_07195_b200 as sw  # noqa: E402
import sw_inputs as si  # noqa: E402
from bench import ClockSampler  # noqa: E402


def timed(q, d, st, reps=10):
    for _ in range(2):
        sw.sw_search_dev(q, si.BLOSUM62, 10, 2, d, st)
    st.synchronize()
    ts, pk = [], []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        sw.sw_search_dev(q, si.BLOSUM62, 10, 2, d, st)
        e1.record(st)
        st.synchronize()
        ts.append(e0.elapsed_time(e1))
        pk.append(sw.sw_last_timing()["pass_kernels_ms"])
    return float(np.median(ts)), float(np.median(pk))


def main():
    torch.cuda.set_device(0)
    st = torch.cuda.Stream()
    rng = np.random.default_rng(77)
    cases = [("cfg0", si.config0().db, [si.config0().queries[0]])]
    cases.append(("one 35k", si.database_from_list([si.rr_residues(rng, 35000)]),
                  [si.rr_residues(rng, L) for L in (144, 1000)]))
    cases.append(("20 x 20-35k", si.database_from_list([si.rr_residues(rng, int(L)) for L in rng.integers(20000, 35001, 20)]),
                  [si.rr_residues(rng, L) for L in (144, 1000, 5478)]))
    cases.append(("cfg0-like 100k", si.config0(scale=10).db, [si.rr_residues(rng, L) for L in (144, 464)]))
    cases.append(("2000 x 5-35k", si.database_from_list([si.rr_residues(rng, int(L)) for L in rng.integers(5000, 35001, 2000)]),
                  [si.rr_residues(rng, L) for L in (144, 1000)]))
    clk = ClockSampler(0)
    clk.start()
    for name, db, qs in cases:
        sw.sw_db_load(db.residues, db.offsets)
        d = torch.empty(db.count, dtype=torch.int32, device="cuda")
        sample = rng.choice(db.count, min(200, db.count), replace=False)
        for q in qs:
            cells = len(q) * db.total_residues
            rec = {"db": name, "seqs": db.count, "residues": db.total_residues, "m": len(q)}
            for mode in (-1, 1, 0):
                sw.sw_set_rows_mode(mode)
                ms, pms = timed(q, d, st, reps=5 if cells > 5e10 else 10)
                s = sw.sw_last_stats()
                got = d.cpu().numpy()
                exp = oracle.batch(q, db.residues, db.offsets, si.BLOSUM62, 10, 2, idx=sample,
                                   threads=os.cpu_count())
                rec[{-1: "off", 1: "on", 0: "auto"}[mode]] = {
                    "ms": round(ms, 4), "kernels_ms": round(pms, 4), "gcups": round(cells / (ms * 1e6), 1),
                    "rows_pairs": s["rows_pairs"], "tile": [s["G"], s["R"]], "passes": s["passes"],
                    "wave": s["wave"], "lat": s["lat"], "sample_mismatches": int((got[sample] != exp).sum())}
            print(json.dumps(rec), flush=True)
    sw.sw_set_rows_mode(0)
    print(json.dumps({"clocks": clk.stop()}))


if __name__ == "__main__":
    main()
