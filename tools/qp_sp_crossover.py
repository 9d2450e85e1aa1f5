"""QP/SP crossover in the real pass kernel (PAPER.md:165,
212): every configs[3] query (20 lengths, 144..5478) against the configs[3]
database, with the query profile (QPM 0) and the score profile (QPM 1), each
on its automatically chosen tile and on common tiles; clocks sampled; a
sampled oracle check of every SP search.  (dev/report tool, 1 GPU)

    python tools/qp_sp_crossover.py [--scale S] > profiles/r02_qp_sp_crossover.jsonl
"""
import argparse
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


def timed(q, d, st, reps):
    sw.sw_search_dev(q, si.BLOSUM62, 10, 2, d, st)
    st.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        sw.sw_search_dev(q, si.BLOSUM62, 10, 2, d, st)
        e1.record(st)
        st.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)), sw.sw_last_timing()["pass_kernels_ms"], sw.sw_last_stats()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--queries", default="")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    w = si.config3(scale=args.scale)
    sw.sw_db_load(w.db.residues, w.db.offsets)
    d = torch.empty(w.db.count, dtype=torch.int32, device="cuda")
    st = torch.cuda.Stream()
    rng = np.random.default_rng(165)
    sample = rng.choice(w.db.count, min(300, w.db.count), replace=False)
    qsel = range(len(w.queries)) if not args.queries else [int(x) for x in args.queries.split(",")]
    for qi in qsel:
        q = w.queries[qi]
        cells = len(q) * w.db.total_residues
        rec = {"query": qi, "m": len(q)}
        clk = ClockSampler(0)
        clk.start()
        time.sleep(0.2)
        for name, prof, tile in [("qp_auto", 1, (0, 0)), ("sp_auto", 2, (0, 0)),
                                 ("qp_16x16", 1, (16, 16)), ("sp_16x16", 2, (16, 16)),
                                 ("qp_32x16", 1, (32, 16)), ("sp_32x16", 2, (32, 16)),
                                 ("qp_32x20", 1, (32, 20)), ("sp_32x20", 2, (32, 20))]:
            sw.sw_set_profile(prof)
            sw.sw_set_tile(*tile)
            ms, pms, s = timed(q, d, st, args.reps)
            rec[name] = {"tile": [s["G"], s["R"]], "passes": s["passes"], "ms": round(ms, 3),
                         "gcups": round(cells / (ms * 1e6), 1), "pass_gcups": round(cells / (pms * 1e6), 1)}
            if prof == 2 and tile == (0, 0):
                got = d.cpu().numpy()
                exp = oracle.batch(q, w.db.residues, w.db.offsets, w.matrix, w.gap_open, w.gap_extend,
                                   idx=sample, threads=os.cpu_count())
                rec["sp_sample_mismatches"] = int((got[sample] != exp).sum())
        rec["clocks"] = clk.stop()
        rec["sp_vs_qp_auto"] = round(rec["sp_auto"]["gcups"] / rec["qp_auto"]["gcups"], 4)
        print(json.dumps(rec), flush=True)
    sw.sw_set_profile(0)
    sw.sw_set_tile(0)


if __name__ == "__main__":
    main()
