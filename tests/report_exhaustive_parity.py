"""Exhaustive parity at full BASELINE.json sizes: every database score of the
CUDA path (through the C-ABI, default tile choice = the bench's launch
configuration) against the CPU oracle on the whole database, plus the top-10
(report tool; the pytest suite samples instead because this takes minutes).

    python tests/report_exhaustive_parity.py [--configs 0,1,2,4] [--cfg3-queries 0,1] [--streamed]

Prints one JSON line per (config, query, path) with the mismatch count and the
oracle's own full-database time and GCUPS on this host.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_1702_07195_b200 as sw  # noqa: E402
import sw_inputs as si  # noqa: E402


def check(label, got, exp, extra):
    bad = np.nonzero(got != exp)[0]
    gi, gs = oracle.topk(got, 10)
    ei, es = oracle.topk(exp, 10)
    line = {"case": label, "sequences": int(exp.size), "mismatches": int(bad.size),
            "first_mismatches": bad[:5].tolist(), "top10_equal": bool((gi == ei).all() and (gs == es).all()),
            "max_score": int(exp.max())}
    line.update(extra)
    print(json.dumps(line), flush=True)
    return bad.size == 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="0,1,2,4")
    ap.add_argument("--cfg3-queries", default="")
    ap.add_argument("--streamed", action="store_true", help="also the out-of-core path on cfg2")
    args = ap.parse_args()
    cores = os.cpu_count() or 1
    ok = True
    cfgs = [int(c) for c in args.configs.split(",") if c]
    if args.cfg3_queries:
        cfgs.append(3)
    for c in cfgs:
        w = si.make_config(c, scale=1.0)
        sw.sw_db_load(w.db.residues, w.db.offsets)
        qsel = [int(x) for x in args.cfg3_queries.split(",")] if c == 3 else [0]
        for qi in qsel:
            q = w.queries[qi]
            got = sw.sw_search(q, w.matrix, w.gap_open, w.gap_extend)
            st = sw.sw_last_stats()
            t0 = time.time()
            exp = oracle.batch(q, w.db.residues, w.db.offsets, w.matrix, w.gap_open, w.gap_extend, threads=cores)
            dt = time.time() - t0
            cells = len(q) * w.db.total_residues
            ok &= check(f"cfg{c} q{qi} resident", got, exp,
                        {"m": len(q), "residues": w.db.total_residues, "tile": [st["G"], st["R"]],
                         "passes": st["passes"], "flagged": st["flagged"], "oracle_s": round(dt, 1),
                         "oracle_gcups": round(cells / dt / 1e9, 2), "oracle_threads": cores})
            if c == 2 and args.streamed:
                sw.sw_db_load_streamed(w.db.residues, w.db.offsets, 256 << 20)
                gs = sw.sw_search(q, w.matrix, w.gap_open, w.gap_extend)
                ok &= check(f"cfg{c} q{qi} streamed 256 MiB chunks", gs, exp, {"m": len(q)})
                sw.sw_db_load(w.db.residues, w.db.offsets)
        if c == 3 and len(qsel) >= 2:
            pair = [w.queries[qsel[0]], w.queries[qsel[1]]]
            allsc = sw.sw_search_batch(pair, w.matrix, w.gap_open, w.gap_extend)
            for k, qi in enumerate(qsel[:2]):
                exp = oracle.batch(w.queries[qi], w.db.residues, w.db.offsets, w.matrix, w.gap_open,
                                   w.gap_extend, threads=cores)
                ok &= check(f"cfg3 q{qi} query-pair path", allsc[k], exp, {"m": len(w.queries[qi])})
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
