"""Run BASELINE.json configurations on one GPU: device GCUPS per query, flag
statistics and a sampled oracle parity check (dev / report tool).  Every
timed region is sampled by bench.ClockSampler (nvidia-smi SM clock and
throttle reasons); each line carries its clocks.

    python tests/report_configs.py 0 1 2 3 4 [--scale S] [--sample N] [--reps K]

Prints one JSON line per (config, query).
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
from bench import ClockSampler, cpu_model  # noqa: E402
import paper_1702_07195_b200 as sw  # noqa: E402
import sw_inputs as si  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", type=int, default=[0, 1])
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--sample", type=int, default=1500)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--queries", type=str, default="")
    ap.add_argument("--batch", action="store_true", help="also time sw_search_batch over all queries")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    cores = os.cpu_count()
    for c in args.configs:
        t0 = time.time()
        w = si.make_config(c, scale=args.scale)
        t1 = time.time()
        sw.sw_db_load(w.db.residues, w.db.offsets)
        t2 = time.time()
        d = torch.empty(w.db.count, dtype=torch.int32, device="cuda")
        st = torch.cuda.Stream()
        L = w.db.lengths()
        rng = np.random.default_rng(17 + c)
        qsel = range(len(w.queries)) if not args.queries else [int(x) for x in args.queries.split(",")]
        for qi in qsel:
            q = w.queries[qi]
            sw.sw_search_dev(q, w.matrix, w.gap_open, w.gap_extend, d, st)
            st.synchronize()
            clk = ClockSampler(0)
            clk.start()
            time.sleep(0.3)
            times, pk = [], []
            for _ in range(args.reps):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(st)
                sw.sw_search_dev(q, w.matrix, w.gap_open, w.gap_extend, d, st)
                e1.record(st)
                st.synchronize()
                times.append(e0.elapsed_time(e1))
                pk.append(sw.sw_last_timing()["pass_kernels_ms"])
            # back to back (throughput; no host round trip between searches)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(args.reps):
                sw.sw_search_dev(q, w.matrix, w.gap_open, w.gap_extend, d, st)
            e1.record(st)
            st.synchronize()
            ms_b2b = e0.elapsed_time(e1) / args.reps
            clocks = clk.stop()
            ms = float(np.median(times))
            tm = {"pass_kernels_ms": float(np.median(pk))}
            stats = sw.sw_last_stats()
            got = d.cpu().numpy()
            # sampled parity: random sample + the longest sequences + planted copies
            idx = [rng.choice(w.db.count, min(args.sample, w.db.count), replace=False), np.argsort(-L)[:20]]
            if w.planted is not None:
                idx.append(w.planted)
            idx = np.unique(np.concatenate(idx))
            # high-scoring extremes: the top-50 GPU scores
            idx = np.unique(np.concatenate([idx, np.argsort(-got)[:50]]))
            tq = time.time()
            exp = oracle.batch(q, w.db.residues, w.db.offsets, w.matrix, w.gap_open, w.gap_extend, idx=idx,
                               threads=cores)
            tq = time.time() - tq
            bad = int((got[idx] != exp).sum())
            cells = len(q) * w.db.total_residues
            print(json.dumps({
                "config": c, "query": qi, "m": len(q), "db_seqs": w.db.count, "db_residues": w.db.total_residues,
                "gen_s": round(t1 - t0, 1), "load_s": round(t2 - t1, 1), "ms": round(ms, 3),
                "gcups": round(cells / (ms * 1e6), 1),
                "gcups_back_to_back": round(cells / (ms_b2b * 1e6), 1),
                "pass_kernel_gcups": round(cells / (tm["pass_kernels_ms"] * 1e6), 1),
                "tile": [stats["G"], stats["R"]], "passes": stats["passes"], "flagged": stats["flagged"],
                "cells32": stats["cells32"], "parity_checked": int(idx.size), "parity_mismatches": bad,
                "oracle_s": round(tq, 1), "max_score": int(got.max()), "reps": args.reps,
                "ms_min_max": [round(min(times), 3), round(max(times), 3)], "clocks": clocks,
                "oracle_cores": cores, "cpu_model": cpu_model()}), flush=True)
            assert bad == 0, f"config {c} query {qi}: {bad} mismatches"
        if args.batch and len(w.queries) > 1:
            dd = torch.empty(len(w.queries) * w.db.count, dtype=torch.int32, device="cuda")
            sw.sw_search_batch_dev(w.queries, w.matrix, w.gap_open, w.gap_extend, dd, st)
            st.synchronize()
            clk = ClockSampler(0)
            clk.start()
            time.sleep(0.3)
            times = []
            for _ in range(max(3, args.reps // 2)):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(st)
                sw.sw_search_batch_dev(w.queries, w.matrix, w.gap_open, w.gap_extend, dd, st)
                e1.record(st)
                st.synchronize()
                times.append(e0.elapsed_time(e1))
            clocks = clk.stop()
            ms = float(np.median(times))
            allsc = dd.view(len(w.queries), w.db.count).cpu().numpy()
            # parity of the batch against the single-query path on every query (exact)
            mism = 0
            for qi, q in enumerate(w.queries):
                sw.sw_search_dev(q, w.matrix, w.gap_open, w.gap_extend, d, st)
                st.synchronize()
                mism += int((d.cpu().numpy() != allsc[qi]).sum())
            cells = sum(len(q) for q in w.queries) * w.db.total_residues
            print(json.dumps({"config": c, "batch_queries": len(w.queries), "ms": round(ms, 1),
                              "gcups": round(cells / (ms * 1e6), 1), "batch_vs_single_mismatches": mism,
                              "reps": len(times), "ms_min_max": [round(min(times), 1), round(max(times), 1)],
                              "clocks": clocks}), flush=True)
            assert mism == 0


if __name__ == "__main__":
    main()
