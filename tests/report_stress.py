"""Randomised stress run of the CUDA path against the oracle (report tool;
`-m gpu` covers fixed cases, this one draws many more).

Each trial draws a database (count, length mix, alphabet use), a query or a
query pair, a scoring matrix (BLOSUM62, random symmetric, random asymmetric,
extreme int8), gap penalties (including 0 and very large), a tile (default or
any compiled one: throughput, latency or score-profile tiles), the cross-pass
wavefront (off / auto / forced), the latency-tile mode, the substitution
profile (query / score profile), rows mode (never / auto / on request), and a path (resident single, resident query
pair, streamed), then compares every score and the top-k (k up to 200: both
sorting paths) with the oracle.

    python tests/report_stress.py [--seconds 600] [--seed 1]

Prints one JSON line per failure and a summary line; exit status 1 on any
mismatch.
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


def draw_matrix(rng):
    kind = int(rng.integers(0, 4))
    if kind == 0:
        return "blosum62", si.BLOSUM62
    if kind == 1:
        return "sym", si.random_symmetric_matrix(rng)
    if kind == 2:
        return "asym", rng.integers(-6, 12, (24, 24)).astype(np.int8)
    m = rng.integers(-128, 128, (24, 24)).astype(np.int8)
    return "int8", m


def draw_gaps(rng):
    kind = int(rng.integers(0, 5))
    if kind == 0:
        return 10, 2
    if kind == 1:
        return int(rng.integers(0, 3)), int(rng.integers(0, 3))
    if kind == 2:
        return int(rng.integers(0, 20)), int(rng.integers(0, 8))
    if kind == 3:
        return int(rng.integers(10000, 40000)), int(rng.integers(0, 40000))
    return int(rng.integers(0, 200)), 0


def draw_db(rng):
    count = int(rng.integers(1, 3000))
    mix = int(rng.integers(0, 3))
    if mix == 0:
        lens = rng.integers(0, 400, count)
    elif mix == 1:
        lens = np.clip(np.rint(rng.lognormal(np.log(150), 0.76, count)), 0, 5000).astype(np.int64)
    else:
        lens = rng.integers(0, 40, count)
        lens[rng.integers(0, count, max(1, count // 200))] = rng.integers(2000, 12000)
    alpha = int(rng.choice([20, 24, 2]))
    seqs = [rng.integers(0, alpha, int(L)).astype(np.uint8) for L in lens]
    if rng.random() < 0.3:   # planted near-copies of a W-rich block (saturating scores)
        block = np.full(int(rng.integers(1500, 4000)), 17, np.uint8)
        for _ in range(int(rng.integers(1, 6))):
            seqs[int(rng.integers(0, count))] = block.copy()
    return si.database_from_list(seqs), alpha


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=600)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--trials", type=int, default=0, help="stop after this many trials (0: time only)")
    ap.add_argument("--verbose", action="store_true", help="print every trial's parameters before running it")
    ap.add_argument("--only", type=int, default=0, help="draw every trial but run only this one")
    ap.add_argument("--start", type=int, default=0, help="draw every trial but run only trials >= start")
    ap.add_argument("--dump", default="", help="with --only: save the trial's inputs to this .npz")
    args = ap.parse_args()
    import torch
    torch.cuda.set_device(0)
    rng = np.random.default_rng(args.seed)
    tiles = [(G, R) for G in (8, 16, 32) for R in range(1, 33)
             if sw.sw_tile_supported(G, R) or sw.sw_tile_supported(G, R, lat=True) or sw.sw_tile_supported(G, R, sp=True)]
    t_end = time.time() + args.seconds
    trials = fails = cells = 0
    while time.time() < t_end and (args.trials == 0 or trials < args.trials):
        trials += 1
        db, alpha = draw_db(rng)
        mname, M = draw_matrix(rng)
        go, ge = draw_gaps(rng)
        m = int(rng.integers(1, 3500))
        q = rng.integers(0, alpha, m).astype(np.uint8)
        if rng.random() < 0.2:
            q[: min(m, 3000)] = 17                       # W-rich query: saturating scores
        path = ["single", "single", "pair", "streamed"][int(rng.integers(0, 4))]
        chunk = int(rng.integers(1, 64)) * 4096
        q2 = rng.integers(0, alpha, int(rng.integers(1, 3500))).astype(np.uint8)
        k = int(min(db.count, rng.integers(1, 40) if rng.random() < 0.7 else rng.integers(33, 200)))
        tile = (0, 0) if rng.random() < 0.5 else tiles[int(rng.integers(0, len(tiles)))]
        sw.sw_set_tile(*tile)
        wave = int(rng.choice([-1, 0, 1, 1]))   # cross-pass wavefront off / auto / forced
        sw.sw_set_wave(wave)
        lat = int(rng.choice([-1, 0, 1]))       # latency tiles never / auto / always
        sw.sw_set_latency_mode(lat)
        prof = int(rng.choice([0, 1, 2]))       # substitution scores: auto / query profile / score profile
        sw.sw_set_profile(prof)
        rows = int(rng.choice([-1, 0, 0, 1]))   # rows mode for the long items: never / auto / on request
        sw.sw_set_rows_mode(rows)
        if (args.only and trials != args.only) or trials < args.start:
            continue
        if args.dump:
            np.savez(args.dump, res=db.residues, offs=db.offsets, q=q, q2=q2, M=M, go=go, ge=ge, path=path,
                     tile=np.array(tile), wave=wave, lat=lat, prof=prof, chunk=chunk, k=k)
        if args.verbose:
            print(json.dumps({"trial": trials, "count": db.count, "max_len": int(db.lengths().max(initial=0)),
                              "alpha": alpha, "matrix": mname, "gaps": [go, ge], "m": m, "path": path,
                              "tile": tile, "wave": wave, "lat": lat, "profile": prof, "rows": rows}), flush=True)
        try:
            if path == "streamed":
                sw.sw_db_load_streamed(db.residues, db.offsets, chunk)
            else:
                sw.sw_db_load(db.residues, db.offsets)
            if path == "pair":
                got = sw.sw_search_batch([q, q2], M, go, ge)
                outs = [(q, got[0]), (q2, got[1])]
            else:
                outs = [(q, sw.sw_search(q, M, go, ge))]
            ok = True
            for qq, g in outs:
                exp = oracle.batch(qq, db.residues, db.offsets, M, go, ge)
                cells += len(qq) * db.total_residues
                bad = np.nonzero(g != exp)[0]
                if bad.size:
                    ok = False
                    print(json.dumps({"trial": trials, "path": path, "tile": tile, "wave": wave, "lat": lat,
                                      "profile": prof, "rows": rows, "matrix": mname, "gaps": [go, ge],
                                      "m": len(qq), "count": db.count, "mismatches": int(bad.size),
                                      "first": bad[:5].tolist(), "got": g[bad[:5]].tolist(),
                                      "exp": exp[bad[:5]].tolist()}), flush=True)
            if ok and path != "pair":
                idx, sc = sw.sw_topk(k)
                eidx, esc = oracle.topk(outs[0][1], k)
                if not ((idx == eidx).all() and (sc == esc).all()):
                    ok = False
                    print(json.dumps({"trial": trials, "path": path, "topk_mismatch": k}), flush=True)
            fails += 0 if ok else 1
        except sw.SWError as e:
            fails += 1
            print(json.dumps({"trial": trials, "path": path, "tile": tile, "wave": wave, "lat": lat, "profile": prof,
                              "m": m, "count": db.count, "error": str(e)}), flush=True)
            if e.code == sw.SW_ECUDA:   # a device fault is sticky: stop at the first one
                break
    sw.sw_set_tile(0)
    sw.sw_set_wave(0)
    sw.sw_set_latency_mode(0)
    sw.sw_set_profile(0)
    sw.sw_set_rows_mode(0)
    print(json.dumps({"trials": trials, "failures": fails, "cells": cells, "seconds": args.seconds}), flush=True)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
