"""Full-size oracle reference values for exhaustive GPU parity (test
infrastructure; calls only oracle/ and the seeded generators).

For every (config, query) of BASELINE.json at full size, runs the CPU oracle
over the WHOLE database and appends one JSON line to
tests/golden/oracle_full_scores.jsonl with the SHA-256 of the int32 score
vector (little endian, original database order), its sum and maximum, and the
oracle's top-10.  tests/test_gpu_full_hashes.py compares the CUDA path against
these lines, so every score of every configuration is checked bit-exactly
without storing gigabytes of scores.

    python tests/report_oracle_hashes.py [--configs 0,1,4,2,3] [--threads N]

Lines already present (same config, query and generator fingerprint) are
skipped, so the script can be resumed.
"""
import argparse
import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import sw_inputs as si  # noqa: E402

GOLDEN_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "oracle_full_scores.jsonl")
OUT = GOLDEN_PATH


def fingerprint(w) -> str:
    """Hash of the generated workload (database and queries): a changed
    generator invalidates the stored oracle values instead of failing obscurely."""
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(w.db.offsets).tobytes())
    h.update(hashlib.sha256(np.ascontiguousarray(w.db.residues).tobytes()).digest())
    for q in w.queries:
        h.update(np.ascontiguousarray(q).tobytes())
    return h.hexdigest()[:32]


def score_record(cfg: int, qi: int, w, scores: np.ndarray, seconds: float) -> dict:
    s32 = np.ascontiguousarray(scores.astype("<i4"))
    idx, top = oracle.topk(scores, 10)
    return {"config": cfg, "query": qi, "m": int(len(w.queries[qi])), "count": int(w.db.count),
            "residues": int(w.db.total_residues), "workload_fp": fingerprint(w),
            "sha256_int32": hashlib.sha256(s32.tobytes()).hexdigest(), "sum": int(scores.sum()),
            "max": int(scores.max()), "top10_idx": idx.tolist(), "top10_score": top.tolist(),
            "oracle_seconds": round(seconds, 1), "numpy": np.__version__}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="0,1,4,2,3")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--queries", default="", help="query range for multi-query configs, e.g. 10-19")
    ap.add_argument("--out", default=OUT)
    args = ap.parse_args()
    out = args.out
    qsel = None
    if args.queries:   # e.g. "17-19,7-9"
        qsel = set()
        for part in args.queries.split(","):
            a, _, b = part.partition("-")
            qsel.update(range(int(a), int(b or a) + 1))
    done = set()
    if os.path.exists(out):
        for ln in open(out):
            if ln.strip():
                r = json.loads(ln)
                done.add((r["config"], r["query"], r["workload_fp"]))
    for cfg in [int(c) for c in args.configs.split(",") if c]:
        w = si.make_config(cfg, scale=1.0)
        fp = fingerprint(w)
        for qi, q in enumerate(w.queries):
            if (cfg, qi, fp) in done or (qsel is not None and len(w.queries) > 1 and qi not in qsel):
                continue
            t0 = time.time()
            sc = oracle.batch(q, w.db.residues, w.db.offsets, w.matrix, w.gap_open, w.gap_extend,
                              threads=args.threads)
            rec = score_record(cfg, qi, w, sc, time.time() - t0)
            with open(out, "a") as f:
                f.write(json.dumps(rec) + "\n")
            print(json.dumps({k: rec[k] for k in ("config", "query", "m", "max", "oracle_seconds")}), flush=True)


if __name__ == "__main__":
    main()
