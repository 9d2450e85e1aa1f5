"""CPU checks of the stored full-size oracle values (tests/golden/
oracle_full_scores.jsonl): every line is well formed and consistent, each
config's workload fingerprint matches the current generator, and the cfg0
line is reproduced by running the oracle again (it takes a fraction of a
second), which pins the hashing itself."""
import hashlib
import json
import os

import numpy as np

import oracle
import sw_inputs as si
from tests.report_oracle_hashes import GOLDEN_PATH, fingerprint, score_record

RECS = [json.loads(ln) for ln in open(GOLDEN_PATH) if ln.strip()] if os.path.exists(GOLDEN_PATH) else []


def test_golden_lines_well_formed():
    assert RECS, "no stored oracle values"
    seen = set()
    for r in RECS:
        key = (r["config"], r["query"], r["workload_fp"])
        assert key not in seen, key
        seen.add(key)
        assert len(r["sha256_int32"]) == 64 and r["max"] >= 0 and r["sum"] >= r["max"]
        assert len(r["top10_idx"]) == min(10, r["count"]) and r["top10_score"][0] == r["max"]
        assert r["top10_score"] == sorted(r["top10_score"], reverse=True)


def test_golden_fingerprints_match_the_generator():
    for cfg in sorted({r["config"] for r in RECS} & {0, 1}):   # the quick ones; the GPU test checks all
        fp = fingerprint(si.make_config(cfg, scale=1.0))
        assert any(r["config"] == cfg and r["workload_fp"] == fp for r in RECS), cfg


def test_golden_cfg0_reproduced_by_the_oracle():
    w = si.make_config(0, scale=1.0)
    sc = oracle.batch(w.queries[0], w.db.residues, w.db.offsets, w.matrix, w.gap_open, w.gap_extend)
    rec = score_record(0, 0, w, sc, 0.0)
    stored = [r for r in RECS if r["config"] == 0 and r["workload_fp"] == rec["workload_fp"]]
    assert stored and stored[0]["sha256_int32"] == rec["sha256_int32"]
    assert stored[0]["sha256_int32"] == hashlib.sha256(np.ascontiguousarray(sc.astype("<i4")).tobytes()).hexdigest()
    assert stored[0]["top10_idx"] == rec["top10_idx"]
