"""The cross-pass wavefront at full size: forced wavefront searches of cfg4 and
of the longest cfg3 queries compared with the stored oracle hashes
(tests/golden/oracle_full_scores.jsonl) -- report tool."""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1702_07195_b200 as sw  # noqa: E402
import sw_inputs as si  # noqa: E402
from tests.report_oracle_hashes import GOLDEN_PATH, fingerprint  # noqa: E402

recs = [json.loads(ln) for ln in open(GOLDEN_PATH) if ln.strip()]
ok = True
for cfg, queries in ((4, [0]), (3, [17, 18, 19])):
    w = si.make_config(cfg, scale=1.0)
    fp = fingerprint(w)
    sw.sw_db_load(w.db.residues, w.db.offsets)
    sw.sw_set_wave(1)
    for qi in queries:
        r = [x for x in recs if x["config"] == cfg and x["query"] == qi and x["workload_fp"] == fp][0]
        got = sw.sw_search(w.queries[qi], w.matrix, w.gap_open, w.gap_extend)
        st = sw.sw_last_stats()
        h = hashlib.sha256(np.ascontiguousarray(got.astype("<i4")).tobytes()).hexdigest()
        good = h == r["sha256_int32"]
        ok &= good
        print(json.dumps({"config": cfg, "query": qi, "wave": st["wave"], "tile": [st["G"], st["R"]],
                          "passes": st["passes"], "flagged": st["flagged"], "equal_to_oracle": good}), flush=True)
    sw.sw_set_wave(0)
sys.exit(0 if ok else 1)
