"""Per-unit timeline of the rows kernel (SW_ROWS_TRACE=1 build, dev tool)."""
import os, sys, json
os.environ["SW_ROWS_TRACE_N"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1702_07195_b200 as sw
import sw_inputs as si
rng = np.random.default_rng(77)
for name, db, m in [("one 35k", si.database_from_list([si.rr_residues(rng, 35000)]), 144),
                    ("one 35k", si.database_from_list([si.rr_residues(rng, 35000)]), 1000),
                    ("cfg0", si.config0().db, 144)]:
    sw.sw_db_load(db.residues, db.offsets)
    sw.sw_set_rows_mode(1)
    q = si.rr_residues(rng, m)
    sw.sw_search(q, si.BLOSUM62, 10, 2)
    sw.sw_search(q, si.BLOSUM62, 10, 2)
    tr = sw.sw_rows_trace(4 * 2000).reshape(-1, 4).astype(np.int64)
    tr = tr[tr[:, 0] > 0]
    t0 = tr[:, 0].min()
    rel = (tr[:, :3] - t0) / 1000.0
    print(json.dumps({"db": name, "m": m, "units": len(tr), "total_us": float(rel[:, 2].max()),
                      "first10": [[round(x, 1) for x in r] + [int(w)] for r, w in zip(rel[:10], tr[:10, 3])],
                      "unit_us_median": float(np.median(rel[:, 2] - rel[:, 1])),
                      "build_us_median": float(np.median(rel[:, 1] - rel[:, 0])),
                      "start_gap_us_median": float(np.median(np.diff(rel[:, 1])))}))
