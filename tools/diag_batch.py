import sys, os, json
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import sw_inputs as si, oracle
import paper_1702_07195_b200 as sw
scale = float(sys.argv[1])
w = si.config3(scale=scale)
sw.sw_db_load(w.db.residues, w.db.offsets)
qs = w.queries
got = sw.sw_search_batch(qs, w.matrix, 10, 2)
L = w.db.lengths()
for qi, q in enumerate(qs):
    single = sw.sw_search(q, w.matrix, 10, 2)
    bad = np.nonzero(single != got[qi])[0]
    if bad.size:
        ex = oracle.batch(q, w.db.residues, w.db.offsets, w.matrix, 10, 2, idx=bad[:5])
        print(json.dumps({"q": qi, "m": len(q), "nbad": int(bad.size), "idx": bad[:5].tolist(), "len": L[bad[:5]].tolist(),
                          "single": single[bad[:5]].tolist(), "batch": got[qi][bad[:5]].tolist(), "oracle": ex.tolist()}))
print("done")
