"""Measure the intrinsic throughput of every compiled (mode, G, R) tile: a
query of exactly G*R residues (one full pass, no phantom rows) against the
cfg1 database (dev tool; feeds the tile-choice table in csrc/api.cu)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import sw_inputs as si
import paper_1702_07195_b200 as sw

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 0.3
modes = [0]
w = si.config1(scale=scale)
sw.sw_db_load(w.db.residues, w.db.offsets)
d = torch.empty(w.db.count, dtype=torch.int32, device='cuda')
st = torch.cuda.Stream()
rng = si.rng_for(77, 2)
out = []
def timed(q):
    for _ in range(2):
        sw.sw_search_dev(q, w.matrix, 10, 2, d, st)
    st.synchronize()
    ts = []
    for _ in range(3):
        sw.sw_search_dev(q, w.matrix, 10, 2, d, st)
        ts.append(sw.sw_last_timing()["pass_kernels_ms"])
    return float(np.median(ts))

for G in (8, 16, 32):
    for R in range(1, 33):
        if not sw.sw_tile_supported(G, R):
            continue
        sw.sw_set_tile(G, R)
        q1 = si.rr_residues(rng, G * R)          # one pass (no boundary input)
        q2 = si.rr_residues(rng, 2 * G * R)      # two passes: the second reads the boundary
        t1, t2 = timed(q1), timed(q2)
        cells_pass = G * R * w.db.total_residues
        r = {"G": G, "R": R, "eff0": round(cells_pass / (t1 * 1e6), 1),
             "eff1": round(cells_pass / (max(t2 - t1, 1e-3) * 1e6), 1)}
        out.append(r)
        print(json.dumps(r), flush=True)
sw.sw_set_tile(0)
