"""Quick kernel timing on a config (dev tool): GCUPS of sw_search_dev per tile."""
import sys, time, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import sw_inputs as si
import paper_1702_07195_b200 as sw

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
tiles = [tuple(map(int, t.split('x'))) for t in sys.argv[3].split(',')] if len(sys.argv) > 3 else [(0, 0)]
t0 = time.time(); w = si.make_config(cfg, scale=scale); t1 = time.time()
sw.sw_db_load(w.db.residues, w.db.offsets); t2 = time.time()
print(json.dumps({"gen_s": round(t1-t0,2), "load_s": round(t2-t1,2), "count": w.db.count, "residues": w.db.total_residues}), flush=True)
d = torch.empty(w.db.count, dtype=torch.int32, device='cuda')
st = torch.cuda.Stream()
for q in w.queries[:3]:
    for (G, R) in tiles:
        sw.sw_set_tile(G, R)
        for _ in range(2): sw.sw_search_dev(q, si.BLOSUM62, 10, 2, d, st)
        st.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        n = 5
        e0.record(st)
        for _ in range(n): sw.sw_search_dev(q, si.BLOSUM62, 10, 2, d, st)
        e1.record(st); st.synchronize()
        ms = e0.elapsed_time(e1) / n
        stats = sw.sw_last_stats()
        print(json.dumps({"m": len(q), "tile": [stats["G"], stats["R"]], "passes": stats["passes"], "ms": round(ms, 3),
                          "gcups": round(len(q) * w.db.total_residues / (ms * 1e6), 1), "flagged": stats["flagged"], "items": stats["items"]}), flush=True)
if len(sys.argv) > 4 and sys.argv[4] == "batch":
    sw.sw_set_tile(0)
    rng = si.rng_for(1, 9)
    qs = [w.queries[0], si.rr_residues(rng, len(w.queries[0]))]
    dd = torch.empty(2 * w.db.count, dtype=torch.int32, device='cuda')
    for _ in range(2): sw.sw_search_batch_dev(qs, si.BLOSUM62, 10, 2, dd, st)
    st.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(5): sw.sw_search_batch_dev(qs, si.BLOSUM62, 10, 2, dd, st)
    e1.record(st); st.synchronize()
    ms = e0.elapsed_time(e1) / 5
    s = sw.sw_last_stats()
    print(json.dumps({"batch_pair_m": [len(q) for q in qs], "tile": [s["G"], s["R"]], "ms": round(ms, 3),
                      "gcups": round(sum(len(q) for q in qs) * w.db.total_residues / (ms * 1e6), 1)}), flush=True)
