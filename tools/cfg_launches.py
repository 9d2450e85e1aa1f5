"""Launch list of configs[CFG] searches (default cfg0) (run under ncu --metrics gpu__time_duration.sum):
where the non-pass-kernel time of a small search goes.  Without ncu it prints
the single-search and back-to-back event times and the pass-kernel time."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import sw_inputs as si
import paper_1702_07195_b200 as sw

CFG = int(os.environ.get("CFG", "0"))
w = si.make_config(CFG)
sw.sw_db_load(w.db.residues, w.db.offsets)
d = torch.empty(w.db.count, dtype=torch.int32, device="cuda")
st = torch.cuda.Stream()
q = w.queries[0]
for _ in range(3):
    sw.sw_search_dev(q, w.matrix, w.gap_open, w.gap_extend, d, st)
st.synchronize()
one, pk = [], []
for _ in range(int(os.environ.get("REPS", "5"))):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    sw.sw_search_dev(q, w.matrix, w.gap_open, w.gap_extend, d, st)
    e1.record(st)
    st.synchronize()
    one.append(e0.elapsed_time(e1))
    pk.append(sw.sw_last_timing()["pass_kernels_ms"])
n = int(os.environ.get("B2B", "50"))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(n):
    sw.sw_search_dev(q, w.matrix, w.gap_open, w.gap_extend, d, st)
e1.record(st)
st.synchronize()
print(json.dumps({"single_ms": float(np.median(one)), "b2b_ms": e0.elapsed_time(e1) / n,
                  "pass_ms": float(np.median(pk)), "stats": sw.sw_last_stats()}, default=str))
