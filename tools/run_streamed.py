"""Out-of-core (streamed) database vs resident: GCUPS per chunk budget (dev / report tool)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import sw_inputs as si
import paper_1702_07195_b200 as sw

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
budgets = [int(float(x) * 2**20) for x in (sys.argv[2].split(',') if len(sys.argv) > 2 else ["256", "1024"])]
# latency-tile modes to run (0 auto: chain-bound chunks get a latency tile; -1 never)
lat_modes = [int(x) for x in sys.argv[3].split(',')] if len(sys.argv) > 3 else [0]
w = si.make_config(cfg)
d = torch.empty(w.db.count, dtype=torch.int32, device='cuda')
st = torch.cuda.Stream()
ref = None
for budget in [0] + budgets:
    if budget == 0:
        sw.sw_db_load(w.db.residues, w.db.offsets)
    else:
        sw.sw_db_load_streamed(w.db.residues, w.db.offsets, budget)
    for q, lm in [(q, lm) for q in w.queries[:1] + ([si.rr_residues(si.rng_for(9, 9), 144)] if cfg != 0 else [])
                  for lm in (lat_modes if budget else [0])]:
        sw.sw_set_latency_mode(lm)
        for _ in range(2):
            sw.sw_search_dev(q, w.matrix, w.gap_open, w.gap_extend, d, st)
        st.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(3):
            sw.sw_search_dev(q, w.matrix, w.gap_open, w.gap_extend, d, st)
        e1.record(st); st.synchronize()
        ms = e0.elapsed_time(e1) / 3
        got = d.cpu().numpy()
        key = len(q)
        if budget == 0:
            ref = ref or {}
            ref[key] = got.copy()
        same = bool((ref[key] == got).all())
        print(json.dumps({"config": cfg, "m": len(q), "lat_mode": lm, "chunk_MiB": budget / 2**20, "chunks": sw.sw_db_chunks(),
                          "ms": round(ms, 2), "gcups": round(len(q) * w.db.total_residues / (ms * 1e6), 1),
                          "image_GB": round(sw.sw_last_stats()["pair_columns"] * 2 / 1e9, 3),
                          "pass_kernels_ms": round(sw.sw_last_timing()["pass_kernels_ms"], 2),
                          "search_ms": round(sw.sw_last_timing()["search_ms"], 2),
                          "identical_to_resident": same}), flush=True)
sw.sw_set_latency_mode(0)
