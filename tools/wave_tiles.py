"""Wavefront tile sweep on databases of long sequences (dev tool)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import sw_inputs as si
import paper_1702_07195_b200 as sw
from tools.wave_perf import timed

rng = np.random.default_rng(5)
st = torch.cuda.Stream()
for n, lo, hi in ((20, 20000, 35000), (200, 20000, 35000), (2000, 5000, 35000), (8000, 1000, 6000)):
    db = si.database_from_list([si.rr_residues(rng, int(L)) for L in rng.integers(lo, hi, n)])
    sw.sw_db_load(db.residues, db.offsets)
    d = torch.empty(db.count, dtype=torch.int32, device="cuda")
    for m in (1000, 5478):
        q = si.rr_residues(rng, m)
        out = {}
        sw.sw_set_wave(-1); sw.sw_set_tile(0)
        ms = timed(q, d, st); s = sw.sw_last_stats()
        out["per_pass_auto"] = [s["G"], s["R"], s["passes"], round(m * db.total_residues / (ms * 1e6), 1)]
        sw.sw_set_wave(1)
        for G, R in ((32, 8), (16, 16), (32, 16), (16, 29), (32, 29), (16, 32), (32, 32)):
            sw.sw_set_tile(G, R)
            ms = timed(q, d, st); s = sw.sw_last_stats()
            out[f"{G}x{R}"] = [s["passes"], s["wave"], round(m * db.total_residues / (ms * 1e6), 1)]
        sw.sw_set_tile(0); sw.sw_set_wave(0)
        ms = timed(q, d, st); s = sw.sw_last_stats()
        out["auto"] = [s["G"], s["R"], s["passes"], s["wave"], round(m * db.total_residues / (ms * 1e6), 1)]
        print(json.dumps({"n": n, "len": [lo, hi], "items": s["items"], "m": m, **out}), flush=True)
