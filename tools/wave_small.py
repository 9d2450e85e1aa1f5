"""few long sequences: per-pass auto vs forced 32x8 wavefront vs auto (dev)"""
import json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import sw_inputs as si
import paper_1702_07195_b200 as sw
from tools.wave_perf import timed
rng = np.random.default_rng(11)
st = torch.cuda.Stream()
for n, lo, hi in ((1, 35000, 35001), (2, 20000, 35000), (6, 20000, 35000), (20, 20000, 35000), (60, 5000, 35000), (200, 20000, 35000)):
    db = si.database_from_list([si.rr_residues(rng, int(L)) for L in rng.integers(lo, hi, n)])
    sw.sw_db_load(db.residues, db.offsets)
    d = torch.empty(db.count, dtype=torch.int32, device="cuda")
    for m in (300, 600, 1000, 2000):
        q = si.rr_residues(rng, m)
        out = {}
        sw.sw_set_wave(-1); sw.sw_set_tile(0)
        ms = timed(q, d, st); s = sw.sw_last_stats()
        out["per_pass"] = [s["G"], s["R"], s["passes"], s["lat"], round(ms, 3)]
        ref = d.cpu().numpy().copy()
        sw.sw_set_wave(1); sw.sw_set_tile(32, 8)
        ms = timed(q, d, st); s = sw.sw_last_stats()
        out["wave32x8"] = [s["passes"], s["wave"], round(ms, 3), bool((d.cpu().numpy() == ref).all())]
        sw.sw_set_tile(0); sw.sw_set_wave(0)
        ms = timed(q, d, st); s = sw.sw_last_stats()
        out["auto"] = [s["G"], s["R"], s["passes"], s["wave"], s["lat"], round(ms, 3), bool((d.cpu().numpy() == ref).all())]
        print(json.dumps({"n": n, "items": s["items"], "m": m, **out}), flush=True)
