"""cfg0 (small database, latency-bound) under every tile, per-pass and
wavefront (dev tool): which launch shape shortens the critical path."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import sw_inputs as si
import paper_1702_07195_b200 as sw
from tools.wave_perf import timed

w = si.config0()
sw.sw_db_load(w.db.residues, w.db.offsets)
d = torch.empty(w.db.count, dtype=torch.int32, device="cuda")
st = torch.cuda.Stream()
q = w.queries[0]
cells = len(q) * w.db.total_residues
out = []
for wave in (-1, 1):
    for G in (8, 16, 32):
        for R in range(1, 33):
            if not sw.sw_tile_supported(G, R):
                continue
            sw.sw_set_wave(wave)
            sw.sw_set_tile(G, R)
            ms = timed(q, d, st, reps=20)
            s = sw.sw_last_stats()
            tm = sw.sw_last_timing()
            out.append({"wave": wave, "G": G, "R": R, "passes": s["passes"], "wave_used": s["wave"],
                        "ms": round(ms, 4), "gcups": round(cells / (ms * 1e6), 1),
                        "pass_ms": round(tm["pass_kernels_ms"], 4)})
sw.sw_set_tile(0); sw.sw_set_wave(0)
ms = timed(q, d, st, reps=20); s = sw.sw_last_stats()
best = sorted(out, key=lambda r: r["ms"])[:8]
print(json.dumps({"auto": {"G": s["G"], "R": s["R"], "passes": s["passes"], "wave": s["wave"], "ms": round(ms, 4),
                           "gcups": round(cells / (ms * 1e6), 1)}, "best": best}))
