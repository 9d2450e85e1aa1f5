"""Calibration of the pass time model (api.cu pass_time_model):
per-column step latency of one group running alone, throughput tiles vs the
latency tiles, and configs[0] under each choice (dev tool, 1 GPU).

    python tools/lat_calibrate.py > profiles/r02_lat_calibration.jsonl
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1702_07195_b200 as sw  # noqa: E402
import sw_inputs as si  # noqa: E402


def timed(q, d, st, reps=10):
    for _ in range(2):
        sw.sw_search_dev(q, si.BLOSUM62, 10, 2, d, st)
    st.synchronize()
    ts, pk = [], []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        sw.sw_search_dev(q, si.BLOSUM62, 10, 2, d, st)
        e1.record(st)
        st.synchronize()
        ts.append(e0.elapsed_time(e1))
        pk.append(sw.sw_last_timing()["pass_kernels_ms"])
    return float(np.median(ts)), float(np.median(pk))


def main():
    torch.cuda.set_device(0)
    st = torch.cuda.Stream()
    rng = np.random.default_rng(11)
    f_mhz = 1965.0
    # (1) step latency: one long sequence, query of exactly G*R rows (one pass)
    n = 12000
    db = si.database_from_list([si.rr_residues(rng, n)])
    sw.sw_db_load(db.residues, db.offsets)
    d = torch.empty(1, dtype=torch.int32, device="cuda")
    tiles = [(32, 8, 0), (32, 12, 0), (32, 16, 0), (16, 16, 0), (16, 29, 0), (32, 29, 0), (8, 18, 0),
             (32, 3, 1), (32, 4, 1), (32, 5, 1), (32, 6, 1), (32, 8, 1), (16, 9, 1)]
    for G, R, lat in tiles:
        sw.sw_set_latency_mode(1 if lat else -1)
        sw.sw_set_tile(G, R)
        q = si.rr_residues(rng, G * R)
        ms, pms = timed(q, d, st)
        s = sw.sw_last_stats()
        assert s["G"] == G and s["R"] == R and s["lat"] == lat and s["passes"] == 1, s
        print(json.dumps({"kind": "step", "G": G, "R": R, "lat": lat, "n": n, "pass_ms": round(pms, 4),
                          "step_cycles": round(pms * 1e-3 * f_mhz * 1e6 / (n + G), 1)}), flush=True)
    # (2) configs[0]: auto, LAT tiles, throughput tiles
    w = si.config0()
    sw.sw_db_load(w.db.residues, w.db.offsets)
    d = torch.empty(w.db.count, dtype=torch.int32, device="cuda")
    q = w.queries[0]
    cells = len(q) * w.db.total_residues
    for G, R, lat in [(0, 0, 0), (32, 8, 0), (8, 18, 0)] + [t for t in tiles if t[2]] + [(0, 0, 1)]:
        sw.sw_set_latency_mode(1 if lat else (0 if G == 0 else -1))
        sw.sw_set_tile(G, R)
        ms, pms = timed(q, d, st, reps=20)
        s = sw.sw_last_stats()
        print(json.dumps({"kind": "cfg0", "forced": [G, R, lat], "tile": [s["G"], s["R"]], "lat": s["lat"],
                          "passes": s["passes"], "ms": round(ms, 4), "pass_ms": round(pms, 4),
                          "gcups": round(cells / (ms * 1e6), 1)}), flush=True)
    # (3) bulk throughput of the LAT tiles relative to the throughput tiles (cfg1 at full size)
    w = si.config1(scale=1.0)
    sw.sw_db_load(w.db.residues, w.db.offsets)
    d = torch.empty(w.db.count, dtype=torch.int32, device="cuda")
    os.environ["SWDB_SOLO"] = "0"   # the latency tiles' bulk rate without solo items (read per search)
    for G, R, lat in [(32, 8, 0), (32, 16, 0)] + [t for t in tiles if t[2]]:
        sw.sw_set_latency_mode(1 if lat else -1)
        sw.sw_set_tile(G, R)
        q = si.rr_residues(rng, G * R)
        ms, pms = timed(q, d, st)
        print(json.dumps({"kind": "bulk", "G": G, "R": R, "lat": lat, "pass_ms": round(pms, 4),
                          "gcups": round(G * R * w.db.total_residues / (pms * 1e6), 1)}), flush=True)
    sw.sw_set_tile(0)
    sw.sw_set_latency_mode(0)
    os.environ.pop("SWDB_SOLO", None)


if __name__ == "__main__":
    main()
