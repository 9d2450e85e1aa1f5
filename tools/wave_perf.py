"""Cross-pass wavefront vs per-pass launches (dev / report tool): GCUPS of
sw_search_dev on (a) databases of few long sequences and (b) cfg1 with a
multi-pass query, wavefront off (-1) and on (1)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import sw_inputs as si
import paper_1702_07195_b200 as sw


def timed(q, d, st, reps=3):
    sw.sw_search_dev(q, si.BLOSUM62, 10, 2, d, st)
    st.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        sw.sw_search_dev(q, si.BLOSUM62, 10, 2, d, st)
    e1.record(st); st.synchronize()
    return e0.elapsed_time(e1) / reps


if __name__ == "__main__":
    rng = np.random.default_rng(5)
    st = torch.cuda.Stream()
    cases = []
    for n, lo, hi in ((20, 20000, 35000), (200, 20000, 35000), (2000, 5000, 35000)):
        cases.append((f"{n} long sequences U[{lo},{hi}]",
                      si.database_from_list([si.rr_residues(rng, int(L)) for L in rng.integers(lo, hi, n)])))
    w = si.config1()
    cases.append(("cfg1 (1 M sequences)", w.db))
    for name, db in cases:
        sw.sw_db_load(db.residues, db.offsets)
        d = torch.empty(db.count, dtype=torch.int32, device="cuda")
        for m in (1000, 5478):
            q = si.rr_residues(rng, m)
            res = {}
            for mode in (-1, 1):
                sw.sw_set_wave(mode)
                print("#", name, m, mode, flush=True, file=sys.stderr)
                ms = timed(q, d, st)
                s = sw.sw_last_stats()
                res[mode] = {"ms": round(ms, 2), "gcups": round(m * db.total_residues / (ms * 1e6), 1),
                             "tile": [s["G"], s["R"]], "passes": s["passes"], "wave": s["wave"]}
            sw.sw_set_wave(0)
            print(json.dumps({"db": name, "residues": db.total_residues, "m": m, "items": sw.sw_last_stats()["items"],
                              "per_pass": res[-1], "wavefront": res[1]}), flush=True)
