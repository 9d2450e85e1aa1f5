"""Replay one dumped stress trial (tests/report_stress.py --only N --dump F)
under variants of its settings, each in its own process (a device fault is
sticky), and report which variants fault or mismatch (dev tool, 1 GPU).

    python tools/stress_repro.py trial.npz [variant ...]
    variant: key=value overrides of tile=GxR, wave=, lat=, prof=, rows=
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_one(path, over):
    sys.path.insert(0, ROOT)
    import numpy as np
    import oracle
    import paper_1702_07195_b200 as sw
    d = np.load(path)
    tile = tuple(int(x) for x in d["tile"])
    settings = {"tile": tile, "wave": int(d["wave"]), "lat": int(d["lat"]), "prof": int(d["prof"]), "rows": 0}
    for kv in over:
        k, v = kv.split("=")
        settings[k] = tuple(int(x) for x in v.split("x")) if k == "tile" else int(v)
    import torch
    torch.cuda.set_device(0)
    sw.sw_set_tile(*settings["tile"])
    sw.sw_set_wave(settings["wave"])
    sw.sw_set_latency_mode(settings["lat"])
    sw.sw_set_profile(settings["prof"])
    sw.sw_set_rows_mode(settings["rows"])
    res, offs, q, M = d["res"], d["offs"], d["q"], d["M"]
    go, ge = int(d["go"]), int(d["ge"])
    path_kind = str(d["path"])
    if path_kind == "streamed":
        sw.sw_db_load_streamed(res, offs, int(d["chunk"]))
    else:
        sw.sw_db_load(res, offs)
    if path_kind == "pair":
        got = sw.sw_search_batch([q, d["q2"]], M, go, ge)[0]
    else:
        got = sw.sw_search(q, M, go, ge)
    st = sw.sw_last_stats()
    exp = oracle.batch(q, res, offs, M, go, ge)
    topk_ok = None
    if path_kind != "pair":
        k = int(settings.get("k", int(d["k"])))
        idx, sc = sw.sw_topk(k)
        eidx, esc = oracle.topk(got, k)
        topk_ok = bool((idx == eidx).all() and (sc == esc).all())
    print(json.dumps({"settings": settings, "path": path_kind, "mismatches": int((got != exp).sum()),
                      "topk_ok": topk_ok,
                      "stats": {k: st[k] for k in ("G", "R", "passes", "wave", "lat", "profile", "rows_pairs")}}))


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[2] == "--child":
        run_one(sys.argv[1], sys.argv[3:])
        sys.exit(0)
    variants = [a.split(",") if a else [] for a in (sys.argv[2:] or [""])]
    for v in variants:
        r = subprocess.run([sys.executable, __file__, sys.argv[1], "--child"] + v, capture_output=True, text=True,
                           timeout=600)
        out = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        print(json.dumps({"variant": v, "rc": r.returncode, "result": json.loads(out[-1]) if out else None,
                          "err": r.stderr.strip().splitlines()[-1][-300:] if r.returncode else ""}), flush=True)
