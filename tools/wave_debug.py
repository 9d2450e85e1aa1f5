import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch, sw_inputs as si, paper_1702_07195_b200 as sw
mode = int(sys.argv[1]); m = int(sys.argv[2]); n = int(sys.argv[3])
rng = np.random.default_rng(5)
db = si.database_from_list([si.rr_residues(rng, int(L)) for L in rng.integers(20000, 35000, n)])
sw.sw_db_load(db.residues, db.offsets)
sw.sw_set_wave(mode)
q = si.rr_residues(rng, m)
got = sw.sw_search(q, si.BLOSUM62, 10, 2)
print("ok", mode, m, n, sw.sw_last_stats(), got[:3])
