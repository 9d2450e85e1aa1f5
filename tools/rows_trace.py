"""Per-pass cycle counts of the rows kernel on one long sequence (build with
SW_ROWS_TRACE=1; dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1702_07195_b200 as sw
import sw_inputs as si
rng = np.random.default_rng(77)
n, m = int(sys.argv[1]) if len(sys.argv) > 1 else 35000, int(sys.argv[2]) if len(sys.argv) > 2 else 144
db = si.database_from_list([si.rr_residues(rng, n)])
sw.sw_db_load(db.residues, db.offsets)
sw.sw_set_rows_mode(1)
q = si.rr_residues(rng, m)
sw.sw_search(q, si.BLOSUM62, 10, 2)
