"""Small end-to-end exercise of every kernel for compute-sanitizer runs (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import sw_inputs as si, oracle
import paper_1702_07195_b200 as sw
torch.cuda.set_device(0)
rng = np.random.default_rng(1)
seqs = [si.rr_residues(rng, int(L)) for L in rng.integers(0, 300, 200)] + [si.encode("W" * 3000)]
db = si.database_from_list(seqs)
qs = [si.rr_residues(rng, 100), si.rr_residues(rng, 700), si.encode("W" * 3000)]
sw.sw_db_load(db.residues, db.offsets)
bad = 0
for q in qs:
    got = sw.sw_search(q, si.BLOSUM62, 10, 2)
    bad += int((got != oracle.batch(q, db.residues, db.offsets, si.BLOSUM62, 10, 2)).sum())
    sw.sw_topk(5); sw.sw_topk(100)
allb = sw.sw_search_batch(qs, si.BLOSUM62, 10, 2)
sw.sw_db_load_streamed(db.residues, db.offsets, 16 * 1024)
for q in qs[:2]:
    got = sw.sw_search(q, si.BLOSUM62, 10, 2)
    bad += int((got != oracle.batch(q, db.residues, db.offsets, si.BLOSUM62, 10, 2)).sum())
print("mismatches", bad)
