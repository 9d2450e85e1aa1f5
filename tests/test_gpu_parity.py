"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle,
element by element, bit-exact (integer scores).

Sizes span several tiles, several query passes and ragged tails; the
BASELINE.json configurations are checked in full where the oracle finishes in
seconds (cfg0) and on seeded samples otherwise (cfg1 full size, in the
launch configuration bench.py times).
"""
import numpy as np
import pytest

import oracle
import sw_inputs as si
from sw_inputs import BLOSUM62, encode
from tests.brute import expand

pytestmark = pytest.mark.gpu

sw = pytest.importorskip("paper_1702_07195_b200")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    yield
    sw.sw_set_tile(0)


def _db(seqs):
    return si.database_from_list(seqs)


def _check_db(db, q, M=BLOSUM62, go=10, ge=2, label=""):
    sw.sw_db_load(db.residues, db.offsets)
    got = sw.sw_search(q, M, go, ge)
    exp = oracle.batch(q, db.residues, db.offsets, M, go, ge)
    bad = np.nonzero(got != exp)[0]
    assert bad.size == 0, f"{label}: {bad.size} mismatches, first {bad[:5]} got {got[bad[:5]]} exp {exp[bad[:5]]}"
    return got


def _flags_ok(st, exp):
    """The 16-bit saturation flags: every sequence whose exact score reaches
    the threshold T is flagged (R7); the biased-unsigned arithmetic
    may also flag high-half partners of flagged low-half sequences (carry
    propagation), never fewer."""
    need = int((np.asarray(exp) >= st["flag_threshold"]).sum())
    return st["flagged"] >= need if st["arith"] == 2 else st["flagged"] == need


def test_hand_examples_on_gpu():
    rows = [ln.rstrip("\n").split("\t") for ln in open("tests/golden/hand_examples.txt")
            if ln.strip() and not ln.startswith("#")]
    # one database per (query, gaps): every subject of that query
    groups = {}
    for r in rows:
        groups.setdefault((r[0], int(r[2]), int(r[3])), []).append((r[1], int(r[4])))
    for (qs, go, ge), subs in groups.items():
        db = _db([encode(expand(s)) for s, _ in subs])
        sw.sw_db_load(db.residues, db.offsets)
        got = sw.sw_search(encode(expand(qs)), BLOSUM62, go, ge)
        assert got.tolist() == [v for _, v in subs], (qs, go, ge)


def test_random_small_databases_random_scoring():
    rng = np.random.default_rng(1234)
    for trial in range(12):
        count = int(rng.integers(1, 400))
        lens = rng.integers(0, 300, count)
        seqs = [rng.integers(0, 24, int(L)).astype(np.uint8) for L in lens]
        m = int(rng.integers(1, 1400))
        q = rng.integers(0, 24, m).astype(np.uint8)
        M = si.random_symmetric_matrix(rng) if trial % 2 == 0 else rng.integers(-4, 12, (24, 24)).astype(np.int8)
        go, ge = int(rng.integers(0, 16)), int(rng.integers(0, 16))
        _check_db(_db(seqs), q, M, go, ge, label=f"trial {trial} m={m} go={go} ge={ge}")


def test_extreme_scoring_parameters():
    """The biased 16-bit arithmetic (stored = score + 16384, DESIGN.md 4.2 / R7)
    at the edges of its argument range: int8 matrices spanning [-128, 127] (the
    32-bit diagonal add must not carry between halves), gap penalties around and
    above 16384 and 32767 (clamped in 16 bit), zero penalties, and scores above
    the 16-bit flag threshold (re-scored in 32 bit)."""
    rng = np.random.default_rng(4242)
    seqs = [rng.integers(0, 24, int(L)).astype(np.uint8) for L in rng.integers(0, 400, 150)]
    seqs += [np.full(600, 3, np.uint8), np.full(300, 7, np.uint8)]   # long runs: large scores
    db = _db(seqs)
    wide = rng.integers(-128, 128, (24, 24)).astype(np.int8)
    wide[np.arange(24), np.arange(24)] = 127
    low = rng.integers(-128, -60, (24, 24)).astype(np.int8)          # every entry negative
    low[3, 3] = 1
    q = np.concatenate([rng.integers(0, 24, 250).astype(np.uint8), np.full(200, 3, np.uint8)])
    for M in (BLOSUM62, wide, low):
        for go, ge in ((0, 0), (10, 2), (16383, 1), (16384, 0), (16385, 0), (30000, 5), (5, 30000),
                       (40000, 40000), (1 << 20, 1 << 20)):
            _check_db(db, q, M, go, ge, label=f"go={go} ge={ge} smax={int(M.max())}")
    # query pairs (QPM 3) with the wide matrix
    qs = [q, rng.integers(0, 24, 333).astype(np.uint8)]
    sw.sw_db_load(db.residues, db.offsets)
    got = sw.sw_search_batch(qs, wide, 7, 3)
    for k, qq in enumerate(qs):
        exp = oracle.batch(qq, db.residues, db.offsets, wide, 7, 3)
        assert (got[k] == exp).all(), k


def test_degenerate_databases_and_queries():
    """Edge cases of the method: only empty sequences, a single residue, a query of
    length 1, many one-residue sequences, identical sequences (ties in the sorting
    stage), and a database whose total length is odd (an empty B half)."""
    rng = np.random.default_rng(77)
    cases = [
        [np.zeros(0, np.uint8)],
        [np.zeros(0, np.uint8)] * 5,
        [encode("W")],
        [encode("W"), np.zeros(0, np.uint8), encode("A")],
        [si.rr_residues(rng, 1) for _ in range(257)],
        [encode("MKVLAAGW")] * 33,
        [si.rr_residues(rng, int(L)) for L in (1, 2, 3, 5000, 7)],
    ]
    queries = [encode("W"), encode("A"), si.rr_residues(rng, 2), si.rr_residues(rng, 700)]
    for ci, seqs in enumerate(cases):
        db = _db(seqs)
        sw.sw_db_load(db.residues, db.offsets)
        for q in queries:
            got = sw.sw_search(q, BLOSUM62, 10, 2)
            exp = oracle.batch(q, db.residues, db.offsets, BLOSUM62, 10, 2)
            assert (got == exp).all(), (ci, len(q), got[:8], exp[:8])
            k = min(10, len(seqs))
            idx, sc = sw.sw_topk(k)
            eidx, esc = oracle.topk(exp, k)
            assert (idx == eidx).all() and (sc == esc).all(), (ci, len(q))


def test_every_tile_is_exact():
    rng = np.random.default_rng(7)
    seqs = [si.rr_residues(rng, int(L)) for L in rng.integers(1, 500, 300)]
    seqs += [np.zeros(0, np.uint8), si.rr_residues(rng, 3000)]
    db = _db(seqs)
    q = si.rr_residues(rng, 700)
    exp = oracle.batch(q, db.residues, db.offsets, BLOSUM62, 10, 2)
    sw.sw_db_load(db.residues, db.offsets)
    for G in (8, 16, 32):
        for R in range(1, 33):
            if not sw.sw_tile_supported(G, R):
                continue
            sw.sw_set_tile(G, R)
            got = sw.sw_search(q, BLOSUM62, 10, 2)
            st = sw.sw_last_stats()
            assert (st["G"], st["R"]) == (G, R)
            assert (got == exp).all(), (G, R, np.nonzero(got != exp)[0][:5])
    sw.sw_set_tile(0)


def test_config0_full_parity():
    w = si.config0()
    got = _check_db(w.db, w.queries[0], label="cfg0")
    assert sw.sw_last_stats()["flagged"] == 0


def test_saturation_boundary_and_rescoring():
    # W^n vs W^n scores 11n: below, at and above the flag threshold T
    # (T = 32757 in the default biased-unsigned and the relu form, 16373 in
    # the biased-signed form; R7), and far above the 16-bit range
    ns = [1487, 1488, 1489, 1490, 2977, 2978, 2979, 2980, 3000, 4000]
    seqs = [encode("W" * n) for n in ns] + [encode("A" * 50)]
    q = encode("W" * 4000)
    got = _check_db(_db(seqs), q, label="W runs")
    assert got[:len(ns)].tolist() == [11 * n for n in ns]
    st = sw.sw_last_stats()
    T = st["flag_threshold"]
    assert T in (32757, 16373)
    assert T == (16373 if sw.sw_last_stats()["arith"] == 1 else 32757)
    assert _flags_ok(st, [11 * n for n in ns])


def test_rescoring_narrow_last_pass():
    """The 32-bit kernel's last query pass runs R/3 or 2R/3 rows per lane when
    that covers the rows left (no phantom rows past the next multiple of 32 rows
    per lane width).  One W^3000 sequence flags in the 16-bit pass holding row
    ~2,978 (8x8 tile: 64 rows per pass, re-scoring from row 2,944); the query
    length sets the rows left at and around every width edge (256 / 512 / 768
    rows per pass of the 24-row kernel).  cells32 pins the rows computed."""
    db = _db([encode("W" * 3000)])
    sw.sw_db_load(db.residues, db.offsets)
    sw.sw_set_tile(8, 8)
    try:
        for k in (40, 255, 256, 257, 511, 512, 513, 767, 768, 769, 1280, 1281, 1537):
            q = encode("W" * (2944 + k))
            got = sw.sw_search(q, BLOSUM62, 10, 2)
            assert int(got[0]) == 11 * min(2944 + k, 3000), k
            st = sw.sw_last_stats()
            assert st["flagged"] == 1, k
            rows = 2944 + k - 2944
            passes = -(-rows // 768)
            left = rows - (passes - 1) * 768
            last = 256 if left <= 256 else (512 if left <= 512 else 768)
            assert st["cells32"] == 3000 * ((passes - 1) * 768 + last), (k, st["cells32"])
    finally:
        sw.sw_set_tile(0)


def test_rescoring_seeded_from_pass_boundaries():
    """Sequences flagged in a later 16-bit pass are re-scored in 32 bit from that
    pass's first row, seeded with its exact input boundary.  A
    prefix of A rows before W^3000 moves the flagging pass; small tiles (64 rows
    per pass) make the 16-bit pass boundaries cut the 32-bit kernel's slices at
    many different offsets."""
    rng = np.random.default_rng(31)
    seqs = [encode("W" * n) for n in (1400, 1489, 1600, 2500, 2979, 3000, 3300)]
    seqs += [np.concatenate([si.rr_residues(rng, 300), encode("W" * 3100), si.rr_residues(rng, 200)])]
    seqs += [si.rr_residues(rng, int(L)) for L in rng.integers(1, 800, 40)]
    db = _db(seqs)
    sw.sw_db_load(db.residues, db.offsets)
    try:
        for x in (0, 37, 700, 1501):
            q = encode("A" * x + "W" * 3400)
            exp = oracle.batch(q, db.residues, db.offsets, BLOSUM62, 10, 2)
            for G, R in ((0, 0), (8, 8), (16, 12), (32, 29)):
                sw.sw_set_tile(G, R)
                got = sw.sw_search(q, BLOSUM62, 10, 2)
                st = sw.sw_last_stats()
                assert (got == exp).all(), (x, G, R, np.nonzero(got != exp)[0][:5])
                assert _flags_ok(st, exp)
    finally:
        sw.sw_set_tile(0)


def test_rescoring_short_sequences_at_fetch_block_edges():
    """The 32-bit kernel fetches lane 0's column inputs in blocks of 32 columns
    (DESIGN.md 4.3).  With every substitution +127 and prohibitive gaps, the
    score is the closed form 127 * min(n, m) (an ungapped diagonal run), so
    sequences from 258 residues on are flagged (129 in the biased-signed
    form); lengths around the multiples of 32 put the sequence end at every
    position of a fetch block, for flagging in the first pass (row 0) and in a
    later one (64-row passes)."""
    M = np.full((24, 24), 127, np.int8)
    lens = [0, 1, 31, 32, 33, 63, 64, 65, 127, 128, 129, 130, 159, 160, 161, 191, 192, 193,
            223, 224, 225, 255, 256, 257, 258, 259, 287, 288, 289, 300, 319, 320, 321, 351, 352, 353,
            383, 384, 385, 415, 416, 417, 447, 448, 449, 479, 480, 481, 511, 512, 513, 1000]
    rng = np.random.default_rng(77)
    db = _db([rng.integers(0, 24, n).astype(np.uint8) for n in lens])
    sw.sw_db_load(db.residues, db.offsets)
    try:
        for m in (300, 700, 1100):
            q = rng.integers(0, 24, m).astype(np.uint8)
            closed = np.array([127 * min(n, m) for n in lens], np.int32)
            exp = oracle.batch(q, db.residues, db.offsets, M, 30000, 30000)
            assert (exp == closed).all()
            for G, R in ((0, 0), (8, 8), (32, 29)):
                sw.sw_set_tile(G, R)
                got = sw.sw_search(q, M, 30000, 30000)
                st = sw.sw_last_stats()
                assert (got == closed).all(), (m, G, R, [(lens[i], int(got[i])) for i in np.nonzero(got != closed)[0][:5]])
                assert _flags_ok(st, closed) and st["flagged"] > 0
    finally:
        sw.sw_set_tile(0)


def test_later_passes_skip_flagged_leading_sequences():
    """Passes after the first start each item behind its leading run of
    flagged sequences (both halves).  Equal-length W-rich
    copies pair up at the head of items like cfg4's planted copies; some items
    have a flagged sequence in one half only, or a flagged run longer in one
    half than in the other, and short unflagged sequences follow them.  Every
    score must still equal the oracle's, for small tiles (many passes) and the
    default one."""
    rng = np.random.default_rng(41)
    block = encode("W" * 3000)
    seqs = [block.copy() for _ in range(24)]
    seqs += [np.concatenate([encode("W" * 2990), si.rr_residues(rng, 10)]) for _ in range(5)]
    seqs += [si.rr_residues(rng, 3000) for _ in range(7)]                  # same length, unflagged
    seqs += [si.rr_residues(rng, int(L)) for L in rng.integers(1, 300, 300)]
    order = rng.permutation(len(seqs))
    seqs = [seqs[i] for i in order]
    db = _db(seqs)
    sw.sw_db_load(db.residues, db.offsets)
    try:
        for x in (0, 300):
            q = encode("A" * x + "W" * 3100)
            exp = oracle.batch(q, db.residues, db.offsets, BLOSUM62, 10, 2)
            for G, R in ((0, 0), (8, 8), (16, 12), (32, 16)):
                sw.sw_set_tile(G, R)
                got = sw.sw_search(q, BLOSUM62, 10, 2)
                st = sw.sw_last_stats()
                assert st["passes"] > 1 or G == 0
                assert (got == exp).all(), (x, G, R, np.nonzero(got != exp)[0][:5])
                assert _flags_ok(st, exp) and st["flagged"] >= 29
                idx, top = sw.sw_topk(10)
                eidx, etop = oracle.topk(exp, 10)
                assert (idx == eidx).all() and (top == etop).all()
    finally:
        sw.sw_set_tile(0)


def test_adversarial_mixed_with_planted_copies():
    w = si.config4(scale=0.002)   # 400 sequences incl. long ones and 8 planted copies
    got = _check_db(w.db, w.queries[0], label="cfg4 small")
    st = sw.sw_last_stats()
    assert _flags_ok(st, got)
    assert (got[w.planted] >= 32757).all()


def test_long_sequences_and_query_passes():
    rng = np.random.default_rng(99)
    seqs = [si.rr_residues(rng, int(L)) for L in (35000, 12000, 5000, 1, 2, 3)]
    seqs += [si.rr_residues(rng, int(L)) for L in rng.integers(5, 200, 60)]
    q = si.rr_residues(rng, 1500)
    _check_db(_db(seqs), q, label="long")


def test_topk_matches_oracle_sort_stage():
    w = si.config0()
    sw.sw_db_load(w.db.residues, w.db.offsets)
    got = sw.sw_search(w.queries[0], BLOSUM62, 10, 2)
    for k in (1, 10, 32, 33, 100, 5000, w.db.count, w.db.count + 10):
        idx, sc = sw.sw_topk(k)
        eidx, esc = oracle.topk(got, k)
        assert (idx == eidx).all() and (sc == esc).all(), k


def test_topk_dev_with_index_ties():
    import torch
    scores = torch.tensor([3, 9, 9, 1, 9], dtype=torch.int32, device="cuda")
    index = torch.tensor([40, 11, 10, 7, 12], dtype=torch.int64, device="cuda")
    oi = torch.empty(5, dtype=torch.int64, device="cuda")
    os_ = torch.empty(5, dtype=torch.int32, device="cuda")
    n = sw.sw_topk_dev(scores, index, 5, 4, oi, os_)
    assert n == 4
    assert oi[:4].tolist() == [10, 11, 12, 40]
    assert os_[:4].tolist() == [9, 9, 9, 3]


def test_search_dev_matches_search():
    import torch
    w = si.config0(scale=0.2)
    sw.sw_db_load(w.db.residues, w.db.offsets)
    host = sw.sw_search(w.queries[0], BLOSUM62, 10, 2)
    d = torch.empty(w.db.count, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    sw.sw_search_dev(w.queries[0], BLOSUM62, 10, 2, d, s)
    s.synchronize()
    assert (d.cpu().numpy() == host).all()


def test_error_paths_on_gpu():
    w = si.config0(scale=0.01)
    sw.sw_db_load(w.db.residues, w.db.offsets)
    with pytest.raises(sw.SWError):
        sw.sw_search(np.array([30], np.uint8), BLOSUM62, 10, 2)
    with pytest.raises(sw.SWError):
        sw.sw_search(np.zeros(0, np.uint8), BLOSUM62, 10, 2)
    with pytest.raises(sw.SWError):
        sw.sw_search(encode("AW"), BLOSUM62, -1, 2)
    # a failed call leaves the database usable
    got = sw.sw_search(w.queries[0], BLOSUM62, 10, 2)
    exp = oracle.batch(w.queries[0], w.db.residues, w.db.offsets, BLOSUM62, 10, 2)
    assert (got == exp).all()


def test_config1_full_size_sampled():
    """BASELINE.json configs[1] at full size (1 M sequences, query 464), in the
    launch configuration bench.py times; oracle on a seeded sample of 3,000
    sequences plus the 200 longest, and properties on all."""
    w = si.config1()
    sw.sw_db_load(w.db.residues, w.db.offsets)
    got = sw.sw_search(w.queries[0], BLOSUM62, 10, 2)
    assert got.min() >= 0
    assert sw.sw_last_stats()["flagged"] == 0
    rng = np.random.default_rng(2024)
    L = w.db.lengths()
    idx = np.unique(np.concatenate([rng.choice(w.db.count, 3000, replace=False), np.argsort(-L)[:200]]))
    exp = oracle.batch(w.queries[0], w.db.residues, w.db.offsets, BLOSUM62, 10, 2, idx=idx)
    assert (got[idx] == exp).all()
    # upper bound: score <= sum over the query of its row maxima
    ub = int(np.maximum(BLOSUM62[w.queries[0], :20].max(axis=1), 0).sum())
    assert got.max() <= ub
    # top-10 agrees with the oracle sort of the GPU scores
    idx10, sc10 = sw.sw_topk(10)
    eidx, esc = oracle.topk(got, 10)
    assert (idx10 == eidx).all() and (sc10 == esc).all()


# ---- multi-query packing: query pairs in the two halves
def test_batch_random_queries_match_oracle():
    rng = np.random.default_rng(4242)
    for trial in range(4):
        seqs = [rng.integers(0, 24, int(L)).astype(np.uint8) for L in rng.integers(0, 400, 300)]
        seqs.append(si.rr_residues(rng, 3000))
        db = _db(seqs)
        nq = int(rng.integers(1, 6))
        qs = [rng.integers(0, 24, int(rng.integers(1, 1300))).astype(np.uint8) for _ in range(nq)]
        M = si.random_symmetric_matrix(rng)
        go, ge = int(rng.integers(0, 16)), int(rng.integers(0, 16))
        sw.sw_db_load(db.residues, db.offsets)
        got = sw.sw_search_batch(qs, M, go, ge)
        for k, q in enumerate(qs):
            exp = oracle.batch(q, db.residues, db.offsets, M, go, ge)
            assert (got[k] == exp).all(), (trial, k, len(q), np.nonzero(got[k] != exp)[0][:5])


def test_batch_with_saturating_pair():
    seqs = [encode("W" * n) for n in (100, 2977, 2978, 3500)] + [encode("AC" * 40)]
    db = _db(seqs)
    qs = [encode("W" * 3600), encode("AC" * 30), encode("W" * 3000)]
    sw.sw_db_load(db.residues, db.offsets)
    got = sw.sw_search_batch(qs, BLOSUM62, 10, 2)
    for k, q in enumerate(qs):
        exp = oracle.batch(q, db.residues, db.offsets, BLOSUM62, 10, 2)
        assert (got[k] == exp).all(), k
    assert got[0][3] == 11 * 3500


def test_batch_equals_single_searches_cfg3_lengths():
    w = si.config0(scale=0.3)
    rng = si.rng_for(3, 2)
    qs = [si.rr_residues(rng, L) for L in si.CFG3_QUERY_LENGTHS[::4]]   # 144 .. 4917
    sw.sw_db_load(w.db.residues, w.db.offsets)
    got = sw.sw_search_batch(qs, BLOSUM62, 10, 2)
    for k, q in enumerate(qs):
        single = sw.sw_search(q, BLOSUM62, 10, 2)
        assert (got[k] == single).all(), k
    exp = oracle.batch(qs[1], w.db.residues, w.db.offsets, BLOSUM62, 10, 2)
    assert (got[1] == exp).all()


def test_single_after_batch_multipass_no_stale_boundary():
    """Regression: a multi-pass single-query search after a batch search on the
    same database must not read the other image's pass boundaries from the
    shared buffer's padding columns."""
    w = si.config2(scale=0.01)
    rng = si.rng_for(3, 2)
    qs = [si.rr_residues(rng, L) for L in (705, 1267, 2109)]
    sw.sw_db_load(w.db.residues, w.db.offsets)
    sw.sw_search_batch(qs, BLOSUM62, 10, 2)
    for G, R in ((8, 30), (16, 22), (32, 29)):
        sw.sw_set_tile(G, R)
        for q in qs:
            got = sw.sw_search(q, BLOSUM62, 10, 2)
            exp = oracle.batch(q, w.db.residues, w.db.offsets, BLOSUM62, 10, 2)
            assert (got == exp).all(), (G, R, len(q), int((got != exp).sum()))
    sw.sw_set_tile(0)


# ---- out-of-core streamed database
def test_streamed_database_matches_resident_and_oracle():
    rng = np.random.default_rng(555)
    seqs = [si.rr_residues(rng, int(L)) for L in rng.integers(0, 600, 3000)]
    seqs += [si.rr_residues(rng, 9000), encode("W" * 3100), encode("W" * 2000)]
    db = _db(seqs)
    queries = [si.rr_residues(rng, 300), si.rr_residues(rng, 1700), encode("W" * 3100)]
    sw.sw_db_load_streamed(db.residues, db.offsets, 64 * 1024)     # many small chunks
    assert sw.sw_db_chunks() > 4
    assert sw.sw_db_head_columns() >= 9000 // 2    # the resident head holds the 9,000-residue sequence's item
    for q in queries:
        got = sw.sw_search(q, BLOSUM62, 10, 2)
        exp = oracle.batch(q, db.residues, db.offsets, BLOSUM62, 10, 2)
        assert (got == exp).all(), (len(q), int((got != exp).sum()))
        again = sw.sw_search(q, BLOSUM62, 10, 2)
        assert (again == got).all()
        idx, sc = sw.sw_topk(10)
        eidx, esc = oracle.topk(exp, 10)
        assert (idx == eidx).all() and (sc == esc).all()
    with pytest.raises(sw.SWError):
        sw.sw_search_batch(queries[:2], BLOSUM62, 10, 2)
    sw.sw_db_load(db.residues, db.offsets)
    assert sw.sw_db_chunks() == 0
    assert (sw.sw_search(queries[1], BLOSUM62, 10, 2) ==
            oracle.batch(queries[1], db.residues, db.offsets, BLOSUM62, 10, 2)).all()


def test_streamed_resident_head_on_and_off(monkeypatch):
    """Streamed database: the resident head (the leading, longest work items,
    scored on a second stream beside the chunks; swdb.h sw_db_head_columns)
    against the same database streamed without it and against the oracle:
    single- and multi-pass queries, flagged sequences in the head and in the
    chunks (32-bit re-scoring after both streams joined), heads of one long
    item and of many items, searches back to back without a synchronize."""
    import torch
    rng = np.random.default_rng(557)
    seqs = [si.rr_residues(rng, int(L)) for L in rng.integers(1, 400, 4000)]
    seqs += [si.rr_residues(rng, 12000), si.rr_residues(rng, 7000), encode("W" * 3200), encode("W" * 3050),
             encode("W" * 200)]
    db = _db(seqs)
    queries = [si.rr_residues(rng, 144), si.rr_residues(rng, 1300), encode("W" * 3100), si.rr_residues(rng, 40)]
    exps = [oracle.batch(q, db.residues, db.offsets, BLOSUM62, 10, 2) for q in queries]
    assert exps[2].max() >= 32_757
    st = torch.cuda.Stream()
    for budget in (64 * 1024, 512 * 1024):
        for head in ("1", "0"):
            monkeypatch.setenv("SWDB_STREAM_HEAD", head)
            sw.sw_db_load_streamed(db.residues, db.offsets, budget)
            assert (sw.sw_db_head_columns() > 0) == (head == "1"), (budget, head)
            assert sw.sw_db_chunks() >= 2
            for rep in range(2):
                outs = [torch.empty(db.count, dtype=torch.int32, device="cuda") for _ in queries]
                for q, d in zip(queries, outs):
                    sw.sw_search_dev(q, BLOSUM62, 10, 2, d, st)
                st.synchronize()
                for q, d, exp in zip(queries, outs, exps):
                    got = d.cpu().numpy()
                    assert (got == exp).all(), (budget, head, len(q), int((got != exp).sum()))
    monkeypatch.delenv("SWDB_STREAM_HEAD")
    sw.sw_db_load(db.residues, db.offsets)
    assert sw.sw_db_head_columns() == 0


def test_streamed_back_to_back_searches_prefetch():
    """Out-of-core database, searches enqueued back to back on one stream with
    no synchronisation: each search's chunk 0 was copied during the previous
    search's last chunk, into the buffer that chunk did not use (odd and even
    chunk counts), with different queries per search."""
    import torch
    rng = np.random.default_rng(556)
    seqs = [si.rr_residues(rng, int(L)) for L in rng.integers(0, 500, 2500)] + [si.rr_residues(rng, 6000)]
    db = _db(seqs)
    st = torch.cuda.Stream()
    queries = [si.rr_residues(rng, int(m)) for m in (60, 300, 144, 1000, 37)]
    exps = [oracle.batch(q, db.residues, db.offsets, BLOSUM62, 10, 2) for q in queries]
    seen = set()
    for budget in (48 * 1024, 64 * 1024, 96 * 1024, 160 * 1024):
        sw.sw_db_load_streamed(db.residues, db.offsets, budget)
        seen.add(sw.sw_db_chunks() % 2)
        outs = [torch.empty(db.count, dtype=torch.int32, device="cuda") for _ in queries]
        for q, d in zip(queries, outs):
            sw.sw_search_dev(q, BLOSUM62, 10, 2, d, st)
        st.synchronize()
        for q, d, exp in zip(queries, outs, exps):
            got = d.cpu().numpy()
            assert (got == exp).all(), (budget, len(q), int((got != exp).sum()))
    assert seen == {0, 1}, seen   # both chunk-count parities were exercised
    sw.sw_db_load(db.residues, db.offsets)


def test_shard_count_invariance_sequential_shards():
    """Multi-GPU without a multi-GPU box (SPEC.md:409 analogue): the
    database is residue-balanced into G shards (parallel.shard_database), each
    shard is loaded and searched in turn on this GPU with the real kernels, the
    per-shard scores are scattered back to original order and the per-shard
    top-10 candidates merged with sw_topk_dev -- the exact host logic of the
    NCCL path.  Scores and top-10 must be identical for G = 1, 2, 4, 8."""
    import torch
    from paper_1702_07195_b200.parallel import assemble_scores, shard_arrays, shard_database
    w = si.config4(scale=0.002)            # long tail + planted (flagged) copies
    q = w.queries[0]
    exp = oracle.batch(q, w.db.residues, w.db.offsets, BLOSUM62, 10, 2)
    eidx, esc = oracle.topk(exp, 10)
    for G in (1, 2, 4, 8):
        shards = shard_database(w.db.lengths(), G)
        parts, cand_i, cand_s = [], [], []
        for idx in shards:
            res, offs = shard_arrays(w.db.residues, w.db.offsets, idx)
            sw.sw_db_load(res, offs)
            sc = sw.sw_search(q, BLOSUM62, 10, 2)
            parts.append(sc)
            d_sc = torch.from_numpy(sc).cuda()
            d_gi = torch.from_numpy(idx.astype(np.int64)).cuda()
            ti = torch.empty(10, dtype=torch.int64, device="cuda")
            ts = torch.empty(10, dtype=torch.int32, device="cuda")
            n = sw.sw_topk_dev(d_sc, d_gi, sc.size, 10, ti, ts)
            cand_i.append(ti[:n])
            cand_s.append(ts[:n])
        got = assemble_scores(parts, shards, w.db.count)
        assert (got == exp).all(), G
        ci, cs = torch.cat(cand_i), torch.cat(cand_s)
        mi = torch.empty(10, dtype=torch.int64, device="cuda")
        ms = torch.empty(10, dtype=torch.int32, device="cuda")
        sw.sw_topk_dev(cs, ci, cs.numel(), 10, mi, ms)
        assert mi.tolist() == eidx.tolist() and ms.tolist() == esc.tolist(), G


def test_wavefront_auto_from_four_passes_and_spread_units(monkeypatch):
    """Few long work items: auto mode takes the 32x8 cross-pass wavefront from 4
    passes on (m >= 769) and keeps the single pass below; with few units only
    ceil(units / CTAs) <= 4 lane groups per CTA claim (the units spread over the
    SMs; SWDB_WAVE_SPREAD=0 lets every group claim).  Scores equal the oracle's
    either way, from 1 item (every CTA but a few sits the launch out) to more
    items than the limit covers, with saturating sequences re-scored in 32 bit."""
    rng = np.random.default_rng(4242)
    cases = [[si.rr_residues(rng, 9000)],
             [si.rr_residues(rng, int(L)) for L in rng.integers(2000, 7000, 7)] + [encode("W" * 3300)] * 2,
             [si.rr_residues(rng, int(L)) for L in rng.integers(600, 1500, 900)]]
    queries = [si.rr_residues(rng, 600), si.rr_residues(rng, 1000), encode("W" * 3100 + "A" * 20)]
    try:
        sw.sw_set_tile(0)
        sw.sw_set_wave(0)
        for ci, seqs in enumerate(cases):
            db = _db(seqs)
            sw.sw_db_load(db.residues, db.offsets)
            for q in queries:
                exp = oracle.batch(q, db.residues, db.offsets, BLOSUM62, 10, 2)
                for spread in ("1", "0"):
                    monkeypatch.setenv("SWDB_WAVE_SPREAD", spread)
                    got = sw.sw_search(q, BLOSUM62, 10, 2)
                    st = sw.sw_last_stats()
                    assert (got == exp).all(), (ci, len(q), spread, st, np.nonzero(got != exp)[0][:5])
                    if len(q) < 769:
                        assert st["wave"] == 0, (ci, len(q), st)
                    elif ci < 2:
                        assert st["wave"] == 1 and (st["G"], st["R"]) == (32, 8), (ci, len(q), st)
    finally:
        monkeypatch.delenv("SWDB_WAVE_SPREAD", raising=False)
        sw.sw_set_tile(0)
        sw.sw_set_wave(0)


def test_cross_pass_wavefront_matches_oracle():
    """The cross-pass wavefront (one launch runs every query pass; an item's
    pass p trails pass p-1 through the boundary buffer and the score chain,
    synchronised by published progress) gives the same scores as the oracle:
    few long sequences (the case it exists for), a random mix with flagged
    sequences, several tiles, and auto mode choosing it by itself."""
    rng = np.random.default_rng(2718)
    dbs = [
        [si.rr_residues(rng, int(L)) for L in rng.integers(3000, 12000, 9)],
        [si.rr_residues(rng, int(L)) for L in rng.integers(0, 700, 500)] + [encode("W" * 3100)] * 3,
    ]
    queries = [si.rr_residues(rng, 1700), encode("W" * 3200 + "A" * 50), si.rr_residues(rng, 5478)]
    try:
        for di, seqs in enumerate(dbs):
            db = _db(seqs)
            sw.sw_db_load(db.residues, db.offsets)
            for q in queries:
                exp = oracle.batch(q, db.residues, db.offsets, BLOSUM62, 10, 2)
                for G, R in ((0, 0), (16, 16), (32, 8), (32, 29)):
                    sw.sw_set_tile(G, R)
                    sw.sw_set_wave(1)
                    got = sw.sw_search(q, BLOSUM62, 10, 2)
                    st = sw.sw_last_stats()
                    assert st["wave"] == (1 if st["passes"] > 1 else 0), (di, len(q), G, R, st)
                    assert (got == exp).all(), (di, len(q), G, R, np.nonzero(got != exp)[0][:5])
                    idx, sc = sw.sw_topk(5)
                    eidx, esc = oracle.topk(exp, 5)
                    assert (idx == eidx).all() and (sc == esc).all()
                # auto mode on the few-long-sequences database picks the wavefront
                sw.sw_set_tile(0)
                sw.sw_set_wave(0)
                got = sw.sw_search(q, BLOSUM62, 10, 2)
                assert (got == exp).all()
                if di == 0 and len(q) >= 8 * 256:   # >= 8 passes of 32x8 tiles (api.cu auto rule)
                    assert sw.sw_last_stats()["wave"] == 1
    finally:
        sw.sw_set_tile(0)
        sw.sw_set_wave(0)



def test_lat_tiles_are_exact():
    """Latency tiles (small R, 256 threads, one CTA per SM; chosen when one
    long item's critical path bounds the pass): every one, forced, on random
    databases with random matrices and gaps, multi-pass queries
    (boundary-reading launches) and saturating sequences (s32 re-scoring)."""
    rng = np.random.default_rng(4711)
    seqs = [rng.integers(0, 24, int(L)).astype(np.uint8) for L in rng.integers(0, 900, 300)]
    seqs += [si.rr_residues(rng, 4000), encode("W" * 3100), np.full(700, 3, np.uint8)]
    db = _db(seqs)
    sw.sw_db_load(db.residues, db.offsets)
    try:
        sw.sw_set_latency_mode(1)
        for G, R in ((32, 3), (32, 4), (32, 5), (32, 6), (32, 8), (16, 9)):
            assert sw.sw_tile_supported(G, R, lat=True)
            sw.sw_set_tile(G, R)
            for trial in range(3):
                m = int(rng.integers(1, 1800)) if trial else 3100
                q = rng.integers(0, 24, m).astype(np.uint8) if trial else encode("W" * 3100)
                M = BLOSUM62 if trial != 1 else si.random_symmetric_matrix(rng)
                go, ge = (10, 2) if trial != 2 else (0, int(rng.integers(0, 5)))
                got = sw.sw_search(q, M, go, ge)
                st = sw.sw_last_stats()
                assert st["lat"] == 1 and st["G"] == G and st["R"] == R, st
                exp = oracle.batch(q, db.residues, db.offsets, M, go, ge)
                bad = np.nonzero(got != exp)[0]
                assert bad.size == 0, (G, R, trial, m, bad[:5], got[bad[:5]], exp[bad[:5]])
        # automatic choice on configs[0] (a small database with one long item)
        sw.sw_set_tile(0)
        sw.sw_set_latency_mode(0)
        w = si.config0()
        sw.sw_db_load(w.db.residues, w.db.offsets)
        got = sw.sw_search(w.queries[0], BLOSUM62, 10, 2)
        exp = oracle.batch(w.queries[0], w.db.residues, w.db.offsets, BLOSUM62, 10, 2)
        assert (got == exp).all()
    finally:
        sw.sw_set_tile(0)
        sw.sw_set_latency_mode(0)


def test_score_profile_tiles_are_exact():
    """Score profile (sw_set_profile(2)): P(r) = SP[pair][q_r]
    read per row at the lane's query letter.  Every score-profile tile, forced,
    on random databases with random (also asymmetric) matrices, random gaps,
    multi-pass queries and saturating sequences; then the automatic switch."""
    rng = np.random.default_rng(1650)
    seqs = [rng.integers(0, 24, int(L)).astype(np.uint8) for L in rng.integers(0, 700, 400)]
    seqs += [si.rr_residues(rng, 3000), encode("W" * 3100), np.full(500, 7, np.uint8)]
    db = _db(seqs)
    sw.sw_db_load(db.residues, db.offsets)
    try:
        sw.sw_set_profile(2)
        for G in (8, 16, 32):
            for R in (8, 12, 16, 20):
                assert sw.sw_tile_supported(G, R, sp=True)
                sw.sw_set_tile(G, R)
                for trial in range(2):
                    m = [3100, int(rng.integers(1, 2500))][trial]
                    q = encode("W" * 3100) if trial == 0 else rng.integers(0, 24, m).astype(np.uint8)
                    M = BLOSUM62 if trial == 0 else (si.random_symmetric_matrix(rng) if G != 16
                                                     else rng.integers(-8, 12, (24, 24)).astype(np.int8))
                    go, ge = (10, 2) if trial == 0 else (int(rng.integers(0, 16)), int(rng.integers(0, 6)))
                    got = sw.sw_search(q, M, go, ge)
                    st = sw.sw_last_stats()
                    assert st["profile"] == 2 and st["G"] == G and st["R"] == R, st
                    exp = oracle.batch(q, db.residues, db.offsets, M, go, ge)
                    bad = np.nonzero(got != exp)[0]
                    assert bad.size == 0, (G, R, trial, m, bad[:5], got[bad[:5]], exp[bad[:5]])
        sw.sw_set_tile(0)
        q = si.rr_residues(rng, 464)
        got = sw.sw_search(q, BLOSUM62, 10, 2)       # automatic SP tile
        assert sw.sw_last_stats()["profile"] == 2
        assert (got == oracle.batch(q, db.residues, db.offsets, BLOSUM62, 10, 2)).all()
        sw.sw_set_profile(0)
        sw.sw_search(q, BLOSUM62, 10, 2)
        assert sw.sw_last_stats()["profile"] == 1   # the measured switch picks QP
    finally:
        sw.sw_set_tile(0)
        sw.sw_set_profile(0)


def test_rows_mode_matches_oracle():
    """Rows mode: the long sequences of a database (one per half
    of the leading items) scored with the sequence along the rows and the query
    as the column stream, passes as a wavefront.  Random
    and asymmetric matrices, zero gap-open, sequences of odd count (an empty
    half), saturating sequences (flag, carry propagation, 32-bit re-scoring),
    query lengths around the stream's 4-column rounding, and one 35,000-residue
    sequence (137 passes).  (Used on request only: sw_set_rows_mode(1).)"""
    rng = np.random.default_rng(2048)
    longs = [si.rr_residues(rng, int(L)) for L in rng.integers(600, 9000, 11)]
    longs += [encode("W" * 3100), encode("W" * 2990 + "A" * 20)]
    shorts = [si.rr_residues(rng, int(L)) for L in rng.integers(0, 200, 300)]
    db = _db(longs + shorts)
    sw.sw_db_load(db.residues, db.offsets)
    try:
        for mode in (1,):
            sw.sw_set_rows_mode(mode)
            for trial, m in enumerate((1, 2, 3, 4, 5, 37, 144, 299)):
                q = rng.integers(0, 24, m).astype(np.uint8) if trial % 3 else si.rr_residues(rng, m)
                M = (BLOSUM62, si.random_symmetric_matrix(rng), rng.integers(-6, 12, (24, 24)).astype(np.int8))[trial % 3]
                go, ge = ((10, 2), (0, 1), (int(rng.integers(0, 16)), int(rng.integers(0, 6))))[trial % 3]
                got = sw.sw_search(q, M, go, ge)
                st = sw.sw_last_stats()
                exp = oracle.batch(q, db.residues, db.offsets, M, go, ge)
                bad = np.nonzero(got != exp)[0]
                assert bad.size == 0, (mode, m, bad[:5], got[bad[:5]], exp[bad[:5]])
                assert st["rows_pairs"] > 0, (mode, m, st)
        # saturating: the W runs score 34,100 / 32,890 against a W query
        sw.sw_set_rows_mode(1)
        q = encode("W" * 3200)
        got = sw.sw_search(q, BLOSUM62, 10, 2)
        st = sw.sw_last_stats()
        exp = oracle.batch(q, db.residues, db.offsets, BLOSUM62, 10, 2)
        assert (got == exp).all() and _flags_ok(st, exp) and st["flagged"] >= 2
        # configs[0] in rows mode (on request) and without
        sw.sw_set_rows_mode(1)
        w = si.config0()
        sw.sw_db_load(w.db.residues, w.db.offsets)
        got = sw.sw_search(w.queries[0], BLOSUM62, 10, 2)
        assert sw.sw_last_stats()["rows_pairs"] > 0
        assert (got == oracle.batch(w.queries[0], w.db.residues, w.db.offsets, BLOSUM62, 10, 2)).all()
        sw.sw_set_rows_mode(-1)
        got2 = sw.sw_search(w.queries[0], BLOSUM62, 10, 2)
        assert sw.sw_last_stats()["rows_pairs"] == 0 and (got2 == got).all()
        # one long sequence (137 passes over one CTA's 8 warps, the warp 7 ->
        # warp 0 hand-over through global memory many times)
        sw.sw_set_rows_mode(1)
        db1 = _db([si.rr_residues(rng, 35000), si.rr_residues(rng, 300)])
        sw.sw_db_load(db1.residues, db1.offsets)
        q = si.rr_residues(rng, 100)
        got = sw.sw_search(q, BLOSUM62, 10, 2)
        assert sw.sw_last_stats()["rows_pairs"] > 0
        assert (got == oracle.batch(q, db1.residues, db1.offsets, BLOSUM62, 10, 2)).all()
    finally:
        sw.sw_set_rows_mode(0)
