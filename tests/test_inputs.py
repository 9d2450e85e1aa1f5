"""Checks of the shared input module sw_inputs (no method arithmetic there).

BLOSUM62 is an input of sw_search; the oracle and the CUDA path both receive
it, so a typo in it could never show up as a parity failure.
These checks pin the embedded table to properties of the published matrix.
"""
import numpy as np
import pytest

import sw_inputs as si

B = si.BLOSUM62.astype(np.int64)
C = si.CODE


def test_blosum62_shape_symmetry_range():
    assert B.shape == (24, 24)
    assert (B == B.T).all()
    std = B[:20, :20]
    assert std.min() == -4 and std.max() == 11


def test_blosum62_spec_values():
    # SPEC.md:68
    assert B[C["A"], C["A"]] == 4
    assert B[C["W"], C["W"]] == 11
    assert B[C["A"], C["V"]] == 0


def test_blosum62_diagonal():
    diag = {"A": 4, "R": 5, "N": 6, "D": 6, "C": 9, "Q": 5, "E": 5, "G": 6, "H": 8, "I": 4,
            "L": 4, "K": 5, "M": 5, "F": 6, "P": 7, "S": 4, "T": 5, "W": 11, "Y": 7, "V": 4}
    for a, v in diag.items():
        assert B[C[a], C[a]] == v, a
    # the diagonal is the strict row maximum over the 20 standard letters
    std = B[:20, :20]
    for i in range(20):
        row = std[i].copy()
        d = row[i]
        row[i] = -100
        assert d > row.max()


def test_blosum62_ambiguity_codes_and_stop():
    # '*' scores -4 against everything but itself (1); B, Z are the N/D and Q/E merges
    star = C["*"]
    assert (B[star, :23] == -4).all() and B[star, star] == 1
    assert B[C["B"], C["N"]] == 3 and B[C["B"], C["D"]] == 4
    assert B[C["Z"], C["Q"]] == 3 and B[C["Z"], C["E"]] == 4


def test_blosum62_negative_expected_score():
    # a log-odds matrix has a negative expected score under background
    # frequencies (otherwise local alignment would degenerate to global)
    p = si.RR_FREQ
    e = float(p @ B[:20, :20] @ p)
    assert -1.5 < e < -0.3


def test_rr_frequencies_and_sampler():
    assert abs(si.RR_FREQ.sum() - 1.0) < 1e-12
    x = si.rr_residues(si.rng_for(0, 9), 2_000_000)
    assert x.max() < 20
    f = np.bincount(x, minlength=20) / x.size
    assert np.abs(f - si.RR_FREQ).max() < 2e-3


def test_lengths_distribution():
    L = si.lognormal_lengths(si.rng_for(0, 0), 400_000, 1, 10**9)
    assert abs(np.median(L) - 150) < 3
    assert abs(L.mean() - 200) < 3
    L2 = si.lognormal_lengths(si.rng_for(0, 0), 1000, 8, 2000)
    assert L2.min() >= 8 and L2.max() <= 2000


def test_generators_deterministic():
    a = si.config0(scale=0.05)
    b = si.config0(scale=0.05)
    assert (a.db.residues == b.db.residues).all() and (a.db.offsets == b.db.offsets).all()
    assert (a.queries[0] == b.queries[0]).all()


def test_config_shapes_small_scale():
    w0 = si.config0()
    assert w0.db.count == 10_000 and len(w0.queries[0]) == 144
    assert 1.85e6 < w0.db.total_residues < 2.1e6
    w3 = si.config3(scale=1e-4)
    assert [len(q) for q in w3.queries] == si.CFG3_QUERY_LENGTHS
    assert si.CFG3_QUERY_LENGTHS[0] == 144 and si.CFG3_QUERY_LENGTHS[-1] == 5478
    assert sum(si.CFG3_QUERY_LENGTHS) == 56_220
    w2 = si.config2(scale=1e-4)
    assert w2.db.lengths().max() == 35_000


def test_config4_structure():
    w = si.config4(scale=0.01)
    q = w.queries[0]
    assert len(q) == 5478
    assert 0.55 < (q == C["W"]).mean() < 0.65
    L = w.db.lengths()
    assert len(w.planted) == 40
    assert (L[w.planted] == 5478).all()
    # planted copies differ from the query by 5-20% substitutions, no indels
    for i in w.planted:
        frac = (w.db.seq(int(i)) != q).mean()
        assert 0.03 < frac < 0.23
    assert ((L >= 5000) & (L != 5478)).sum() >= 100


def test_config_db_subset_equals_full_generation():
    """bench.py's per-rank generation (sw_inputs.config_db_subset streams the
    residue generator and keeps only the shard) equals the full configuration's
    sub-database, across residue chunk boundaries (2^26)."""
    rng = np.random.default_rng(5)
    for k, sc in [(0, 1.0), (1, 0.4), (2, 0.005), (3, 0.005)]:
        w = si.make_config(k, scale=sc)
        assert np.array_equal(si.config_lengths(k, sc), w.db.lengths())
        assert all(np.array_equal(a, b) for a, b in zip(si.config_queries(k), w.queries))
        for frac in (0.5, 0.02):
            idx = np.sort(rng.choice(w.db.count, max(1, int(w.db.count * frac)), replace=False))
            sub = si.config_db_subset(k, idx, sc)
            ref = w.db.subset(idx)
            assert np.array_equal(sub.offsets, ref.offsets) and np.array_equal(sub.residues, ref.residues)
    # a sequence straddling the first 2^26-residue chunk boundary
    w = si.config1(scale=0.4)
    b = int(np.searchsorted(w.db.offsets, 1 << 26, side="right") - 1)
    sub = si.config_db_subset(1, np.array([b - 1, b, b + 1]), 0.4)
    for j, i in enumerate((b - 1, b, b + 1)):
        assert np.array_equal(sub.seq(j), w.db.seq(i))
