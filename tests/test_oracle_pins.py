"""Pins of the CPU oracle against things other than itself (task rule 3).

Every function of oracle/ is pinned here by at least one of: values printed
in SPEC.md / worked by hand (tests/golden/), brute-force enumeration, textbook
reductions (LCS, Kadane), the -inf-boundary textbook recurrence, closed forms
and invariants.  A plausible oracle bug (dropped E or F term, Goe vs Ge swap,
wrong diagonal index, transposed matrix, missing 0 floor) fails one of them.
"""
from __future__ import annotations

import os

import numpy as np
import pytest
from hypothesis import given, settings, HealthCheck, strategies as st

import oracle
from sw_inputs import BLOSUM62, CODE, encode, random_symmetric_matrix, rng_for, rr_residues
from tests.brute import brute_force_score, expand, gotoh_neg_inf, kadane_best_diagonal, lcs_length

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden_rows(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for ln in f:
            ln = ln.strip()
            if not ln or ln.startswith("#"):
                continue
            rows.append(ln.split("\t"))
    return rows


HAND = _golden_rows("hand_examples.txt")


@pytest.mark.parametrize("row", HAND, ids=[f"{r[0][:12]}-{r[1][:16]}-{r[2]}/{r[3]}" for r in HAND])
def test_hand_examples(oracle_lib, row):
    q, d, go, ge, expected = expand(row[0]), expand(row[1]), int(row[2]), int(row[3]), int(row[4])
    assert oracle.score(encode(q), encode(d), BLOSUM62, go, ge) == expected


def test_full_matrix_A_vs_A(oracle_lib):
    # H = [[0,0],[0,4]]
    H, E, F, best = oracle.full(encode("A"), encode("A"), BLOSUM62, 10, 2)
    assert H.tolist() == [[0, 0], [0, 4]]
    assert best == 4


def test_full_matrix_boundaries_and_max(oracle_lib):
    rng = np.random.default_rng(5)
    for _ in range(50):
        m, n = rng.integers(1, 12, size=2)
        q, d = rng.integers(0, 20, m).astype(np.uint8), rng.integers(0, 20, n).astype(np.uint8)
        M = random_symmetric_matrix(rng)
        go, ge = rng.integers(0, 16, size=2)
        H, E, F, best = oracle.full(q, d, M, go, ge)
        assert (H[0, :] == 0).all() and (H[:, 0] == 0).all()   # PAPER.md:66 initialisation
        assert (H >= 0).all()
        assert best == H.max() == oracle.score(q, d, M, go, ge)


# ---- brute force (P2) ---------------------------------------------------
_small = st.integers(min_value=0, max_value=5)


@settings(max_examples=300, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(m=_small, n=_small, seed=st.integers(0, 2**32 - 1), go=st.integers(0, 15), ge=st.integers(0, 15),
       sym=st.booleans())
def test_brute_force(oracle_lib, m, n, seed, go, ge, sym):
    rng = np.random.default_rng(seed)
    # few letters so that matches (and therefore gaps between them) are common
    q = rng.integers(0, 4, m).astype(np.uint8)
    d = rng.integers(0, 4, n).astype(np.uint8)
    M = random_symmetric_matrix(rng) if sym else rng.integers(-4, 12, size=(24, 24)).astype(np.int8)
    assert oracle.score(q, d, M, go, ge) == brute_force_score(q, d, M, go, ge)


def test_brute_force_adjacent_gap_runs(oracle_lib):
    # A case where the optimum uses an I run immediately followed by a D run:
    # q = A C, d = G A ... built so that skipping one letter on each side is best.
    M = np.full((24, 24), -4, dtype=np.int8)
    a, c, g, t = 0, 1, 2, 3
    M[a, a] = 10
    M[c, c] = 10
    q = np.array([a, g, c], dtype=np.uint8)
    d = np.array([a, t, c], dtype=np.uint8)
    # mismatch G/T costs -4; a D+I pair costs 2*(0+1) = 2 with open 0, extend 1
    assert brute_force_score(q, d, M, 0, 1) == 18
    assert oracle.score(q, d, M, 0, 1) == 18


# ---- textbook reductions (P3) -------------------------------------------
@settings(max_examples=100, deadline=None)
@given(seed=st.integers(0, 2**32 - 1), m=st.integers(0, 40), n=st.integers(0, 40))
def test_lcs_reduction(oracle_lib, seed, m, n):
    # +1 on identity, -1 otherwise, zero gap costs: mismatches never help
    # (an I+D pair costs 0), so the score is the LCS length.
    rng = np.random.default_rng(seed)
    q = rng.integers(0, 4, m).astype(np.uint8)
    d = rng.integers(0, 4, n).astype(np.uint8)
    M = -np.ones((24, 24), dtype=np.int8)
    np.fill_diagonal(M, 1)
    assert oracle.score(q, d, M, 0, 0) == lcs_length(q.tolist(), d.tolist())


@settings(max_examples=100, deadline=None)
@given(seed=st.integers(0, 2**32 - 1), m=st.integers(0, 30), n=st.integers(0, 30))
def test_kadane_reduction(oracle_lib, seed, m, n):
    # Goe > smax*min(m,n): no gapped alignment can beat an ungapped one.
    rng = np.random.default_rng(seed)
    q = rng.integers(0, 20, m).astype(np.uint8)
    d = rng.integers(0, 20, n).astype(np.uint8)
    M = random_symmetric_matrix(rng)
    assert oracle.score(q, d, M, 400, 1) == kadane_best_diagonal(q, d, M)


@settings(max_examples=100, deadline=None)
@given(seed=st.integers(0, 2**32 - 1), m=st.integers(0, 25), n=st.integers(0, 25),
       go=st.integers(0, 15), ge=st.integers(0, 15))
def test_neg_inf_boundary_equivalence(oracle_lib, seed, m, n, go, ge):
    # Reading C2: the paper's zero initialisation of E and F gives the same H
    # as the textbook -inf initialisation whenever Ge >= 0.
    rng = np.random.default_rng(seed)
    q = rng.integers(0, 20, m).astype(np.uint8)
    d = rng.integers(0, 20, n).astype(np.uint8)
    M = random_symmetric_matrix(rng)
    assert oracle.score(q, d, M, go, ge) == gotoh_neg_inf(q, d, M, go, ge)


def test_all_nonpositive_matrix_scores_zero(oracle_lib):
    rng = np.random.default_rng(11)
    for _ in range(30):
        M = -rng.integers(0, 5, size=(24, 24)).astype(np.int8)
        q = rng.integers(0, 24, 30).astype(np.uint8)
        d = rng.integers(0, 24, 40).astype(np.uint8)
        assert oracle.score(q, d, M, 0, 0) == 0


def test_blosum62_self_score_closed_form(oracle_lib):
    # P3: for BLOSUM62 over the 20 standard letters the diagonal is the strict
    # row maximum and gaps only cost, so score(x, x) = sum of SM(x_i, x_i).
    rng = rng_for(99, 1)
    for L in (1, 2, 7, 50, 333):
        x = rr_residues(rng, L)
        assert oracle.score(x, x, BLOSUM62, 10, 2) == int(BLOSUM62[x, x].astype(np.int64).sum())


# ---- invariants (P4) ----------------------------------------------------
@settings(max_examples=150, deadline=None)
@given(seed=st.integers(0, 2**32 - 1), m=st.integers(0, 40), n=st.integers(0, 40),
       go=st.integers(0, 15), ge=st.integers(0, 15))
def test_invariants(oracle_lib, seed, m, n, go, ge):
    rng = np.random.default_rng(seed)
    q = rng.integers(0, 20, m).astype(np.uint8)
    d = rng.integers(0, 20, n).astype(np.uint8)
    M = random_symmetric_matrix(rng)
    s = oracle.score(q, d, M, go, ge)
    assert s >= 0
    # symmetry under swapping the sequences (transpose M; symmetric here)
    assert oracle.score(d, q, M.T.copy(), go, ge) == s
    # asymmetric matrix: swapping sequences needs the transposed matrix
    A = rng.integers(-4, 12, size=(24, 24)).astype(np.int8)
    assert oracle.score(q, d, A, go, ge) == oracle.score(d, q, A.T.copy(), go, ge)
    # non-increasing in gap_open and in gap_extend
    assert oracle.score(q, d, M, go + 1, ge) <= s
    assert oracle.score(q, d, M, go, ge + 1) <= s
    # non-decreasing when residues are appended / prepended
    extra = rng.integers(0, 20, 3).astype(np.uint8)
    assert oracle.score(np.concatenate([q, extra]), d, M, go, ge) >= s
    assert oracle.score(q, np.concatenate([extra, d]), M, go, ge) >= s
    # >= best ungapped diagonal segment
    assert s >= kadane_best_diagonal(q, d, M)
    # <= min(sum of row maxima over q, sum of column maxima over d)
    ub_q = int(np.maximum(M[q, :].max(axis=1), 0).sum()) if m else 0
    ub_d = int(np.maximum(M[:, d].max(axis=0), 0).sum()) if n else 0
    assert s <= min(ub_q, ub_d)


def test_empty_sequences_score_zero(oracle_lib):
    q = encode("ARND")
    assert oracle.score(q, np.zeros(0, np.uint8), BLOSUM62, 10, 2) == 0
    assert oracle.score(np.zeros(0, np.uint8), q, BLOSUM62, 10, 2) == 0


# ---- batch, sort stage, Eq. 4 -------------------------------------------
def test_batch_matches_single_and_thread_invariance(oracle_lib):
    rng = np.random.default_rng(3)
    seqs = [rng.integers(0, 20, int(L)).astype(np.uint8) for L in rng.integers(0, 120, 300)]
    offs = np.zeros(len(seqs) + 1, np.int64)
    offs[1:] = np.cumsum([len(s) for s in seqs])
    res = np.concatenate(seqs).astype(np.uint8)
    q = rng.integers(0, 20, 77).astype(np.uint8)
    single = np.array([oracle.score(q, s, BLOSUM62, 10, 2) for s in seqs])
    for th in (1, 2, 4, 8):
        assert (oracle.batch(q, res, offs, BLOSUM62, 10, 2, threads=th) == single).all()
    idx = np.array([5, 0, 299, 17])
    assert (oracle.batch(q, res, offs, BLOSUM62, 10, 2, idx=idx) == single[idx]).all()


def test_topk_tie_example():
    # scores [3,9,9,1] -> order [1,2,0,3]
    idx, sc = oracle.topk(np.array([3, 9, 9, 1]), 4)
    assert idx.tolist() == [1, 2, 0, 3]
    assert sc.tolist() == [9, 9, 3, 1]
    idx, sc = oracle.topk(np.array([3, 9, 9, 1]), 2)
    assert idx.tolist() == [1, 2]
    assert oracle.topk(np.array([5]), 10)[0].tolist() == [0]


@pytest.mark.parametrize("row", _golden_rows("gcups.txt"))
def test_gcups_eq4(row):
    q, dres, t, expected = int(row[0]), int(row[1]), float(row[2]), float(row[3])
    assert oracle.gcups(q, dres, t) == pytest.approx(expected, rel=1e-9)
    with pytest.raises(ValueError):
        oracle.gcups(q, dres, 0.0)
