"""Independent pins for the oracle (test-only; imports nothing from oracle/ or
the product package).

* brute_force_score -- exhaustive enumeration of every local alignment of
  tiny sequences (BASELINE.json north_star "brute-force
  enumeration of all local alignments").  An alignment is a path of columns
  M (q_i aligned to d_j), I (d_j against a gap) and D (q_i against a gap)
  starting anywhere; it scores the sum of SM over M columns minus, for every
  maximal run of k consecutive I columns or k consecutive D columns,
  gap_open + k*gap_extend (Goe = open + extend for the
  first gap position, Ge = extend for each further one).  Adjacent I and D
  runs are allowed.  The score is the maximum over all alignments including
  the empty one (0).
* lcs_length -- textbook longest-common-subsequence DP.
* kadane_best_diagonal -- best ungapped segment (max-subarray on every
  diagonal of the substitution scores).
* gotoh_neg_inf -- textbook Gotoh with -infinity E/F boundaries (the usual
  initialisation, for the C2 reading).
"""
from __future__ import annotations

import sys

import numpy as np


def brute_force_score(q, d, M, gap_open: int, gap_extend: int) -> int:
    q = [int(x) for x in q]
    d = [int(x) for x in d]
    M = np.asarray(M, dtype=np.int64)
    m, n = len(q), len(d)
    best = 0
    sys.setrecursionlimit(max(1000, 4 * (m + n) + 100))

    def dfs(i: int, j: int, score: int, last: str) -> None:
        nonlocal best
        if score > best:
            best = score
        if i < m and j < n:
            dfs(i + 1, j + 1, score + int(M[q[i], d[j]]), "M")
        if j < n:
            cost = gap_extend if last == "I" else gap_open + gap_extend
            dfs(i, j + 1, score - cost, "I")
        if i < m:
            cost = gap_extend if last == "D" else gap_open + gap_extend
            dfs(i + 1, j, score - cost, "D")

    for i0 in range(m + 1):
        for j0 in range(n + 1):
            dfs(i0, j0, 0, "")
    return best


def lcs_length(a, b) -> int:
    a = list(a)
    b = list(b)
    L = [[0] * (len(b) + 1) for _ in range(len(a) + 1)]
    for i in range(1, len(a) + 1):
        for j in range(1, len(b) + 1):
            if a[i - 1] == b[j - 1]:
                L[i][j] = L[i - 1][j - 1] + 1
            else:
                L[i][j] = max(L[i - 1][j], L[i][j - 1])
    return L[len(a)][len(b)]


def kadane_best_diagonal(q, d, M) -> int:
    """max(0, best sum of a contiguous run along any diagonal of SM(q_i, d_j))."""
    M = np.asarray(M, dtype=np.int64)
    m, n = len(q), len(d)
    best = 0
    for off in range(-(m - 1), n):
        cur = 0
        for i in range(m):
            j = i + off
            if 0 <= j < n:
                cur = max(0, cur + int(M[q[i], d[j]]))
                best = max(best, cur)
    return best


def gotoh_neg_inf(q, d, M, gap_open: int, gap_extend: int) -> int:
    """Textbook Gotoh local alignment with E = F = -inf on the boundary."""
    NEG = -(1 << 60)
    M = np.asarray(M, dtype=np.int64)
    m, n = len(q), len(d)
    goe, ge = gap_open + gap_extend, gap_extend
    H = [[0] * (n + 1) for _ in range(m + 1)]
    E = [[NEG] * (n + 1) for _ in range(m + 1)]
    F = [[NEG] * (n + 1) for _ in range(m + 1)]
    best = 0
    for i in range(1, m + 1):
        for j in range(1, n + 1):
            E[i][j] = max(E[i][j - 1] - ge, H[i][j - 1] - goe)
            F[i][j] = max(F[i - 1][j] - ge, H[i - 1][j] - goe)
            H[i][j] = max(0, H[i - 1][j - 1] + int(M[q[i - 1], d[j - 1]]), E[i][j], F[i][j])
            best = max(best, H[i][j])
    return best


def expand(spec: str) -> str:
    """'W{5}A{3}' -> 'WWWWWAAA'."""
    out = []
    i = 0
    while i < len(spec):
        c = spec[i]
        i += 1
        if i < len(spec) and spec[i] == "{":
            j = spec.index("}", i)
            out.append(c * int(spec[i + 1:j]))
            i = j + 1
        else:
            out.append(c)
    return "".join(out)
