"""CPU oracle for Smith-Waterman database search (Section 2, Eqs. 1-4).

TEST INFRASTRUCTURE.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_1702_07195_b200``) never imports it, and
this package never imports the product path; the two share no code.  The only
module both sides use is ``sw_inputs`` (seeded input generators, no method
arithmetic).

Functions and the passage each follows:

* ``score(q, d, M, open, ext)``    -- Eqs. 1-3 two-row, max over H
* ``full(q, d, M, open, ext)``     -- the full H, E, F matrices of Eqs. 1-3
* ``batch(q, db, M, open, ext)``   -- one score per database sequence (the SW
  stage), one sequence per task on a thread pool
* ``topk(scores, k)``              -- the sorting stage, descending,
  ties by ascending index (reading R5)
* ``gcups(qres, dres, t)``         -- Eq. 4

Pins: tests/test_oracle_pins.py.  Parity unpinned: none.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sw_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

ALPHA = 24


def build(force: bool = False) -> str:
    """Compile the C oracle (plain gcc -O2, no vectorisation tricks)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-pthread",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        i64, p = ctypes.c_int64, ctypes.c_void_p
        lib.oracle_sw_score.restype = i64
        lib.oracle_sw_score.argtypes = [p, i64, p, i64, p, i64, i64]
        lib.oracle_sw_full.restype = i64
        lib.oracle_sw_full.argtypes = [p, i64, p, i64, p, i64, i64, p, p, p]
        lib.oracle_sw_batch.restype = ctypes.c_int
        lib.oracle_sw_batch.argtypes = [p, i64, p, p, p, i64, p, i64, i64, p, ctypes.c_int]
        _lib = lib
    return _lib


def _u8(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint8))


def _mat(M) -> np.ndarray:
    M = np.ascontiguousarray(np.asarray(M, dtype=np.int8))
    assert M.shape == (ALPHA, ALPHA), M.shape
    return M


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p) if a.size else ctypes.c_void_p(0)


def score(q, d, M, gap_open: int, gap_extend: int) -> int:
    """Optimal local alignment score of query q (rows) vs subject d (columns)."""
    q, d, M = _u8(q), _u8(d), _mat(M)
    s = _load().oracle_sw_score(_ptr(q), q.size, _ptr(d), d.size, _ptr(M), int(gap_open), int(gap_extend))
    if s < 0:
        raise MemoryError("oracle_sw_score")
    return int(s)


def full(q, d, M, gap_open: int, gap_extend: int):
    """(H, E, F, best): the full (m+1)x(n+1) int64 matrices of Eqs. 1-3."""
    q, d, M = _u8(q), _u8(d), _mat(M)
    m, n = q.size, d.size
    H = np.zeros((m + 1, n + 1), dtype=np.int64)
    E = np.zeros_like(H)
    F = np.zeros_like(H)
    best = _load().oracle_sw_full(_ptr(q), m, _ptr(d), n, _ptr(M), int(gap_open), int(gap_extend),
                                  _ptr(H), _ptr(E), _ptr(F))
    return H, E, F, int(best)


def batch(q, residues, offsets, M, gap_open: int, gap_extend: int, idx=None,
          threads: int | None = None) -> np.ndarray:
    """int64 scores of q against database sequences (all, or those in idx)."""
    q, M = _u8(q), _mat(M)
    residues = _u8(residues)
    offsets = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
    if idx is None:
        count = offsets.size - 1
        idx_arr = None
    else:
        idx_arr = np.ascontiguousarray(np.asarray(idx, dtype=np.int64))
        count = idx_arr.size
    out = np.zeros(count, dtype=np.int64)
    if count == 0:
        return out
    nth = int(threads or os.cpu_count() or 1)
    rc = _load().oracle_sw_batch(_ptr(q), q.size, _ptr(residues), _ptr(offsets),
                                 _ptr(idx_arr) if idx_arr is not None else ctypes.c_void_p(0),
                                 count, _ptr(M), int(gap_open), int(gap_extend), _ptr(out), nth)
    if rc != 0:
        raise MemoryError("oracle_sw_batch")
    return out


def topk(scores, k: int):
    """Sorting stage: indices and scores of the k best, score
    descending, ties by ascending index.  k >= len(scores) gives the full order."""
    scores = np.asarray(scores, dtype=np.int64)
    order = np.lexsort((np.arange(scores.size), -scores))
    order = order[: max(0, min(int(k), scores.size))]
    return order.astype(np.int64), scores[order]


def gcups(query_residues: int, db_residues: int, seconds: float) -> float:
    """Eq. 4: |Q| x |D| / (t x 1e9)."""
    if seconds <= 0:
        raise ValueError("t must be > 0")
    return float(query_residues) * float(db_residues) / (seconds * 1e9)
