"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO Smith-Waterman arithmetic: it only defines the residue
alphabet, the BLOSUM62 table (an *input* of ``sw_search``), the Robinson &
Robinson background frequencies and the seeded generators for the five
BASELINE.json configurations.  Both ``oracle/`` (via tests) and the product
path (via tests / bench) consume what it produces; neither side's arithmetic
lives here (task rule ③: "only the seeded input generators serve both").

Recipe (DESIGN.md §"Input recipe"):

* RNG: ``numpy.random.Generator(PCG64(SeedSequence([1702, 7195, cfg, stream])))``,
  streams 0 lengths, 1 DB residues, 2 queries, 3 planting/positions,
  4 substitutions.
* residues: codes 0..19 (NCBI order ``ARNDCQEGHILKMFPSTWYV``) drawn i.i.d.
  from the Robinson-Robinson frequencies, quantised to 1/65536 through a
  65,536-entry lookup table (fast for 1.3 G draws; the quantisation error is
  < 2e-5 per letter).
* lengths: ``clip(rint(lognormal(ln 150, sqrt(2 ln(4/3)))), lo, hi)`` -> median
  150, mean 200 before clipping (BASELINE.json configs[0]).
* The paper's benchmark (Environmental NR 2016_11 searched with 20 Swiss-Prot
  queries) is not available; these synthetic inputs stand in
  for it with its shape (mean length ~200, ~1.3 G residues, BLOSUM62, gaps
  10/2).
"""
from __future__ import annotations

import dataclasses
import numpy as np

# --------------------------------------------------------------------------
# Alphabet (NCBI matrix order).  Codes 0..23.
# --------------------------------------------------------------------------
ALPHABET = "ARNDCQEGHILKMFPSTWYVBZX*"
ALPHA = 24
STANDARD = ALPHABET[:20]
CODE = {c: i for i, c in enumerate(ALPHABET)}

# --------------------------------------------------------------------------
# BLOSUM62 (Henikoff & Henikoff 1992), the matrix named at PAPER.md:179,
# standard NCBI 24x24 layout.  Rows = first letter, columns = second letter.
# Validated by tests/test_inputs.py (symmetry, SPEC.md:68 values, diagonal
# strict row maximum, negative expected score).
# --------------------------------------------------------------------------
_BLOSUM62_TEXT = """
   A  R  N  D  C  Q  E  G  H  I  L  K  M  F  P  S  T  W  Y  V  B  Z  X  *
A  4 -1 -2 -2  0 -1 -1  0 -2 -1 -1 -1 -1 -2 -1  1  0 -3 -2  0 -2 -1  0 -4
R -1  5  0 -2 -3  1  0 -2  0 -3 -2  2 -1 -3 -2 -1 -1 -3 -2 -3 -1  0 -1 -4
N -2  0  6  1 -3  0  0  0  1 -3 -3  0 -2 -3 -2  1  0 -4 -2 -3  3  0 -1 -4
D -2 -2  1  6 -3  0  2 -1 -1 -3 -4 -1 -3 -3 -1  0 -1 -4 -3 -3  4  1 -1 -4
C  0 -3 -3 -3  9 -3 -4 -3 -3 -1 -1 -3 -1 -2 -3 -1 -1 -2 -2 -1 -3 -3 -2 -4
Q -1  1  0  0 -3  5  2 -2  0 -3 -2  1  0 -3 -1  0 -1 -2 -1 -2  0  3 -1 -4
E -1  0  0  2 -4  2  5 -2  0 -3 -3  1 -2 -3 -1  0 -1 -3 -2 -2  1  4 -1 -4
G  0 -2  0 -1 -3 -2 -2  6 -2 -4 -4 -2 -3 -3 -2  0 -2 -2 -3 -3 -1 -2 -1 -4
H -2  0  1 -1 -3  0  0 -2  8 -3 -3 -1 -2 -1 -2 -1 -2 -2  2 -3  0  0 -1 -4
I -1 -3 -3 -3 -1 -3 -3 -4 -3  4  2 -3  1  0 -3 -2 -1 -3 -1  3 -3 -3 -1 -4
L -1 -2 -3 -4 -1 -2 -3 -4 -3  2  4 -2  2  0 -3 -2 -1 -2 -1  1 -4 -3 -1 -4
K -1  2  0 -1 -3  1  1 -2 -1 -3 -2  5 -1 -3 -1  0 -1 -3 -2 -2  0  1 -1 -4
M -1 -1 -2 -3 -1  0 -2 -3 -2  1  2 -1  5  0 -2 -1 -1 -1 -1  1 -3 -1 -1 -4
F -2 -3 -3 -3 -2 -3 -3 -3 -1  0  0 -3  0  6 -4 -2 -2  1  3 -1 -3 -3 -1 -4
P -1 -2 -2 -1 -3 -1 -1 -2 -2 -3 -3 -1 -2 -4  7 -1 -1 -4 -3 -2 -2 -1 -2 -4
S  1 -1  1  0 -1  0  0  0 -1 -2 -2  0 -1 -2 -1  4  1 -3 -2 -2  0  0  0 -4
T  0 -1  0 -1 -1 -1 -1 -2 -2 -1 -1 -1 -1 -2 -1  1  5 -2 -2  0 -1 -1  0 -4
W -3 -3 -4 -4 -2 -2 -3 -2 -2 -3 -2 -3 -1  1 -4 -3 -2 11  2 -3 -4 -3 -2 -4
Y -2 -2 -2 -3 -2 -1 -2 -3  2 -1 -1 -2 -1  3 -3 -2 -2  2  7 -1 -3 -2 -1 -4
V  0 -3 -3 -3 -1 -2 -2 -3 -3  3  1 -2  1 -1 -2 -2  0 -3 -1  4 -3 -2 -1 -4
B -2 -1  3  4 -3  0  1 -1  0 -3 -4  0 -3 -3 -2  0 -1 -4 -3 -3  4  1 -1 -4
Z -1  0  0  1 -3  3  4 -2  0 -3 -3  1 -1 -3 -1  0 -1 -3 -2 -2  1  4 -1 -4
X  0 -1 -1 -1 -2 -1 -1 -1 -1 -1 -1 -1 -1 -1 -2  0  0 -2 -1 -1 -1 -1 -1 -4
* -4 -4 -4 -4 -4 -4 -4 -4 -4 -4 -4 -4 -4 -4 -4 -4 -4 -4 -4 -4 -4 -4 -4  1
"""


def _parse_matrix(text: str) -> np.ndarray:
    lines = [ln.split() for ln in text.strip().splitlines()]
    header = lines[0]
    assert "".join(header) == ALPHABET, header
    m = np.zeros((ALPHA, ALPHA), dtype=np.int8)
    for row in lines[1:]:
        a = CODE[row[0]]
        m[a, :] = [int(v) for v in row[1:]]
    return m


BLOSUM62 = _parse_matrix(_BLOSUM62_TEXT)
BLOSUM62.setflags(write=False)

# Gap penalties of the paper's experiments: open 10, extend 2;
# a gap of length k costs open + k*extend (Goe = open + extend).
GAP_OPEN = 10
GAP_EXTEND = 2

# --------------------------------------------------------------------------
# Robinson & Robinson (1991) background frequencies, ARNDCQEGHILKMFPSTWYV
# (BASELINE.json configs[0] "Robinson-Robinson background frequencies").
# --------------------------------------------------------------------------
RR_FREQ = np.array([
    0.07805, 0.05129, 0.04487, 0.05364, 0.01925, 0.04264, 0.06295, 0.07377, 0.02199, 0.05142,
    0.09019, 0.05744, 0.02243, 0.03856, 0.05203, 0.07120, 0.05841, 0.01330, 0.03216, 0.06441,
], dtype=np.float64)
RR_FREQ = RR_FREQ / RR_FREQ.sum()

_LUT_BITS = 16


def _rr_lut() -> np.ndarray:
    cum = np.cumsum(RR_FREQ)
    cum[-1] = 1.0
    u = (np.arange(1 << _LUT_BITS, dtype=np.float64) + 0.5) / float(1 << _LUT_BITS)
    return np.searchsorted(cum, u, side="right").astype(np.uint8)


_RR_LUT = _rr_lut()


def rng_for(cfg: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([1702, 7195, int(cfg), int(stream)])))


def rr_residues(rng: np.random.Generator, n: int, chunk: int = 1 << 26) -> np.ndarray:
    """n i.i.d. Robinson-Robinson residue codes (uint8, 0..19)."""
    out = np.empty(int(n), dtype=np.uint8)
    for s in range(0, int(n), chunk):
        e = min(int(n), s + chunk)
        u = rng.integers(0, 1 << _LUT_BITS, size=e - s, dtype=np.uint16)
        out[s:e] = _RR_LUT[u]
    return out


def lognormal_lengths(rng: np.random.Generator, count: int, lo: int, hi: int,
                      median: float = 150.0, mean: float = 200.0) -> np.ndarray:
    """clip(rint(lognormal(mu, sigma)), lo, hi) with the given median and mean."""
    mu = np.log(median)
    sigma = np.sqrt(2.0 * np.log(mean / median))
    x = rng.lognormal(mu, sigma, size=int(count))
    return np.clip(np.rint(x), lo, hi).astype(np.int64)


@dataclasses.dataclass
class Database:
    """A protein database as the C-ABI takes it: concatenated residue codes and
    count+1 offsets (sequence i is residues[offsets[i]:offsets[i+1]])."""
    residues: np.ndarray   # uint8 [sum n]
    offsets: np.ndarray    # int64 [count+1]

    @property
    def count(self) -> int:
        return int(self.offsets.shape[0] - 1)

    @property
    def total_residues(self) -> int:
        return int(self.offsets[-1])

    def seq(self, i: int) -> np.ndarray:
        return self.residues[self.offsets[i]:self.offsets[i + 1]]

    def lengths(self) -> np.ndarray:
        return np.diff(self.offsets)

    def subset(self, idx) -> "Database":
        idx = np.asarray(idx, dtype=np.int64)
        lens = self.lengths()[idx]
        offs = np.zeros(idx.shape[0] + 1, dtype=np.int64)
        np.cumsum(lens, out=offs[1:])
        res = np.empty(int(offs[-1]), dtype=np.uint8)
        for k, i in enumerate(idx):
            res[offs[k]:offs[k + 1]] = self.seq(int(i))
        return Database(res, offs)


def database_from_lengths(rng: np.random.Generator, lengths: np.ndarray) -> Database:
    offs = np.zeros(lengths.shape[0] + 1, dtype=np.int64)
    np.cumsum(lengths, out=offs[1:])
    return Database(rr_residues(rng, int(offs[-1])), offs)


def database_from_list(seqs) -> Database:
    seqs = [np.asarray(s, dtype=np.uint8) for s in seqs]
    offs = np.zeros(len(seqs) + 1, dtype=np.int64)
    np.cumsum([len(s) for s in seqs], out=offs[1:])
    res = np.concatenate(seqs) if seqs else np.zeros(0, dtype=np.uint8)
    return Database(res.astype(np.uint8), offs)


def encode(text: str) -> np.ndarray:
    return np.array([CODE[c] for c in text.upper()], dtype=np.uint8)


# --------------------------------------------------------------------------
# The five BASELINE.json configurations.
# --------------------------------------------------------------------------
CFG3_QUERY_LENGTHS = [int(round(144 + k * 5334 / 19)) for k in range(20)]


@dataclasses.dataclass
class Workload:
    name: str
    queries: list            # list of uint8 arrays
    db: Database
    matrix: np.ndarray = dataclasses.field(default_factory=lambda: BLOSUM62)
    gap_open: int = GAP_OPEN
    gap_extend: int = GAP_EXTEND
    planted: np.ndarray | None = None   # cfg4: indices of planted query copies
    notes: str = ""


def _scaled(count: int, scale: float) -> int:
    return max(1, int(round(count * scale)))


def config0(scale: float = 1.0) -> Workload:
    """configs[0]: query of 144 vs 10,000 sequences, lengths clip [8, 2000]."""
    lens = lognormal_lengths(rng_for(0, 0), _scaled(10_000, scale), 8, 2000)
    db = database_from_lengths(rng_for(0, 1), lens)
    q = rr_residues(rng_for(0, 2), 144)
    return Workload("cfg0", [q], db)


def config1(scale: float = 1.0) -> Workload:
    """configs[1]: query of 464 vs 1,000,000 sequences (~200 M residues)."""
    lens = lognormal_lengths(rng_for(1, 0), _scaled(1_000_000, scale), 8, 2000)
    db = database_from_lengths(rng_for(1, 1), lens)
    q = rr_residues(rng_for(1, 2), 464)
    return Workload("cfg1", [q], db)


def _cfg2_db(scale: float) -> Database:
    count = _scaled(6_500_000, scale)
    lens = lognormal_lengths(rng_for(2, 0), count, 8, 35_000)
    # Reading of "max 35,000": the log-normal reaches only
    # ~9.2 k naturally, so one sequence of exactly 35,000 is planted at a
    # seeded index to realise the stated maximum.
    pos = int(rng_for(2, 3).integers(0, count))
    lens[pos] = 35_000
    return database_from_lengths(rng_for(2, 1), lens)


def config2(scale: float = 1.0) -> Workload:
    """configs[2]: query of 1,000 vs 6.5 M sequences / ~1.3 G residues."""
    db = _cfg2_db(scale)
    q = rr_residues(rng_for(2, 2), 1000)
    return Workload("cfg2", [q], db)


def config3(scale: float = 1.0, lengths=None) -> Workload:
    """configs[3]: 20 queries, lengths 144..5478 evenly spaced, vs the cfg2 DB."""
    db = _cfg2_db(scale)
    rng = rng_for(3, 2)
    qs = [rr_residues(rng, L) for L in (lengths or CFG3_QUERY_LENGTHS)]
    return Workload("cfg3", qs, db)


def config4(scale: float = 1.0, w_fraction: float = 0.6) -> Workload:
    """configs[4]: query of 5,478 vs 200,000 sequences: 5% long (5,000-35,000),
    2% planted query copies with 5-20% substitutions (scores > 32,767).

    Reading: an RR query cannot score above 32,767
    against anything, because every BLOSUM62 score is bounded by the query's
    self-score (~28.7 k at 5,478 residues).  The query is therefore
    W-enriched: each position is W with probability ``w_fraction`` and an RR
    draw otherwise.  Planted copies substitute each position, with per-copy
    rate s ~ U[0.05, 0.20], by an RR residue different from the original; no
    indels.
    """
    m = 5478
    rq = rng_for(4, 2)
    q = rr_residues(rq, m)
    wmask = rq.random(m) < w_fraction
    q[wmask] = CODE["W"]
    n_total = _scaled(200_000, scale)
    n_long = _scaled(10_000, scale)
    n_plant = _scaled(4_000, scale)
    n_bulk = max(0, n_total - n_long - n_plant)
    r0 = rng_for(4, 0)
    bulk_lens = lognormal_lengths(r0, n_bulk, 8, 2000)
    long_lens = r0.integers(5_000, 35_001, size=n_long).astype(np.int64)
    r1 = rng_for(4, 1)
    seqs = [rr_residues(r1, int(L)) for L in np.concatenate([bulk_lens, long_lens])]
    r4 = rng_for(4, 4)
    planted = []
    for _ in range(n_plant):
        s = r4.uniform(0.05, 0.20)
        p = q.copy()
        sub = r4.random(m) < s
        k = int(sub.sum())
        # replacement residue: RR draw conditioned on != original (rejection)
        repl = rr_residues(r4, k)
        orig = p[sub]
        bad = repl == orig
        while bad.any():
            repl[bad] = rr_residues(r4, int(bad.sum()))
            bad = repl == orig
        p[sub] = repl
        planted.append(p)
    allseqs = seqs + planted
    perm = rng_for(4, 3).permutation(len(allseqs))
    db = database_from_list([allseqs[i] for i in perm])
    inv = np.empty_like(perm)
    inv[perm] = np.arange(len(perm))
    planted_idx = np.sort(inv[len(seqs):])
    return Workload("cfg4", [q], db, planted=planted_idx,
                    notes=f"W-enriched query (w_fraction={w_fraction})")


CONFIGS = {0: config0, 1: config1, 2: config2, 3: config3, 4: config4}


def make_config(k: int, scale: float = 1.0, **kw) -> Workload:
    return CONFIGS[int(k)](scale=scale, **kw)


# --------------------------------------------------------------------------
# Per-rank generation for the multi-GPU benchmark: the sequence lengths of a
# configuration (cheap), its queries, and the residues of any subset of its
# sequences, generated by streaming the configuration's residue RNG chunk by
# chunk so that a rank holds only its own shard.  The values are identical to
# make_config(k, scale).db / .queries (tests/test_inputs.py checks it).
# Configurations 0-3 only (cfg4 is built from a shuffled list).
# --------------------------------------------------------------------------
_RES_CHUNK = 1 << 26   # rr_residues' chunk: the subset stream must draw the same chunks


def config_lengths(k: int, scale: float = 1.0) -> np.ndarray:
    k = int(k)
    if k == 0:
        return lognormal_lengths(rng_for(0, 0), _scaled(10_000, scale), 8, 2000)
    if k == 1:
        return lognormal_lengths(rng_for(1, 0), _scaled(1_000_000, scale), 8, 2000)
    if k in (2, 3):
        count = _scaled(6_500_000, scale)
        lens = lognormal_lengths(rng_for(2, 0), count, 8, 35_000)
        lens[int(rng_for(2, 3).integers(0, count))] = 35_000   # as _cfg2_db
        return lens
    raise ValueError("config_lengths: configurations 0-3 only")


def config_queries(k: int) -> list:
    k = int(k)
    if k == 0:
        return [rr_residues(rng_for(0, 2), 144)]
    if k == 1:
        return [rr_residues(rng_for(1, 2), 464)]
    if k == 2:
        return [rr_residues(rng_for(2, 2), 1000)]
    if k == 3:
        rng = rng_for(3, 2)
        return [rr_residues(rng, L) for L in CFG3_QUERY_LENGTHS]
    raise ValueError("config_queries: configurations 0-3 only")


def config_db_subset(k: int, idx, scale: float = 1.0) -> Database:
    """Sub-database of configuration k's sequences idx (strictly ascending),
    equal to make_config(k, scale).db.subset(idx), generated without holding
    the whole database."""
    k = int(k)
    lens = config_lengths(k, scale)
    idx = np.asarray(idx, dtype=np.int64)
    if idx.size and (np.any(np.diff(idx) <= 0) or idx[0] < 0 or idx[-1] >= lens.size):
        raise ValueError("idx must be strictly ascending sequence indices")
    if idx.size == lens.size:   # the whole database
        return database_from_lengths(rng_for(2 if k == 3 else k, 1), lens)
    offs = np.zeros(lens.size + 1, dtype=np.int64)
    np.cumsum(lens, out=offs[1:])
    starts, ends = offs[idx], offs[idx + 1]
    L = ends - starts
    noffs = np.zeros(idx.size + 1, dtype=np.int64)
    np.cumsum(L, out=noffs[1:])
    out = np.empty(int(noffs[-1]), dtype=np.uint8)
    rng = rng_for(2 if k == 3 else k, 1)
    n = int(offs[-1])
    for s in range(0, n, _RES_CHUNK):
        e = min(n, s + _RES_CHUNK)
        codes = _RR_LUT[rng.integers(0, 1 << _LUT_BITS, size=e - s, dtype=np.uint16)]
        lo = int(np.searchsorted(ends, s, side="right"))
        hi = int(np.searchsorted(starts, e, side="left"))
        if hi <= lo:
            continue
        seg_s = np.maximum(starts[lo:hi], s)
        seg_len = np.minimum(ends[lo:hi], e) - seg_s
        dst0 = noffs[lo:hi] + (seg_s - starts[lo:hi])
        cum = np.zeros(seg_len.size + 1, dtype=np.int64)
        np.cumsum(seg_len, out=cum[1:])
        rel = np.arange(int(cum[-1]), dtype=np.int64) - np.repeat(cum[:-1], seg_len)
        out[np.repeat(dst0, seg_len) + rel] = codes[np.repeat(seg_s - s, seg_len) + rel]
    return Database(out, noffs)


# --------------------------------------------------------------------------
# Random small cases for property tests (random symmetric
# matrices in [-4, 11], gaps in [0, 15]).
# --------------------------------------------------------------------------
def random_symmetric_matrix(rng: np.random.Generator, lo: int = -4, hi: int = 11) -> np.ndarray:
    a = rng.integers(lo, hi + 1, size=(ALPHA, ALPHA))
    a = np.triu(a) + np.triu(a, 1).T
    return a.astype(np.int8)


def random_sequence(rng: np.random.Generator, n: int, letters: int = 20) -> np.ndarray:
    return rng.integers(0, letters, size=int(n)).astype(np.uint8)
