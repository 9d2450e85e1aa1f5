"""The C oracle under AddressSanitizer + UndefinedBehaviorSanitizer (SURVEY.md 5:
"build the oracle with ASan/UBSan").  oracle/sw_oracle.c is compiled, unmodified,
with a small driver into an instrumented executable that runs oracle_sw_score,
oracle_sw_full and oracle_sw_batch (threads, an index list, empty sequences, a
one-residue sequence, large penalties) on seeded inputs read from a file.  The
run must be clean (no sanitizer report) and print what the ordinary -O2 build
returns; two of the printed values are also the paper-derived closed forms of
tests/test_oracle_pins.py (W^300 self-score 3300; "AW"/"AW" 15,
SPEC.md:124), so the instrumented build is pinned, not only self-consistent.
"""
import os
import shutil
import subprocess

import numpy as np
import pytest

import oracle
import sw_inputs as si
from sw_inputs import BLOSUM62, encode

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(os.path.dirname(HERE), "oracle", "sw_oracle.c")

DRIVER = r"""
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
int64_t oracle_sw_score(const uint8_t *, int64_t, const uint8_t *, int64_t, const int8_t *, int64_t, int64_t);
int64_t oracle_sw_full(const uint8_t *, int64_t, const uint8_t *, int64_t, const int8_t *, int64_t, int64_t,
                       int64_t *, int64_t *, int64_t *);
int oracle_sw_batch(const uint8_t *, int64_t, const uint8_t *, const int64_t *, const int64_t *, int64_t,
                    const int8_t *, int64_t, int64_t, int64_t *, int);
/* file: int64 m, count, total, nidx, open, ext; q[m]; offs[count+1]; res[total]; idx[nidx]; SM[576] */
int main(int argc, char **argv) {
  if (argc < 2) return 2;
  FILE *f = fopen(argv[1], "rb");
  if (!f) return 2;
  int64_t h[6];
  if (fread(h, 8, 6, f) != 6) return 2;
  const int64_t m = h[0], count = h[1], total = h[2], nidx = h[3], go = h[4], ge = h[5];
  uint8_t *q = malloc((size_t)m + 1), *res = malloc((size_t)total + 1);
  int64_t *offs = malloc(8 * (size_t)(count + 1)), *idx = malloc(8 * (size_t)(nidx + 1));
  int8_t SM[576];
  if (fread(q, 1, (size_t)m, f) != (size_t)m) return 2;
  if (fread(offs, 8, (size_t)count + 1, f) != (size_t)count + 1) return 2;
  if (fread(res, 1, (size_t)total, f) != (size_t)total) return 2;
  if (fread(idx, 8, (size_t)nidx, f) != (size_t)nidx) return 2;
  if (fread(SM, 1, 576, f) != 576) return 2;
  fclose(f);
  int64_t *sc = malloc(8 * (size_t)(count + 1));
  if (oracle_sw_batch(q, m, res, offs, NULL, count, SM, go, ge, sc, 4)) return 3;
  for (int64_t i = 0; i < count; ++i) printf("b %lld\n", (long long)sc[i]);
  if (oracle_sw_batch(q, m, res, offs, idx, nidx, SM, go, ge, sc, 3)) return 3;
  for (int64_t i = 0; i < nidx; ++i) printf("i %lld\n", (long long)sc[i]);
  for (int64_t i = 0; i < count; ++i)
    printf("s %lld\n", (long long)oracle_sw_score(q, m, res + offs[i], offs[i + 1] - offs[i], SM, go, ge));
  for (int64_t i = 0; i < count && i < 6; ++i) {   /* full matrices of the first sequences */
    const int64_t n = offs[i + 1] - offs[i];
    if (n > 64 || m > 400) continue;
    const size_t cells = (size_t)(m + 1) * (size_t)(n + 1);
    int64_t *H = malloc(8 * cells), *E = malloc(8 * cells), *F = malloc(8 * cells);
    const int64_t best = oracle_sw_full(q, m, res + offs[i], n, SM, go, ge, H, E, F);
    int64_t sum = 0;
    for (size_t c = 0; c < cells; ++c) sum += H[c] * 3 + E[c] * 5 + F[c] * 7;
    printf("f %lld %lld\n", (long long)best, (long long)sum);
    free(H); free(E); free(F);
  }
  free(q); free(res); free(offs); free(idx); free(sc);
  return 0;
}
"""


@pytest.fixture(scope="module")
def sanitized(tmp_path_factory):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    d = tmp_path_factory.mktemp("oracle_san")
    drv = d / "driver.c"
    drv.write_text(DRIVER)
    exe = d / "oracle_san"
    cmd = ["gcc", "-O1", "-g", "-std=c11", "-pthread", "-fsanitize=address,undefined", "-fno-sanitize-recover=all",
           "-fno-omit-frame-pointer", "-o", str(exe), str(drv), SRC]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0 and "sanitize" in r.stderr and "cannot find" in r.stderr:
        pytest.skip("sanitizer runtimes not installed")
    assert r.returncode == 0, r.stderr
    return exe, d


def _run(sanitized, name, q, seqs, idx, gap_open, gap_extend, M=BLOSUM62):
    exe, d = sanitized
    q = np.asarray(q, dtype=np.uint8)
    lens = np.array([len(s) for s in seqs], dtype=np.int64)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    res = np.concatenate([np.asarray(s, dtype=np.uint8) for s in seqs] + [np.zeros(0, np.uint8)])
    idx = np.asarray(idx, dtype=np.int64)
    blob = d / f"{name}.bin"
    with open(blob, "wb") as f:
        f.write(np.array([len(q), len(seqs), len(res), len(idx), gap_open, gap_extend], dtype=np.int64).tobytes())
        f.write(q.tobytes()); f.write(offs.tobytes()); f.write(res.tobytes()); f.write(idx.tobytes())
        f.write(np.ascontiguousarray(M, dtype=np.int8).tobytes())
    env = dict(os.environ, ASAN_OPTIONS="detect_leaks=1:abort_on_error=0", UBSAN_OPTIONS="print_stacktrace=1")
    r = subprocess.run([str(exe), str(blob)], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0, (r.returncode, r.stderr[-2000:])
    assert "runtime error" not in r.stderr and "Sanitizer" not in r.stderr, r.stderr[-2000:]
    out = {"b": [], "i": [], "s": [], "f": []}
    for ln in r.stdout.split("\n"):
        if ln:
            k, *v = ln.split()
            out[k].append(tuple(int(x) for x in v) if len(v) > 1 else int(v[0]))
    # the ordinary build returns the same
    exp = oracle.batch(q, res, offs, M, gap_open, gap_extend)
    assert out["b"] == [int(x) for x in exp]
    assert out["s"] == [int(x) for x in exp]
    assert out["i"] == [int(exp[j]) for j in idx]
    k = 0
    for i, s in enumerate(seqs[:6]):
        if len(s) > 64 or len(q) > 400:
            continue
        H, E, F, best = oracle.full(q, s, M, gap_open, gap_extend)
        assert out["f"][k] == (best, int((H * 3 + E * 5 + F * 7).sum())), i
        k += 1
    return out


def test_sanitized_oracle_on_pins_and_edge_cases(sanitized):
    rng = np.random.default_rng(1702)
    seqs = [encode("W" * 300), encode("AW"), encode("A"), np.zeros(0, np.uint8), encode("V"),
            si.rr_residues(rng, 1), si.rr_residues(rng, 63), si.rr_residues(rng, 700)]
    out = _run(sanitized, "pins_w", encode("W" * 300), seqs, [7, 0, 3, 3, 1], 10, 2)
    assert out["b"][0] == 3300                 # SPEC.md:324 (W:W = 11, 300 residues)
    assert out["b"][3] == 0                    # empty database sequence (reading R4)
    out = _run(sanitized, "pins_aw", encode("AW"), seqs, [1, 2, 4], 10, 2)
    assert out["b"][1] == 15 and out["b"][2] == 4 and out["b"][4] == 0


def test_sanitized_oracle_random_matrices_and_gaps(sanitized):
    rng = np.random.default_rng(7195)
    for trial in range(6):
        M = rng.integers(-8, 12, (24, 24)).astype(np.int8)
        if trial % 2 == 0:
            M = np.maximum(M, M.T)             # symmetric and asymmetric matrices
        seqs = [rng.integers(0, 24, int(n)).astype(np.uint8) for n in rng.integers(0, 90, 40)]
        q = rng.integers(0, 24, int(rng.integers(1, 120))).astype(np.uint8)
        go, ge = [(0, 0), (10, 2), (0, 5), (40000, 1), (3, 0), (2 ** 29, 2 ** 29)][trial]
        _run(sanitized, f"rand{trial}", q, seqs, rng.integers(0, 40, 17), go, ge, M)
