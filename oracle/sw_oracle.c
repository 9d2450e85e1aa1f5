/*
 * oracle/sw_oracle.c -- plain, slow, obviously correct CPU oracle for
 * Smith-Waterman local alignment with affine (Gotoh) gaps.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this code.  It
 * shares no code, header, table or constant with the CUDA path
 * (paper_1702_07195_b200/csrc/), and never includes anything from it.
 *
 * What it computes (Section 2, Eqs. 1-3):
 *
 *   E_{i,j} = max{ H_{i,j-1} - Goe, E_{i,j-1} - Ge }                (Eq. 2)
 *   F_{i,j} = max{ H_{i-1,j} - Goe, F_{i-1,j} - Ge }                (Eq. 3)
 *   H_{i,j} = max{ 0, H_{i-1,j-1} + SM(S1[i], S2[j]), E_{i,j}, F_{i,j} }  (Eq. 1)
 *
 *   "The recurrences should be calculated with 1 <= i <= m and 1 <= j <= n,
 *   after initializing H, E and F with 0 when i = 0 or j = 0.  The maximum
 *   value in the alignment matrix H is the optimal local alignment score."
 *   (PAPER.md:66).  Goe = gap open + gap extend, Ge = gap extend.
 *
 * Readings:
 *   R1  S1 = query (rows i), S2 = database sequence (columns j), SM indexed
 *       SM[q*24 + d].
 *   R2  E and F are computed exactly as written: no floor at 0,
 *       boundary values 0 as written (C2).
 *   R3  The score is the max over the whole H matrix including its zero row
 *       and column, so it is >= 0 and an empty sequence scores 0 (C5).
 *   All arithmetic in int64: no overflow is possible for |SM| <= 127 and
 *   lengths < 2^31 with penalties < 2^31.
 *
 * Parity pins: tests/test_oracle_pins.py (brute-force enumeration, LCS and
 * Kadane reductions, hand-worked closed forms in tests/golden/, invariants).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define ORACLE_ALPHA 24

static inline int64_t max2(int64_t a, int64_t b) { return a > b ? a : b; }

/* Two-row form of Eqs. 1-3.  work must hold 2*(n+1) int64.
 * Hp[j] holds H_{i-1,j} (then H_{i,j} once column j of row i is done),
 * Fp[j] holds F_{i-1,j} (then F_{i,j}). */
static int64_t score_two_row(const uint8_t *q, int64_t m, const uint8_t *d, int64_t n,
                             const int8_t *SM, int64_t Goe, int64_t Ge, int64_t *work) {
  int64_t *Hp = work, *Fp = work + (n + 1);
  for (int64_t j = 0; j <= n; ++j) { Hp[j] = 0; Fp[j] = 0; }   /* i = 0: H = F = 0 */
  int64_t best = 0;                                             /* H_{0,*} = 0 */
  for (int64_t i = 1; i <= m; ++i) {
    int64_t Hdiag = Hp[0];  /* H_{i-1,0} = 0 */
    int64_t Hleft = 0;      /* H_{i,0} = 0 */
    int64_t Eleft = 0;      /* E_{i,0} = 0 */
    const int8_t *row = SM + (size_t)q[i - 1] * ORACLE_ALPHA;
    for (int64_t j = 1; j <= n; ++j) {
      int64_t E = max2(Hleft - Goe, Eleft - Ge);                        /* Eq. 2 */
      int64_t F = max2(Hp[j] - Goe, Fp[j] - Ge);                        /* Eq. 3 */
      int64_t H = max2(max2(0, Hdiag + (int64_t)row[d[j - 1]]), max2(E, F)); /* Eq. 1 */
      Hdiag = Hp[j];
      Hp[j] = H;
      Fp[j] = F;
      Hleft = H;
      Eleft = E;
      if (H > best) best = H;
    }
  }
  return best;
}

/* Score of one pair.  Returns -1 on allocation failure. */
int64_t oracle_sw_score(const uint8_t *q, int64_t m, const uint8_t *d, int64_t n,
                        const int8_t *SM, int64_t gap_open, int64_t gap_extend) {
  int64_t *work = (int64_t *)malloc(sizeof(int64_t) * 2 * (size_t)(n + 1));
  if (!work) return -1;
  int64_t s = score_two_row(q, m, d, n, SM, gap_open + gap_extend, gap_extend, work);
  free(work);
  return s;
}

/* Full (m+1) x (n+1) matrices H, E, F (row-major), literal Eqs. 1-3 with the
 * zero boundary of PAPER.md:66.  For tiny inputs (test utility). */
int64_t oracle_sw_full(const uint8_t *q, int64_t m, const uint8_t *d, int64_t n,
                       const int8_t *SM, int64_t gap_open, int64_t gap_extend,
                       int64_t *H, int64_t *E, int64_t *F) {
  const int64_t Goe = gap_open + gap_extend, Ge = gap_extend, W = n + 1;
  for (int64_t i = 0; i <= m; ++i)
    for (int64_t j = 0; j <= n; ++j) { H[i * W + j] = 0; E[i * W + j] = 0; F[i * W + j] = 0; }
  int64_t best = 0;
  for (int64_t i = 1; i <= m; ++i)
    for (int64_t j = 1; j <= n; ++j) {
      E[i * W + j] = max2(H[i * W + j - 1] - Goe, E[i * W + j - 1] - Ge);
      F[i * W + j] = max2(H[(i - 1) * W + j] - Goe, F[(i - 1) * W + j] - Ge);
      int64_t h = H[(i - 1) * W + j - 1] + (int64_t)SM[(size_t)q[i - 1] * ORACLE_ALPHA + d[j - 1]];
      h = max2(max2(0, h), max2(E[i * W + j], F[i * W + j]));
      H[i * W + j] = h;
      if (h > best) best = h;
    }
  return best;
}

/* ---- batch: one database sequence per task on a pthread pool ---------- */
typedef struct {
  const uint8_t *q; int64_t m;
  const uint8_t *res; const int64_t *offs; const int64_t *idx; int64_t count;
  const int8_t *SM; int64_t Goe, Ge;
  int64_t *scores;
  int64_t next;          /* atomic task cursor */
  int64_t max_len;
  int failed;
} batch_t;

static void *batch_worker(void *arg) {
  batch_t *b = (batch_t *)arg;
  int64_t *work = (int64_t *)malloc(sizeof(int64_t) * 2 * (size_t)(b->max_len + 1));
  if (!work) { __atomic_store_n(&b->failed, 1, __ATOMIC_RELAXED); return NULL; }
  for (;;) {
    int64_t t = __atomic_fetch_add(&b->next, 1, __ATOMIC_RELAXED);
    if (t >= b->count) break;
    int64_t s = b->idx ? b->idx[t] : t;
    int64_t beg = b->offs[s], n = b->offs[s + 1] - beg;
    b->scores[t] = score_two_row(b->q, b->m, b->res + beg, n, b->SM, b->Goe, b->Ge, work);
  }
  free(work);
  return NULL;
}

/* Scores of the query against sequences idx[0..count) of a database given as
 * residues + offsets (sequence s = res[offs[s] .. offs[s+1])).  idx == NULL
 * means sequences 0..count-1.  scores[t] is the score of sequence idx[t].
 * Returns 0, or -1 on allocation / thread failure. */
int oracle_sw_batch(const uint8_t *q, int64_t m, const uint8_t *res, const int64_t *offs,
                    const int64_t *idx, int64_t count, const int8_t *SM, int64_t gap_open,
                    int64_t gap_extend, int64_t *scores, int nthreads) {
  batch_t b;
  memset(&b, 0, sizeof b);
  b.q = q; b.m = m; b.res = res; b.offs = offs; b.idx = idx; b.count = count; b.SM = SM;
  b.Goe = gap_open + gap_extend; b.Ge = gap_extend; b.scores = scores;
  for (int64_t t = 0; t < count; ++t) {
    int64_t s = idx ? idx[t] : t;
    int64_t n = offs[s + 1] - offs[s];
    if (n > b.max_len) b.max_len = n;
  }
  if (nthreads < 1) nthreads = 1;
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
  if (!th) return -1;
  int started = 0;
  for (int k = 0; k < nthreads; ++k) {
    if (pthread_create(&th[k], NULL, batch_worker, &b) != 0) break;
    ++started;
  }
  if (started == 0) batch_worker(&b);
  for (int k = 0; k < started; ++k) pthread_join(th[k], NULL);
  free(th);
  return b.failed ? -1 : 0;
}
