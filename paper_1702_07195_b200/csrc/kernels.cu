// sm_100a kernels of the inter-task Smith-Waterman database search.
//
// The recurrence (Eqs. 1-3), per cell (i = query row, j =
// database column), in the equivalent relu form (readings R2, R3):
//   H_ij = max{0, H_{i-1,j-1} + SM(q_i, d_j), E_ij, F_ij}
//   E_{i,j+1} = max{E_ij - Ge, max(H_ij - Goe, 0)}
//   F_{i+1,j} = max{F_ij - Ge, max(H_ij - Goe, 0)}
//   S = max over all H_ij
// is evaluated on packed s16x2 registers: each 32-bit value holds the same
// cell of two different database sequences ("halves" A and B, inter-task
// parallelism), or of two queries (query pairs).  Default
// arithmetic (SW_ARITH=1, kernels.cuh): every value is stored
// + 16384 per half, so H_diag + SM is one 32-bit IMAD on the FMA pipe and
// Eq. 1 one VIMNMX3 -- 4.5 Blackwell DPX instructions (VIMNMX3.S16x2 +
// 3 VIADDMNMX.S16x2 + 1/2 VIMNMX3 for S) and 2 IMADs per pair of cells.  DPX
// adds wrap instead of saturating (R7): a sequence whose stored
// 16-bit score reaches 32768 - smax is flagged and re-scored exactly by the
// s32 kernel ("recalculated using the next wider integer range"),
// starting from the last exact 16-bit pass boundary; later
// 16-bit passes start each work item behind its leading run of flagged
// sequences (item_skip_kernel).
//
// Mapping: a *group* of G lanes (G in 8/16/32) is a systolic
// array over the query: lane t owns R consecutive query rows of the current
// pass, keeps H and E of its rows in registers, and passes the bottom-row
// (H, F), the column's descriptor words and the running score chain to lane
// t+1 with one SHFL each per column.  A group streams one work item (two lane
// streams of whole sequences separated by END/NUL columns) at a time, claimed
// longest-first from an atomic counter (PAPER.md:119 dynamic distribution).
// The substitution scores come from a query profile in shared
// memory, one score per (letter, row) 32-bit word, read with conflict-free
// LDS.128 (4 rows per load).
#include "kernels.cuh"

#include <algorithm>
#include <type_traits>
#include <climits>
#include <cstdio>

// SW_ROWAHEAD: 1 = biased rows form the next row's diagonal add before the
// current row's H is overwritten (see the pass kernel); 0 = plain row order.
#ifndef SW_BRING
#define SW_BRING 0   // 1: boundary prefetch ring in every boundary-reading kernel (experiment)
#endif
#ifndef SW_ROWAHEAD
#define SW_ROWAHEAD -1   // -1: per kernel instantiation (kRowPlain); 0 / 1 force every one
#endif
#ifndef SW_ROWS_TRACE
#define SW_ROWS_TRACE 0   // 1: the rows kernel prints per-pass cycle counts of item 0 (experiments)
#endif
#ifndef SW_EARLY
#define SW_EARLY 1   // latency tiles load each column's descriptor and profile one step ahead
#endif
#ifndef SW_LATROWS
#define SW_LATROWS 1   // EARLY tiles: Eq. 3 with a one-instruction vertical chain (Goe >= Ge)
#endif
#ifndef SW_SHFLORD
#define SW_SHFLORD 0   // 1: shuffle the chain values before the descriptor words (experiment)
#endif
#ifndef SW_SCEND
#define SW_SCEND 0   // 1: lane G-1 stores the score chain at separator columns only (experiment)
#endif
#ifndef SW_DESCADDR
// lane G-1's descriptor address from its own s_qp (1) or from the shared base s_desc (0),
// per kernel instantiation from a calibration (-1, kernels.cu desc_from_qp); 0 / 1 force
// every instantiation (the calibration builds)
#define SW_DESCADDR -1
#endif
#ifndef SW_TAILADDR
#define SW_TAILADDR 0   // narrow-tail address: 0 = IMAD from the profile offset, 1 = from the chunk address
#endif
// SW_ABLATE (performance experiments only, wrong results): see the pass kernel.
#ifndef SW_ABLATE
#define SW_ABLATE 0
#endif
// SW_DEBUG: device-side bounds checks on every global / shared access of the
// pass kernel (a debug build; compute-sanitizer is not available on the GPU
// pool).  A violation traps with a device assert.
#ifndef SW_DEBUG
#define SW_DEBUG 0
#endif
#if SW_DEBUG
#include <cassert>
#define SW_CHECK(cond) assert(cond)
#else
#define SW_CHECK(cond) ((void)0)
#endif

namespace swdb {

namespace {

constexpr int kThreads = 512;
constexpr int kWavePublish = 64;   // wavefront: columns between progress publications
constexpr uint32_t kB2 = (uint32_t)kBias16 * 0x10001u;   // the stored zero, both halves
constexpr uint32_t kNulWord = (uint32_t)((kNul * kNL + kNul) * kDescBytes);

// 16x2 max operations of the cell: unsigned halves in the biased-unsigned
// form (SW_ARITH 2), signed otherwise (kernels.cuh).
__device__ __forceinline__ uint32_t hmax3(uint32_t a, uint32_t b, uint32_t c) {
  return kArith == 2 ? __vimax3_u16x2(a, b, c) : __vimax3_s16x2(a, b, c);
}
__device__ __forceinline__ uint32_t haddmax(uint32_t a, uint32_t b, uint32_t c) {   // max(a + b, c)
  return kArith == 2 ? __viaddmax_u16x2(a, b, c) : __viaddmax_s16x2(a, b, c);
}
__device__ __forceinline__ uint32_t hmax(uint32_t a, uint32_t b) {
  return kArith == 2 ? __vmaxu2(a, b) : __vmaxs2(a, b);
}

__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// ---------------------------------------------------------------------------
// s16x2 pass kernel: query rows [pass*G*R, (pass+1)*G*R) against every item.
//
// Shared memory: descriptor table [kNL*kNL] x 16 B, then the profile slice of
// this pass, int16, laid out [letter][8-row chunk][lane t][8 x int16] so that
// the 8 lanes of a quarter-warp always hit 8 distinct 16-B bank groups.
// Descriptor of letter pair (cA, cB): {offA | offB << 16 (profile offsets
// in 16-B units), notsep bits (1 per non-separator half), END bits (0x8000 in
// a half whose sequence ENDs; informational), 0}.  Only lane 0 of a group reads it; lanes
// t > 0 receive it from lane t-1 with the column.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t umulhi(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ uint2 lds64(uint32_t addr) {
  uint2 v;
  asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}

// 1-D bulk copy global -> shared (TMA engine, cp.async.bulk) completing on an
// mbarrier: one thread arms the barrier with the byte count and issues the
// copies; every thread waits on the barrier's phase.
__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(mbar), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arm(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(mbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(dst), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t phase) {
  asm volatile("{\n\t.reg .pred P;\n"
               "WAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
               "\t@!P bra WAIT_%=;\n}" :: "r"(mbar), "r"(phase) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t mbar) {   // release.cta: prior writes are visible to waiters
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(mbar) : "memory");
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

// L2-coherent loads (the cross-pass wavefront reads data other SMs write
// during the launch; __ldg / L1-cached loads could return stale lines).
__device__ __forceinline__ uint2 ld_cg_v2(const uint2 *p) {
  uint2 v;
  asm volatile("ld.global.cg.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ld_cg(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int *p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" :: "r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

__device__ __forceinline__ void st_global_v2(uint2 *p, uint32_t a, uint32_t b) {
  asm volatile("st.global.v2.u32 [%0], {%1, %2};" :: "l"(p), "r"(a), "r"(b) : "memory");
}

__device__ __forceinline__ void st_global_v4(uint4 *p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" :: "l"(p), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

__device__ __forceinline__ void st_global_v2(uint2 *p, uint32_t a, uint32_t b);

__device__ __forceinline__ void st_global_u32(uint32_t *p, uint32_t a) {
  asm volatile("st.global.u32 [%0], %1;" :: "l"(p), "r"(a) : "memory");
}

// Descriptor of a letter pair -> the column-chain words (see qp_build_kernel).
struct DescWords { uint32_t w0, ngoe, nge, kneg; };
__device__ __forceinline__ DescWords load_desc(uint32_t addr) {
  const uint4 d = lds128(addr);
  return DescWords{d.x, d.y, d.z, d.w};
}

template <class T>
__device__ __forceinline__ T *ptr_add(T *p, uint32_t n) {  // p + n elements, on the FMA pipe
  uint64_t d;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(n), "r"((uint32_t)sizeof(T)), "l"((uint64_t)p));
  return reinterpret_cast<T *>(d);
}

// Profile modes (what the two 16-bit halves of a register hold):
//   QPM 0: two database sequences, one query.  Profile: one score per
//          (letter,row) 32-bit word (sign-extended; zero-extended in the relu
//          form), 4 rows per 16-B chunk; the two halves' scores are packed into
//          SM_B * 65536 + SM_A with one IMAD(B, 65536, A) (FMA pipe).
//          (int16-pair profiles were measured slower: DESIGN.md 3 and 4.2.)
//   QPM 3: one database sequence, two queries (multi-query packing, SURVEY
//          8(f) NEXT-2).  Profile word = SM(q2_r, c) * 65536 + SM(q1_r, c)
//          (relu form: the two halves): no packing at all; the stream holds one
//          sequence per column (column word of the letter pair (c, c)).
//
// Lane roles inside a group (shuffles rotate: lane 0 receives from lane G-1):
//   lane G-1 after computing its column: stores the column's score chain value
//   (and the pass boundary), loads the descriptor of lane 0's next column from
//   smem (its stream word was prefetched U columns ahead) and overwrites its
//   outgoing registers with lane 0's next-column inputs, including the
//   previous pass's boundary (prefetched U columns ahead).  No per-lane
//   selects at lane 0.
template <int R, int G, bool BIN, int QPM, int NT, int U, bool WAVE = false, bool DA = false, bool RA = true>
__global__ void __launch_bounds__(NT, 1) sw16_pass_kernel(const SW16Params p) {
  static_assert(!WAVE || BIN, "the wavefront kernel reads boundaries (from pass 1 on)");
  static_assert(U == 1 || U == 2 || U == 4, "U: columns per unrolled block / prefetch distance");
  static_assert(!(SW_EARLY && NT == 256) || U % 2 == 0, "EARLY alternates two profile sets per column");
  static_assert(QPM == 0 || QPM == 1 || QPM == 3, "profile mode");
  static_assert(QPM != 1 || kBiased, "the score profile is built for the biased arithmetic");
  constexpr int RPC = 4;                    // rows per 16-B profile chunk
  constexpr int KC = (R + RPC - 1) / RPC;   // chunks per lane (the last may be a narrow tail)
  constexpr int KCF = qp_full_chunks(R);    // chunks read with LDS.128 (kernels.cuh layout)
  constexpr int TW = qp_tail_w(R) == 16 ? 0 : qp_tail_w(R);   // narrow tail: 4 or 8 B per lane
  constexpr int LS = qp_letter_bytes(G, R); // bytes per letter in the profile slice
  constexpr int QP_U4 = QPM == 1 ? kSPBytes / 16 : kNL * LS / 16;   // profile words in shared memory
  static_assert(LS % 128 == 0, "letter slices are 128-B aligned");
  constexpr int DESC_U4 = kNL * kNL;
  // Lane G-1 prefetches the previous pass's boundary U columns ahead through a
  // register ring only in the wavefront kernel; the per-pass boundary-reading
  // kernel loads it at the start of the column (the rows hide the latency):
  // the ring's 8 registers push that variant past the register cap (spills,
  // register shuffles at the loop back-edge).
  constexpr bool BRING = WAVE || SW_BRING;
  extern __shared__ uint4 smem[];
  __shared__ uint64_t s_mbar;
  __shared__ int s_solo[4];   // EARLY solo items: per SM sub-partition, warp q's first claim (-1: not yet, 1: solo)
  {
    // the descriptor table and this pass's profile slice arrive by two 1-D
    // bulk copies (TMA) on one mbarrier
    const uint32_t mbar = (uint32_t)__cvta_generic_to_shared(&s_mbar);
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
    if (threadIdx.x == 0) {
      mbar_init(mbar, 1);
      mbar_arm(mbar, (DESC_U4 + QP_U4) * 16);
      bulk_g2s(sbase, p.desc, DESC_U4 * 16, mbar);
      // QPM 1: the score profile does not depend on the pass
      bulk_g2s(sbase + DESC_U4 * 16, p.qp + (QPM == 1 ? (size_t)0 : (size_t)p.pass * QP_U4), QP_U4 * 16, mbar);
    }
    if (threadIdx.x < 4) s_solo[threadIdx.x] = -1;
    __syncthreads();   // the barrier is initialised before anyone waits on it
    mbar_wait(mbar, 0);
  }

  const int lane = threadIdx.x & 31;
  const int t = lane & (G - 1);
  const int gbase = lane & ~(G - 1);
  const int src = gbase + ((t + G - 1) & (G - 1));   // lane t-1; lane 0 <- lane G-1
  const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << gbase);
  const bool last = t == G - 1;
  const uint32_t nlast = last ? 0u : 1u;
  const uint32_t bdef = last ? kB2 : 0u;   // lane 0's boundary without a previous pass (via lane G-1)
  const uint32_t zero = p.zero;
  const uint32_t s_desc = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t s_qp = s_desc + DESC_U4 * 16 + t * 16;
  // narrow tail block: lane t of group g reads copy g % ncopy at lane stride TW
  const uint32_t s_qpt = s_desc + DESC_U4 * 16 + KCF * G * 16 +
                         (uint32_t)(((lane / G) % qp_tail_ncopy(G, R)) * G + t) * (uint32_t)(TW ? TW : 16);
  const uint32_t s_dqt = s_qpt - s_qp;
  // QPM 1 (score profile): the byte address in SP of each of the lane's query
  // rows' letter (24 = phantom row); the column's pair offset is added per row
  uint32_t qoff[QPM == 1 ? R : 1];
  if (QPM == 1) {
    const uint32_t s_sp = s_desc + DESC_U4 * 16;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = p.pass * G * R + t * R + r;
      qoff[r] = s_sp + 4u * (row < p.m ? (uint32_t)__ldg(p.query + row) : (uint32_t)kAlpha);
    }
  }
  __syncthreads();
  const DescWords nul = load_desc(s_desc + kNulWord);

  const uint32_t one = p.one;
  uint32_t H[R], E[R];
#pragma unroll
  for (int r = 0; r < R; ++r) { H[r] = kB2; E[r] = kB2; }
  uint32_t S = 0u, hout = kB2, fout = kB2, sc = 0u, hprev = kB2;
  uint32_t w0 = nul.w0;                          // column chain (NUL): profile offsets
  uint32_t kneg = 0u;                            // S-reset value after the previous column
  uint32_t ngoe = nul.ngoe, nge = nul.nge, knext = nul.kneg;   // descriptor penalty words of the column chain

  // Lane G-1 prefetches the stream and the previous pass's boundary 4 columns
  // ahead, and stores per column the score chain value (sc_out) and the
  // boundary for the next pass.  A group without items keeps feeding NUL
  // columns; its pointers stop (increment 0) on the NUL padding / own slot.
  uint2 *const dummy = p.dummy + (blockIdx.x * blockDim.x + threadIdx.x);
  const uint32_t *sptr = p.nul_stream;
  const uint2 *bptr = p.zero_bnd;
  // SW_SCEND (not in the wavefront): every lane stores the chain at separator
  // columns, lanes t < G-1 into their own dummy slot (no lane predicate)
  constexpr bool SCEND = SW_SCEND && !WAVE;
  uint32_t *scp = reinterpret_cast<uint32_t *>(dummy);
  uint32_t scinc = 0u;
  uint2 *bop = dummy;
  uint32_t inc = 0u;
  int rem = 0;                                   // steps left in the current item
  int bcols = 0;  // BIN: boundary columns left to read (columns >= ncols read as 0: the
                  // boundary buffer's padding may hold another image's or search's data)
  bool done = false;
  uint32_t sring[U];
  uint2 bring[U];
  uint32_t scring[WAVE ? U : 1];   // WAVE: the previous pass's score chain, per column
#pragma unroll
  for (int u = 0; u < U; ++u) { sring[u] = 0u; bring[u] = make_uint2(kB2, kB2); }
#pragma unroll
  for (int u = 0; u < (WAVE ? U : 1); ++u) scring[u] = 0u;
  const uint32_t *scin = nullptr;  // WAVE: sc_out of the item's columns (previous pass)
  int cur_it = 0, cur_ncols = 0, sdone = 0, avail = 0;   // WAVE progress bookkeeping
  // EARLY (latency tiles): a group's step is a latency chain
  // when one long item bounds the pass.  Each lane receives its NEXT column's
  // profile offsets one step early and loads that column's profile chunks
  // during the current column's rows; lane G-1 loads lane 0's descriptors one
  // column ahead.  The per-step chain is then shuffle -> rows -> shuffle,
  // without the descriptor load, the second shuffle and the profile load.
  constexpr bool EARLY = SW_EARLY && NT == 256 && QPM == 0 && !WAVE;
  // LROWS (EARLY tiles): with the loads off the step's chain, the chain is the
  // vertical F recurrence through the lane's R rows (3 dependent DPX per row).
  // Eq. 3 as F' = max(F - Ge, max(max(t, E) - Goe, 0)) -- equal to
  // max(F - Ge, max(H - Goe, 0)) since Goe >= Ge (H - Goe's F term is below
  // F - Ge) -- is one VIADDMNMX per row on the chain, for 1.5 more ALU
  // instructions per pair of cells off it (profiles/r02_lat_calibration_early.jsonl).
  constexpr bool LROWS = EARLY && SW_LATROWS && R >= 5;   // measured slower at R = 3, 4
  constexpr int KCE = EARLY ? KC : 1;
  // EARLY: profile chunks and offsets (descriptor word 0) of the lane's
  // current column ([u & 1]) and next column ([(u + 1) & 1]): U is even, so
  // the two sets alternate through the unrolled block without copies
  uint4 pa[2][KCE], pb[2][KCE];
  uint32_t w0b[2] = {nul.w0, nul.w0};
  bool solo_left = true, solo_checked = false, solo_idle = false;   // EARLY solo claims (lane G-1)
  // EARLY, lane G-1: descriptors of lane 0's next column ([u & 1]) and the one
  // after ([(u + 1) & 1]); other lanes keep zeros (word 0 enters an IMAD)
  DescWords dq[2] = {{0u, 0u, 0u, 0u}, {0u, 0u, 0u, 0u}};
  // EARLY: all KC profile chunks (4 rows each; the narrow tail) of the column whose
  // descriptor word 0 is w
  auto load_prof = [&](uint32_t w, uint4 *xa, uint4 *xb) {
    const uint32_t oB = umulhi(w, 65536u);
    const uint32_t oA = imad(oB, 0xffff0000u, w);
    const uint32_t a = imad(oA, 16u, s_qp), b = imad(oB, 16u, s_qp);
    const uint32_t at = TW ? imad(oA, 16u, s_qpt) : 0u, bt = TW ? imad(oB, 16u, s_qpt) : 0u;
#pragma unroll
    for (int kk = 0; kk < KCE; ++kk) {
      if (kk < KCF) {
        xa[kk] = lds128(a + kk * G * 16);
        xb[kk] = lds128(b + kk * G * 16);
      } else if (TW == 4) {
        xa[kk] = make_uint4(lds32(at), 0u, 0u, 0u);
        xb[kk] = make_uint4(lds32(bt), 0u, 0u, 0u);
      } else {
        const uint2 va = lds64(at), vb = lds64(bt);
        xa[kk] = make_uint4(va.x, va.y, 0u, 0u);
        xb[kk] = make_uint4(vb.x, vb.y, 0u, 0u);
      }
    }
  };
  if (EARLY) load_prof(nul.w0, pa[0], pb[0]);

  // Passes: one per launch (p.pass), or all of them in a cross-pass wavefront
  // (WAVE): the CTA runs pass p's items (profile slice p in shared memory)
  // until pass p's cursor is exhausted, then moves to pass p+1.  An item of
  // pass p reads the boundary and score chain that pass p-1 writes, after
  // checking pass p-1's published progress on that item.
  // (Without WAVE the do-while runs once; the profile slice of p.pass was
  // loaded in the prologue.)
  int pass = p.pass;
  do {
  int *const counter = WAVE ? p.pcounters + pass : p.counter;
  const uint2 *const bnd_in = WAVE ? (pass > 0 ? p.bndbuf[(pass - 1) & 1] : nullptr) : p.bnd_in;
  uint2 *const bnd_out = WAVE ? (pass + 1 < p.npass ? p.bndbuf[pass & 1] : nullptr) : p.bnd_out;
  const bool bout = last && bnd_out != nullptr;
  const int *const prog_in = (WAVE && pass > 0) ? p.progress + (size_t)(pass - 1) * p.num_items : nullptr;
  int *const prog_out = (WAVE && pass + 1 < p.npass) ? p.progress + (size_t)pass * p.num_items : nullptr;
  rem = 0;
  done = false;

  for (;;) {
    if (rem <= 0) {  // group-uniform: claim the next work item
      int it = 0;
      if (last) {
        if (EARLY && G == 32 && p.solo_counter) {
          // solo items (chain-bound, the longest): claimed by warps 0-3 only;
          // warp q + 4 shares warp q's SM sub-partition and stays idle when
          // q's first item is one (the chain keeps the issue slots)
          const int w = (int)(threadIdx.x >> 5);
          volatile int *sl = &s_solo[w & 3];
          if (w < 4) {
            it = solo_left ? atomicAdd(p.solo_counter, 1) : p.solo_end;
            if (it >= p.solo_end) {
              solo_left = false;
              it = atomicAdd(counter, 1);
            }
            if (*sl < 0) *sl = it < p.solo_end ? 1 : 0;
          } else if (!solo_checked) {
            int v;
            while ((v = *sl) < 0) __nanosleep(100);   // warp q claims at once: no dependency
            solo_checked = true;
            solo_idle = v == 1;
            it = solo_idle ? INT_MAX : atomicAdd(counter, 1);
          } else {
            it = solo_idle ? INT_MAX : atomicAdd(counter, 1);
          }
        } else if (WAVE && p.group_limit > 0 &&
                   (int)(threadIdx.x >> 5) + (NT / 32) * (int)((threadIdx.x & 31) / G) >= p.group_limit) {
          it = INT_MAX;   // this group sits the launch out (few units: one or two per SM)
        } else {
          it = atomicAdd(counter, 1);
        }
      }
      it = __shfl_sync(gmask, it, gbase + G - 1);
      if (it < p.num_items) {
        const int sk = (!WAVE && p.skip) ? p.skip[it] : 0;   // dead leading columns (flagged)
        const int64_t c0 = p.items[it].col_begin + sk;
        const int ncols = p.items[it].ncols - sk;
        rem = (ncols + G - 1 + U - 1) & ~(U - 1);
        inc = (uint32_t)U;
        sptr = p.stream + c0;
        if (BIN) bptr = bnd_in ? bnd_in + c0 : p.zero_bnd;
        bcols = (BIN && bnd_in) ? ncols : 0;   // no input boundary: every column reads as zero
        scp = (SCEND && !last) ? reinterpret_cast<uint32_t *>(dummy) : p.sc_out + (c0 - (G - 1));
        scinc = (SCEND && !last) ? 0u : (uint32_t)U;
        if (bnd_out) bop = bnd_out + (c0 - (G - 1));
        if (WAVE) {
          scin = p.sc_out + c0;
          cur_it = it;
          cur_ncols = ncols;
          sdone = 0;
          avail = 0;
          if (prog_in && last) {   // columns 0..U are read below
            const int need = min(ncols, U + 1);
            while ((avail = ld_acquire(prog_in + it)) < need) __nanosleep(200);
          }
        }
        if (last) {
          // ring slot x % U holds column x; columns 1..U (EARLY: 2..U+1) are prefetched here
          if (EARLY) dq[0] = load_desc(s_desc + __ldg(sptr + 1));   // lane 0's second column (u = 0 next)
#pragma unroll
          for (int u = 1; u <= U; ++u) {
            sring[(u + EARLY) % U] = __ldg(sptr + u + EARLY);
            if (BIN && BRING)
              bring[u % U] = u < bcols ? (WAVE ? ld_cg_v2(bptr + u) : __ldg(bptr + u)) : make_uint2(kB2, kB2);
            if (WAVE) scring[u % U] = u < bcols ? ld_cg(scin + u) : 0u;
          }
          const DescWords d = load_desc(s_desc + __ldg(sptr));   // lane 0's first column
          w0 = d.w0;
          ngoe = d.ngoe;
          nge = d.nge;
          knext = d.kneg;
          const uint2 b0 = bcols > 0 ? (WAVE ? ld_cg_v2(bptr) : __ldg(bptr)) : make_uint2(kB2, kB2);   // ncols >= 4
          hout = b0.x;
          fout = b0.y;
          sc = (WAVE && bcols > 0) ? ld_cg(scin) : 0u;
        }
      } else {
        done = true;
        rem = INT_MAX;
        inc = 0u;
        bcols = 0;
        sptr = p.nul_stream;               // NUL columns
        if (BIN) bptr = p.zero_bnd;        // zero boundary
        scp = reinterpret_cast<uint32_t *>(dummy);
        scinc = 0u;
        bop = dummy;
        if (WAVE) {
          scin = nullptr;
          cur_ncols = 0;
        }
        if (last) {
#pragma unroll
          for (int u = 0; u < U; ++u) { sring[u] = kNulWord; bring[u] = make_uint2(kB2, kB2); }
#pragma unroll
          for (int u = 0; u < (WAVE ? U : 1); ++u) scring[u] = 0u;
          w0 = nul.w0;
          ngoe = nul.ngoe;
          nge = nul.nge;
          knext = nul.kneg;
          if (EARLY) dq[0] = nul;
          hout = kB2;
          fout = kB2;
          sc = 0u;
        }
      }
      if (EARLY) {   // lane 0 starts a new stream: its current column's profile (others keep theirs)
        const uint32_t w00 = __shfl_sync(gmask, w0, gbase + G - 1);
        if (t == 0) {   // the block starts at u = 0
          w0b[0] = w00;
          load_prof(w00, pa[0], pb[0]);
        }
      }
    }
    if (__all_sync(0xffffffffu, done)) break;
    if (WAVE && prog_in && last && cur_ncols > 0) {
      // this block reads the boundary of columns up to sdone + 2U: wait until
      // pass p-1 has published them
      const int need = min(cur_ncols, sdone + 2 * U + 1);
      while (avail < need) {
        avail = ld_acquire(prog_in + cur_it);
        if (avail < need) __nanosleep(200);
      }
    }

#pragma unroll
    for (int u = 0; u < U; ++u) {
      // ---- this column's inputs from lane t-1 (lane 0: from lane G-1)
#if SW_SHFLORD
      // (experiment) the chain values first, then the descriptor words
      const uint32_t hu = __shfl_sync(0xffffffffu, hout, src);
      uint32_t F = __shfl_sync(0xffffffffu, fout, src);
      if (!EARLY) w0 = __shfl_sync(0xffffffffu, w0, src);
      ngoe = __shfl_sync(0xffffffffu, ngoe, src);
      nge = __shfl_sync(0xffffffffu, nge, src);
      knext = __shfl_sync(0xffffffffu, knext, src);
      const uint32_t sc_in = __shfl_sync(0xffffffffu, sc, src);
#else
      if (!EARLY) w0 = __shfl_sync(0xffffffffu, w0, src);
      ngoe = __shfl_sync(0xffffffffu, ngoe, src);
      nge = __shfl_sync(0xffffffffu, nge, src);
      knext = __shfl_sync(0xffffffffu, knext, src);
      const uint32_t hu = __shfl_sync(0xffffffffu, hout, src);
      uint32_t F = __shfl_sync(0xffffffffu, fout, src);
      const uint32_t sc_in = __shfl_sync(0xffffffffu, sc, src);
#endif
      // EARLY: the next column's profile offsets (lane G-1 sends lane 0's next
      // column's) and its profile chunks, loaded during this column's rows
      if (EARLY) {
        w0b[(u + 1) & 1] = __shfl_sync(0xffffffffu, imad(w0b[u & 1], nlast, dq[u & 1].w0), src);
        load_prof(w0b[(u + 1) & 1], pa[(u + 1) & 1], pb[(u + 1) & 1]);
      }
      // ---- profile addresses (FMA pipe)
      const uint32_t offB = umulhi(w0, 65536u);           // profile offsets / 16
      const uint32_t offA = imad(offB, 0xffff0000u, w0);
      const uint32_t aA = imad(offA, 16u, s_qp);
      const uint32_t aB = imad(offB, 16u, s_qp);
#if SW_TAILADDR == 0
      const uint32_t aAt = TW ? imad(offA, 16u, s_qpt) : 0u;   // narrow tail chunk
      const uint32_t aBt = TW ? imad(offB, 16u, s_qpt) : 0u;
#else
      const uint32_t aAt = TW ? imad(aA, one, s_dqt) : 0u;   // narrow tail chunk
      const uint32_t aBt = TW ? imad(aB, one, s_dqt) : 0u;
#endif
      // profile chunk kk of the lane's rows (4 rows; the narrow tail: R % 4 rows)
      auto ldq = [&](uint32_t a, uint32_t at, int kk) -> uint4 {
        if (kk < KCF) return lds128(a + kk * G * 16);
        if (TW == 4) return make_uint4(lds32(at), 0u, 0u, 0u);
        const uint2 v = lds64(at);
        return make_uint4(v.x, v.y, 0u, 0u);
      };
      // S is reset after every separator column (END: the score was just read
      // from the chain; NUL: S is already 0): -32768 in each separator half.
      const uint32_t kneg_prev = kneg;
      kneg = knext;
      // ---- lane G-1: lane 0's next column (s+u+1) descriptor; refill its ring slot
      uint2 bnext = make_uint2(bdef, bdef);   // added to the outgoing (H, F): 0 for lanes t < G-1
      uint32_t scnext = 0u;                   // WAVE: lane 0's score-chain input (previous pass)
      // descriptor of lane 0's next column: loaded after the rows (lane G-1
      // still needs its own column's penalty words)
      const uint32_t dnext = sring[(u + 1) % U];
      if (last) {
        SW_CHECK(sptr == p.nul_stream ? (u + 1 + EARLY + U < 16)
                                      : (sptr + u + 1 + EARLY + U - p.stream >= p.col_lo &&
                                         sptr + u + 1 + EARLY + U - p.stream < p.col_hi));
        if (EARLY) {   // lane 0's column after next
          // (s_desc + word, from lane G-1's s_qp: s_desc is otherwise rematerialised per column)
          dq[(u + 1) & 1] = load_desc(s_qp + sring[(u + 2) % U] - (uint32_t)(DESC_U4 * 16 + (G - 1) * 16));
          sring[(u + 2) % U] = __ldg(sptr + u + 2 + U);
        } else {
          sring[(u + 1) % U] = __ldg(sptr + u + 1 + U);
        }
        if (BIN && BRING) {
          bnext = bring[(u + 1) % U];
          SW_CHECK(u + 1 + U >= bcols || (bptr + u + 1 + U - bnd_in >= p.col_lo &&
                                           bptr + u + 1 + U - bnd_in < p.col_hi));
          bring[(u + 1) % U] = (u + 1 + U < bcols)
                                   ? (WAVE ? ld_cg_v2(bptr + u + 1 + U) : __ldg(bptr + u + 1 + U))
                                   : make_uint2(kB2, kB2);
        } else if (BIN) {
          // no ring: the boundary is loaded here and first used after the rows
          SW_CHECK(u + 1 >= bcols || (bptr + u + 1 - bnd_in >= p.col_lo && bptr + u + 1 - bnd_in < p.col_hi));
          bnext = (u + 1 < bcols) ? __ldg(bptr + u + 1) : make_uint2(kB2, kB2);
        }
        if (WAVE) {
          scnext = scring[(u + 1) % U];
          scring[(u + 1) % U] = (u + 1 + U < bcols) ? ld_cg(scin + u + 1 + U) : 0u;
        }
      }
      uint32_t hd = hprev;
      hprev = hu;
      if (QPM == 1) {
        // Score profile: P(r) = SP[pair][q_r], one
        // 32-bit word SM(q_r, dB) * 65536 + SM(q_r, dA) per (letter pair, query
        // letter), read with one LDS.32 per row at the lane's own query letter;
        // no packing IMAD.  w0 is the column pair's byte offset in SP.
        uint32_t tcur = imad(hd, one, lds32(imad(w0, one, qoff[0])));
#pragma unroll
        for (int r = 0; r < R; ++r) {
          uint32_t tnext = 0u;
          if (r + 1 < R) tnext = imad(H[r], one, lds32(imad(w0, one, qoff[r + 1 < R ? r + 1 : 0])));
          const uint32_t h = hmax3(tcur, E[r], F);     // Eq. 1 (0 implicit: E >= kB2)
          H[r] = h;
          const uint32_t hg = haddmax(h, ngoe, kB2);  // max(H-Goe, 0)
          E[r] = haddmax(E[r], nge, hg);              // Eq. 2 (next column)
          F = haddmax(F, nge, hg);                    // Eq. 3 (next row)
          tcur = tnext;
        }
      } else if (kBiased && (SW_ROWAHEAD >= 0 ? (SW_ROWAHEAD == 1 || EARLY) : RA) && SW_ABLATE == 0) {
        // Biased rows with the diagonal add one row ahead: t(r+1) = H_old[r] + P(r+1)
        // is formed before H[r] is overwritten, so the new H can take the old H's
        // register (no per-column rotation of the H registers, which otherwise
        // costs a register permutation at every loop back-edge).
        // P(r) = SM(q_r, dB) * 65536 + SM(q_r, dA) (QPM 0) or the profile word (QPM 3).
        uint4 ca = EARLY ? pa[u & 1][0] : ldq(aA, aAt, 0);
        uint4 cb = EARLY ? pb[u & 1][0] : (QPM == 0 ? ldq(aB, aBt, 0) : make_uint4(0u, 0u, 0u, 0u));
        uint32_t tcur = imad(hd, one, QPM == 0 ? imad(cb.x, 65536u, ca.x) : ca.x);
#pragma unroll
        for (int kk = 0; kk < KC; ++kk) {
          SW_CHECK(kk >= KCF || (aA + kk * G * 16 + 16 <= s_desc + (DESC_U4 + QP_U4) * 16 &&
                                 aB + kk * G * 16 + 16 <= s_desc + (DESC_U4 + QP_U4) * 16));
          SW_CHECK(kk < KCF || (aAt + TW <= s_desc + (DESC_U4 + QP_U4) * 16 &&
                                aBt + TW <= s_desc + (DESC_U4 + QP_U4) * 16));
          uint4 na = make_uint4(0u, 0u, 0u, 0u), nb = make_uint4(0u, 0u, 0u, 0u);
          if (kk + 1 < KC) {
            na = EARLY ? pa[u & 1][EARLY ? kk + 1 : 0] : ldq(aA, aAt, kk + 1);
            if (QPM == 0) nb = EARLY ? pb[u & 1][EARLY ? kk + 1 : 0] : ldq(aB, aBt, kk + 1);
          }
          const uint32_t av[8] = {ca.x, ca.y, ca.z, ca.w, na.x, na.y, na.z, na.w};
          const uint32_t bv[8] = {cb.x, cb.y, cb.z, cb.w, nb.x, nb.y, nb.z, nb.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int r = kk * RPC + j;
            if (r < R) {
              uint32_t tnext = 0u;
              if (r + 1 < R)
                tnext = imad(H[r], one, QPM == 0 ? imad(bv[j + 1], 65536u, av[j + 1]) : av[j + 1]);
              if (LROWS) {
                const uint32_t a = hmax(tcur, E[r]);
                const uint32_t uu = haddmax(a, ngoe, kB2);  // max(max(t, E) - Goe, 0): off the F chain
                const uint32_t h = hmax(a, F);              // Eq. 1
                H[r] = h;
                const uint32_t hg = haddmax(h, ngoe, kB2);  // max(H-Goe, 0)
                E[r] = haddmax(E[r], nge, hg);              // Eq. 2 (next column)
                F = haddmax(F, nge, uu);                    // Eq. 3 (next row), Goe >= Ge
              } else {
                const uint32_t h = hmax3(tcur, E[r], F);     // Eq. 1 (0 implicit: E >= kB2)
                H[r] = h;
                const uint32_t hg = haddmax(h, ngoe, kB2);  // max(H-Goe, 0)
                E[r] = haddmax(E[r], nge, hg);              // Eq. 2 (next column)
                F = haddmax(F, nge, hg);                    // Eq. 3 (next row)
              }
              tcur = tnext;
            }
          }
          ca = na;
          cb = nb;
        }
      } else {
#pragma unroll
      for (int kk = 0; kk < KC; ++kk) {
        const uint4 a = ldq(aA, aAt, kk);
        const uint4 b = (QPM == 0 && SW_ABLATE < 2) ? ldq(aB, aBt, kk) : make_uint4(0u, 0u, 0u, 0u);
        const uint32_t av[4] = {a.x, a.y, a.z, a.w};
        const uint32_t bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int r0 = kk * RPC + j;
          if (r0 < R) {
            // QPM 0: (SM(q_r, dA), SM(q_r, dB)); QPM 3: (SM(q1_r, d), SM(q2_r, d))
            // SW_ABLATE (performance experiments only; results are wrong): 1 = no
            // half packing, 2 = no B profile load and no packing
            const uint32_t sub0 = (QPM == 0 && SW_ABLATE == 0) ? imad(bv[j], 65536u, av[j]) : av[j];
#pragma unroll
            for (int e = 0; e < 1; ++e) {
              const int r = r0 + e;
              if (r < R) {
                const uint32_t sub = sub0;
                uint32_t h;
                if (kBiased) {
                  // biased: H, E, F >= kB2 halfwise, so Hdiag + SM never crosses a
                  // half boundary and is one 32-bit add (FMA pipe); E >= kB2
                  // makes the 0 of Eq. 1 implicit
                  h = hmax3(imad(hd, one, sub), E[r], F);     // Eq. 1
                  hd = H[r];
                  H[r] = h;
                  const uint32_t hg = haddmax(h, ngoe, kB2);  // max(H-Goe, 0)
                  E[r] = haddmax(E[r], nge, hg);              // Eq. 2 (next column)
                  F = haddmax(F, nge, hg);                    // Eq. 3 (next row)
                } else {
                  h = __viaddmax_s16x2_relu(hd, sub, E[r]);  // max(Hdiag+SM, E, 0)
                  h = __vmaxs2(h, F);                        // Eq. 1
                  hd = H[r];
                  H[r] = h;
                  const uint32_t hg = __viaddmax_s16x2_relu(h, ngoe, ngoe);  // max(H-Goe, 0): ngoe <= 0, one register read fewer
                  E[r] = __viaddmax_s16x2(E[r], nge, hg);                    // Eq. 2 (next column)
                  F = __viaddmax_s16x2(F, nge, hg);                          // Eq. 3 (next row)
                }
              }
            }
          }
        }
      }
      }
      // S = max(S reset at the previous END, H_0 .. H_{R-1}); the reset adds
      // -32768 to a half in [0, 32767] (no wrap), folded into the first max.
      S = haddmax(S, kneg_prev, H[0]);
#pragma unroll
      for (int r = 1; r + 1 < R; r += 2) S = hmax3(S, H[r], H[r + 1]);
      if ((R & 1) == 0) S = hmax(S, H[R - 1]);
      const uint32_t so = hmax(sc_in, S);   // max over lanes 0..t (read at END columns)
      SW_CHECK(!last || scp == reinterpret_cast<uint32_t *>(dummy) ||
               (scp + u - p.sc_out >= p.col_lo && scp + u - p.sc_out < p.col_hi));
      SW_CHECK(!bout || bop == dummy || (bop + u - bnd_out >= p.col_lo && bop + u - bnd_out < p.col_hi));
      if (last) {
        // s_desc + dnext, written from lane G-1's own s_qp (t = G-1): a register
        // the loop keeps anyway (s_desc itself is rematerialised per column
        // from SR_CgaCtaId under the register cap: 4 instructions)
        // DA (per instantiation, desc_from_qp): the same address from lane G-1's
        // own s_qp; the two forms compile to different register allocations
        // of the main loop, worth -1..+2% by tile (profiles/r02b_descaddr_calibration.jsonl)
        constexpr bool DAx = SW_DESCADDR >= 0 ? SW_DESCADDR == 1 : DA;
        const DescWords d = EARLY ? dq[u & 1]
                                  : load_desc(DAx ? s_qp + dnext - (uint32_t)(DESC_U4 * 16 + (G - 1) * 16)
                                                  : s_desc + dnext);
        if (!EARLY) w0 = d.w0;   // (EARLY: word 0 went to lane 0 one step ago)
        ngoe = d.ngoe;
        nge = d.nge;
        knext = d.kneg;
      }
      // the score chain is read at END columns only (and, in the wavefront,
      // at every column by the next pass): SW_SCEND stores separator columns only
      if (SCEND ? kneg != 0u : last) st_global_u32(scp + u, so);
      if (bout) st_global_v2(bop + u, H[R - 1], F);
      // outgoing registers; lane G-1 hands over lane 0's next-column inputs
      hout = imad(H[R - 1], nlast, bnext.x);
      fout = imad(F, nlast, bnext.y);
      sc = imad(so, nlast, scnext);
    }
    rem -= U;
    if (BIN) bcols -= U;
    sptr = ptr_add(sptr, inc);
    if (BIN) bptr = ptr_add(bptr, inc);
    scp = ptr_add(scp, SCEND ? scinc : inc);
    bop = ptr_add(bop, inc);
    if (WAVE) {
      if (scin) scin += U;
      sdone += U;
      // publish the columns whose boundary and chain value are now stored
      // (lane G-1 stores column s - (G-1) at step s); release orders the
      // stores.  A release store waits for the earlier stores to complete, so
      // it is issued every kWavePublish columns and when the item ends.
      if (prog_out && last && cur_ncols > 0 && ((sdone & (kWavePublish - 1)) == 0 || rem <= 0))
        st_release(prog_out + cur_it, min(cur_ncols, max(0, sdone - (G - 1))));
    }
  }
  if (WAVE) {   // next pass: every group of the CTA has left this slice
    if (++pass >= p.npass) break;
    __syncthreads();
    const uint4 *gq = p.qp + (size_t)pass * QP_U4;
    for (int i = threadIdx.x; i < QP_U4; i += blockDim.x) smem[DESC_U4 + i] = gq[i];
    __syncthreads();
  }
  } while (WAVE);
}

// ---------------------------------------------------------------------------
// Rows mode (row a5): long database sequences laid along the
// ROWS.  A long pair (one sequence per half of a leading work item) is the
// "query" of a wavefront over its passes and the real query is the column
// stream: the same recurrence on the transposed matrix (E and F swap roles,
// both use Goe / Ge; the score is the maximum over the matrix, so it is
// unchanged).  One CTA takes one item at a time (atomic item counter); warp w
// runs passes w, w+8, w+16, ... (32 lanes x kRowsR rows each), building the
// pass's pre-packed profile (SM(c, dB_row) * 65536 + SM(c, dA_row) per query
// letter: no packing IMAD) in its own shared memory.  Warp w hands its bottom
// boundary (H, F) and score chain to warp w+1 per column through a
// shared-memory ring with producer / consumer counters (the wavefront stays
// on the SM: no release/acquire round trip through L2 per hand-over); warp 7
// hands to warp 0 (the next pass after a multiple of 8) through a per-CTA
// buffer of one pass in global memory -- one buffer is enough: warp 7 can only
// produce column c of its next pass after warp 0 has read column c of this
// one.  The chain value at the query's END column after the last pass is the
// pair's score; it is written into the END columns of the sequences in the
// stream image, where the ordinary score gather reads it.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kRowsWarps * 32, 1) sw16_rows_kernel(const RowsParams p) {
  constexpr int R = kRowsR, G = 32, KC = R / 4, NW = kRowsWarps, RS = kRowsRing, D = kRowsAhead;
  static_assert(R % 4 == 0, "rows-mode profile chunks");
  static_assert((RS & (RS - 1)) == 0 && (D & (D - 1)) == 0 && D >= 2, "ring sizes (D even: two column register sets)");
  extern __shared__ uint4 rsm[];
  uint4 *sdesc = rsm;                                          // [kNL] column descriptors
  int32_t *sM = reinterpret_cast<int32_t *>(rsm + kNL);        // [kNL][kNL]: SM(query letter, db letter)
  char *const sraw = reinterpret_cast<char *>(rsm);
  uint4 *ring = reinterpret_cast<uint4 *>(sraw + kRowsHeadBytes + NW * kNL * kRowsLS);   // [NW-1][RS]
  // ring w: NB batch slots of kRowsBatch columns, each with a "full" and an "empty" mbarrier
  constexpr int B = kRowsBatch, NB = RS / B;
  uint64_t *mb = reinterpret_cast<uint64_t *>(ring + (NW - 1) * RS);                    // [NW-1][2][NB]
  const uint32_t s_mb = (uint32_t)__cvta_generic_to_shared(mb);
  auto mb_full = [&](int w, int j) { return s_mb + (uint32_t)(((w * 2 + 0) * NB + j) * 8); };
  auto mb_empty = [&](int w, int j) { return s_mb + (uint32_t)(((w * 2 + 1) * NB + j) * 8); };
  volatile int *prod = reinterpret_cast<volatile int *>(mb + (NW - 1) * 2 * NB);        // [NW] (prod[7]: the wrap)
  volatile int *cons = prod + NW;                                                       // [NW] columns consumed
  volatile int *s_item = cons + NW;
  uint8_t *sq = reinterpret_cast<uint8_t *>(const_cast<int *>(s_item + 4));   // [ncq] query stream letters
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(rsm);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = lane;
  const int src = (t + G - 1) & (G - 1);
  const bool last = t == G - 1;
  const uint32_t nlast = last ? 0u : 1u;
  const uint32_t bdef = last ? kB2 : 0u;
  const uint32_t one = p.one;
  const uint32_t s_qp = sbase + kRowsHeadBytes + (uint32_t)warp * (kNL * kRowsLS) + t * 16;
  uint4 *const wrap = p.wrap + (size_t)blockIdx.x * p.ncq;    // warp 7 -> warp 0, one pass
  for (int i = threadIdx.x; i < kNL; i += blockDim.x) {
    const bool sep = i >= kAlpha;
    const uint32_t pgoe = (uint32_t)(uint16_t)(-(int)min(p.goe, 32767));
    const uint32_t pge = (uint32_t)(uint16_t)(-(int)min(p.ge, 32767));
    const uint32_t wgoe = sep ? 0x80018001u : (pgoe | (pgoe << 16));
    const uint32_t wge = sep ? 0x80018001u : (pge | (pge << 16));
    sdesc[i] = make_uint4((uint32_t)(i * kRowsLS / 16), wgoe, wge, sep ? 0x80008000u : 0u);
  }
  for (int i = threadIdx.x; i < kNL * kNL; i += blockDim.x) {
    const int c = i / kNL, d = i % kNL;
    sM[i] = (c < kAlpha && d < kAlpha) ? (int32_t)p.matrix[c * kAlpha + d] : kDummy16;
  }
  const int ncq = p.ncq, m = p.m;
  for (int i = threadIdx.x; i < ncq; i += blockDim.x)
    sq[i] = (uint8_t)(i < m ? p.query[i] : (i == m ? kEnd : kNul));

  for (;;) {
    __syncthreads();   // every warp has left the previous item
    if (threadIdx.x == 0) {
      *s_item = atomicAdd(p.counter, 1);
      for (int w = 0; w < NW; ++w) { prod[w] = 0; cons[w] = 0; }
      for (int w = 0; w + 1 < NW; ++w)
        for (int j = 0; j < NB; ++j) {
          mbar_init(mb_full(w, j), 1);
          mbar_init(mb_empty(w, j), 1);
        }
    }
    __syncthreads();
    const int k = *s_item;
    if (k >= p.n_items) break;
    const Item it = p.items[k];
    const int32_t sA = p.slots[it.seqA];
    const int32_t sB = it.nB ? p.slots[it.seqB] : -1;
    const int64_t oA = p.offs[sA], nA = p.offs[sA + 1] - oA;
    const int64_t oB = sB >= 0 ? p.offs[sB] : 0, nB = sB >= 0 ? p.offs[sB + 1] - oB : 0;
    const int npass = (int)((max(nA, nB) + G * R - 1) / (G * R));

    for (int pass = warp; pass < npass; pass += NW) {
      // ---- this lane's profile rows: SM(c, dB_row) * 65536 + SM(c, dA_row)
      __syncwarp();
#pragma unroll
      for (int kk = 0; kk < KC; ++kk) {
        int a[4], b[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int64_t row = (int64_t)pass * G * R + t * R + kk * 4 + e;
          a[e] = row < nA ? (int)__ldg(p.res + oA + row) : -1;
          b[e] = row < nB ? (int)__ldg(p.res + oB + row) : -1;
        }
        for (int c = 0; c < kNL; ++c) {
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int lo = a[e] >= 0 ? sM[c * kNL + a[e]] : kDummy16;
            const int hi = b[e] >= 0 ? sM[c * kNL + b[e]] : kDummy16;
            w[e] = (uint32_t)(hi * 65536 + lo);
          }
          st_shared_v4(s_qp + c * kRowsLS + kk * G * 16, w[0], w[1], w[2], w[3]);
        }
      }
      __syncwarp();
      // inputs: pass 0 none; warp w > 0 from ring[w-1]; warp 0 from the wrap buffer
      const bool has_in = pass > 0;
      const bool in_ring = has_in && warp > 0;
      const int nbp = (ncq + B - 1) / B;   // ring batches per pass (a pass starts a batch)
      const int in_base = in_ring ? (pass / NW) * nbp * B : (pass / NW - 1) * ncq;   // producer's running column
      // outputs: the last pass none; warp w < 7 into ring[w]; warp 7 into the wrap buffer
      const bool has_out = pass + 1 < npass;
      const bool out_ring = has_out && warp < NW - 1;
      const int out_base = out_ring ? (pass / NW) * nbp * B : (pass / NW) * ncq;
      uint4 *const rin = ring + (warp > 0 ? warp - 1 : 0) * RS;
      uint4 *const rout = ring + (warp < NW - 1 ? warp : 0) * RS;

      uint32_t H[R], E[R];
#pragma unroll
      for (int r = 0; r < R; ++r) { H[r] = kB2; E[r] = kB2; }
      uint32_t S = 0u, hprev = kB2, kneg_prev = 0u, final_sc = 0u;
      uint32_t hout = kB2, fout = kB2, sc = 0u;
      // Every lane knows its own column (lane t: s - t at step s): the query
      // is the column stream.  Its letter, descriptor and profile chunks are
      // loaded one step ahead, into two register sets that alternate with the
      // unrolled step index (the pass kernel's EARLY scheme, without the
      // descriptor shuffles): the step's chain is shuffle -> rows -> shuffle.
      DescWords dc[2];
      uint4 pc[2][KC];
      auto load_col = [&](int x, DescWords &d, uint4 *pk) {
        const int l = (x >= 0 && x < ncq) ? (int)sq[x] : kNul;
        d = load_desc(sbase + (uint32_t)l * 16u);
        const uint32_t a = imad(d.w0, 16u, s_qp);
#pragma unroll
        for (int kk = 0; kk < KC; ++kk) pk[kk] = lds128(a + kk * G * 16);
      };
      load_col(-t, dc[0], pc[0]);
      // lane 31's prefetch ring of the previous pass's boundary (H, F, chain)
      // for lane 0's columns: slot j holds column s + 1 (+ j rotation), D
      // columns ahead.  The producer's count is re-read (and fenced) only when
      // the cached value does not cover the column.
      uint4 rv[D];
      int avail = 0;
      auto fetch = [&](int col, uint4 &v) {
        v = make_uint4(kB2, kB2, 0u, 0u);
        if (col < ncq && has_in) {
          const int tix = in_base + col;
          if (in_ring) {
            // the first column of a batch: wait (suspended, no spinning) for the producer's arrival
            const int bt = tix / B;
            if ((tix & (B - 1)) == 0) mbar_wait(mb_full(warp - 1, bt & (NB - 1)), (uint32_t)((bt / NB) & 1));
            v = rin[tix & (RS - 1)];
            if ((tix & (B - 1)) == B - 1 || col + 1 == ncq) {   // the batch is read: free its slot
              __threadfence_block();
              mbar_arrive(mb_empty(warp - 1, bt & (NB - 1)));
            }
          } else {   // the wrap from warp 7: a count, polled with a sleep (one waiter per CTA)
            if (avail < tix + 1) {
              while ((avail = prod[NW - 1]) < tix + 1) __nanosleep(64);
              __threadfence_block();
            }
            v = wrap[col];
          }
        }
      };
      if (last) {
        uint4 v0;
        fetch(0, v0);   // columns in order: a batch's first column waits for the batch
#pragma unroll
        for (int j = 0; j < D; ++j) fetch(j + 1, rv[j]);
        hout = v0.x;
        fout = v0.y;
        sc = v0.z;
      }
      const int nsteps = ncq + G - 1;
#if SW_ROWS_TRACE
      const long long tr0 = clock64();
#endif
      for (int s0 = 0; s0 < nsteps; s0 += D) {
#pragma unroll
        for (int v = 0; v < D; ++v) {
          const int s = s0 + v;
          const uint32_t hu = __shfl_sync(0xffffffffu, hout, src);
          uint32_t F = __shfl_sync(0xffffffffu, fout, src);
          const uint32_t sc_in = __shfl_sync(0xffffffffu, sc, src);
          load_col(s + 1 - t, dc[(v + 1) & 1], pc[(v + 1) & 1]);   // the next column, during these rows
          const uint32_t ngoe = dc[v & 1].ngoe, nge = dc[v & 1].nge;
          uint2 bnext = make_uint2(bdef, bdef);
          uint32_t scnext = 0u;
          if (last) {   // slot v holds column s + 1; refill it with column s + 1 + D
            bnext = make_uint2(rv[v].x, rv[v].y);
            scnext = rv[v].z;
            fetch(s + 1 + D, rv[v]);
          }
          uint32_t hd = hprev;
          hprev = hu;
          uint32_t tcur = imad(hd, one, pc[v & 1][0].x);
#pragma unroll
          for (int kk = 0; kk < KC; ++kk) {
            const uint4 ca = pc[v & 1][kk];
            const uint4 na = kk + 1 < KC ? pc[v & 1][kk + 1 < KC ? kk + 1 : 0] : make_uint4(0u, 0u, 0u, 0u);
            const uint32_t av[8] = {ca.x, ca.y, ca.z, ca.w, na.x, na.y, na.z, na.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int r = kk * 4 + j;
              uint32_t tnext = 0u;
              if (r + 1 < R) tnext = imad(H[r], one, av[j + 1]);
              // Eq. 3 with a one-instruction chain (LROWS, the pass kernel): Goe >= Ge
              const uint32_t a = hmax(tcur, E[r]);
              const uint32_t uu = haddmax(a, ngoe, kB2);  // max(max(t, E) - Goe, 0)
              const uint32_t h = hmax(a, F);              // Eq. 1
              H[r] = h;
              const uint32_t hg = haddmax(h, ngoe, kB2);  // max(H-Goe, 0)
              E[r] = haddmax(E[r], nge, hg);              // Eq. 2 (along the query)
              F = haddmax(F, nge, uu);                    // Eq. 3 (along the database sequence)
              tcur = tnext;
            }
          }
          S = haddmax(S, kneg_prev, H[0]);
#pragma unroll
          for (int r = 1; r + 1 < R; r += 2) S = hmax3(S, H[r], H[r + 1]);
          if ((R & 1) == 0) S = hmax(S, H[R - 1]);
          kneg_prev = dc[v & 1].kneg;
          const uint32_t so = hmax(sc_in, S);
          if (last) {
            const int col = s - (G - 1);
            if (col >= 0 && col < ncq) {
              if (col == m) final_sc = so;
              if (has_out) {
                const int tix = out_base + col;
                const uint4 o = make_uint4(H[R - 1], F, so, 0u);
                if (out_ring) {
                  const int bt = tix / B;
                  // a new batch slot: wait until warp w+1 has read it in the previous round
                  if ((tix & (B - 1)) == 0 && bt >= NB)
                    mbar_wait(mb_empty(warp, bt & (NB - 1)), (uint32_t)((bt / NB - 1) & 1));
                  rout[tix & (RS - 1)] = o;
                  if ((tix & (B - 1)) == B - 1 || col + 1 == ncq) mbar_arrive(mb_full(warp, bt & (NB - 1)));
                } else {
                  wrap[col] = o;
                  if (((col + 1) & (kRowsPublish - 1)) == 0 || col + 1 == ncq) {
                    __threadfence_block();
                    prod[warp] = tix + 1;
                  }
                }
              }
            }
          }
          hout = imad(H[R - 1], nlast, bnext.x);
          fout = imad(F, nlast, bnext.y);
          sc = imad(so, nlast, scnext);
        }
      }
#if SW_ROWS_TRACE
      if (last && k == 0 && pass < 64)
        printf("trace item 0 pass %d warp %d block %d: %lld cycles for %d steps (%lld per step), start %lld\n", pass,
               warp, blockIdx.x, clock64() - tr0, nsteps, (clock64() - tr0) / nsteps, tr0);
#endif
      // the pair's scores (chain at the END column after the last pass) into
      // the END columns of its sequences in the stream image
      if (last && pass + 1 == npass) {
        st_global_u32(p.sc_out + (p.endcol[sA] >> 1), final_sc);
        if (sB >= 0) st_global_u32(p.sc_out + (p.endcol[sB] >> 1), final_sc);
      }
    }
  }
}

// Scores of one pass from the per-column score chain: the value at a
// sequence's END column.  Max over passes;
// flag the 16-bit saturation test.  Two launches per pass:
//   detect: a sequence whose stored 16-bit score reaches thresh is flagged
//           (flag byte = first flagging pass + 1); with the biased-unsigned
//           arithmetic a flagged LOW half (half A, or query 1 of a pair) marks
//           its work item "hot": once its H passes 65536 - SM the 32-bit
//           diagonal add carries into the high half (R7);
//   update: every HIGH-half sequence of a hot item (every query-2 half of a
//           sequence whose query-1 half flagged) is flagged in the same pass
//           -- its 16-bit values may carry that +1 from this pass on, and its
//           32-bit re-scoring starts from this pass's exact input boundary --
//           the other unflagged sequences take max(score, this pass's value).
__global__ void sw16_detect_kernel(const int64_t *__restrict__ endcol, int64_t count,
                                   const uint32_t *__restrict__ sc_out, uint8_t *flagged, uint8_t *flagged2,
                                   bool pairq, int pass, int thresh, const int32_t *__restrict__ seq_idx,
                                   const int32_t *__restrict__ item_of, uint8_t *item_hot) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    // seq_idx (streamed databases): entry i describes original sequence seq_idx[i]
    // and endcol is relative to the current chunk
    const int64_t o = seq_idx ? (int64_t)seq_idx[i] : i;
    const int64_t e = endcol[i];
    const uint32_t w = sc_out[e >> 1];
    const int flag = min(pass + 1, 255);
    if (flagged[o] == 0) {
      const int v = (int)((!pairq && (e & 1)) ? (w >> 16) : (w & 0xffffu));
      if (v >= thresh) {
        flagged[o] = (uint8_t)flag;
        if (kArith == 2) {   // a flagged low half may carry into the high half
          if (pairq) {
            if (flagged2[o] == 0) flagged2[o] = (uint8_t)flag;
          } else if ((e & 1) == 0 && item_of) {
            item_hot[item_of[o]] = 1;
          }
        }
      }
    }
    if (pairq && flagged2[o] == 0 && (int)(w >> 16) >= thresh) flagged2[o] = (uint8_t)flag;
  }
}

__global__ void sw16_update_kernel(const int64_t *__restrict__ endcol, int64_t count,
                                   const uint32_t *__restrict__ sc_out, int32_t *scores, uint8_t *flagged,
                                   int32_t *scores2, const uint8_t *__restrict__ flagged2, int pass,
                                   const int32_t *__restrict__ seq_idx, const int32_t *__restrict__ item_of,
                                   const uint8_t *__restrict__ item_hot, int32_t *list, int *nlist,
                                   int32_t *list2, int *nlist2, int want) {
  const int lane = threadIdx.x & 31;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < count; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    bool f1 = false, f2 = false;
    int64_t o = 0;
    if (i < count) {
      o = seq_idx ? (int64_t)seq_idx[i] : i;
      const int64_t e = endcol[i];
      const uint32_t w = sc_out[e >> 1];
      // once flagged, the 32-bit kernel owns the score (started from the last
      // exact pass boundary, or from row 0)
      int fl = flagged[o];
      if (fl == 0) {
        if (kArith == 2 && !scores2 && (e & 1) && item_of && item_hot[item_of[o]]) {
          fl = min(pass + 1, 255);
          flagged[o] = (uint8_t)fl;
        } else {
          const int v = (int)((!scores2 && (e & 1)) ? (w >> 16) : (w & 0xffffu));
          scores[o] = max(pass == 0 ? 0 : scores[o], v - kBias16);
        }
      }
      if (scores2 && flagged2[o] == 0) scores2[o] = max(pass == 0 ? 0 : scores2[o], (int)(w >> 16) - kBias16);
      // the sequences first flagged in this pass, compacted for the 32-bit
      // kernel (flag_compact_kernel's job, fused: one launch fewer per pass)
      f1 = want && fl == want;
      f2 = want && list2 && flagged2[o] == want;
    }
    if (!want) continue;   // uniform
    const unsigned b1 = __ballot_sync(0xffffffffu, f1), b2 = __ballot_sync(0xffffffffu, f2);
    if (b1) {
      int pos = 0;
      if (lane == 0) pos = atomicAdd(nlist, __popc(b1));
      pos = __shfl_sync(0xffffffffu, pos, 0);
      if (f1) list[pos + __popc(b1 & ((1u << lane) - 1u))] = (int32_t)o;
    }
    if (b2) {
      int pos = 0;
      if (lane == 0) pos = atomicAdd(nlist2, __popc(b2));
      pos = __shfl_sync(0xffffffffu, pos, 0);
      if (f2) list2[pos + __popc(b2 & ((1u << lane) - 1u))] = (int32_t)o;
    }
  }
}

// ---------------------------------------------------------------------------
// Exact s32 re-scoring of flagged sequences ("recalculated using
// the next wider integer range").  One warp (G = 32 lanes x R rows) per
// flagged sequence, read from the plain database copy.  The warps of a CTA
// step through the query passes together so that the pass's int32 profile
// slice sits in shared memory ([letter][4-row chunk][lane][16 B]); the pass
// boundary (H, F) goes through per-warp scratch.
// ---------------------------------------------------------------------------
template <int R>
__global__ void __launch_bounds__(kSW32Threads) sw32_kernel(const SW32Params p) {
  extern __shared__ uint4 sq[];
  __shared__ int s_base;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const int gwarp = blockIdx.x * nw + warp;
  const bool first = lane == 0, last = lane == 31;
  const int nfirst = first ? 0 : 1;
  uint2 *buf0 = p.scratch + (size_t)gwarp * 2 * p.stride + 32;
  uint2 *buf1 = buf0 + p.stride;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sq) + lane * 16;
  const int nflag = *p.flag_count;
  const uint32_t one = p.one;

  // First round: a static round-robin share of at most one sequence per warp
  // (CTA b takes b, b + grid, ...: every CTA, and so every SM, gets the same
  // number of sequences when fewer are flagged than there are warps -- with
  // CTA-wide claims of nw sequences, the first CTAs to arrive took them all
  // and a third of the SMs ran one CTA or none).  Later rounds: dynamic
  // claims of nw sequences (uneven lengths).
  const int share = min(nw, (nflag + (int)gridDim.x - 1) / (int)gridDim.x);
  for (int round = 0;; ++round) {
    int idx;
    if (round == 0) {
      if ((int)blockIdx.x >= nflag) continue;     // CTA-uniform: nothing static for this CTA
      idx = warp < share ? (int)blockIdx.x + warp * (int)gridDim.x : nflag;
    } else {
      __syncthreads();
      if (threadIdx.x == 0) s_base = share * (int)gridDim.x + atomicAdd(p.cursor, nw);
      __syncthreads();
      const int base = s_base;
      if (base >= nflag) break;                    // CTA-uniform
      idx = base + warp;
    }
    const bool active = idx < nflag;
    int orig = 0, n = 0;
    const uint8_t *res = p.res;
    if (active) {
      orig = p.flag_list[idx];
      const int64_t b = p.offs[orig];
      n = (int)(p.offs[orig + 1] - b);
      res = p.res + b;
    }
    // rows < row0 were exact in 16 bit: their maximum is already in scores,
    // and the 16-bit pass boundary of row row0-1 seeds the first pass below
    int best = 0;
    int64_t col0 = 0;
    int half = 0;
    if (active && p.row0 > 0) {
      best = p.scores[orig];
      const int64_t e = p.endcol[orig];
      col0 = (e >> 1) - n;                   // the sequence's first stream column
      half = p.half >= 0 ? p.half : (int)(e & 1);
    }
    // One query pass of RR rows per lane (RR = R, or a narrower last pass:
    // only the rows the query still has are computed, no phantom rows beyond
    // the next multiple of 32 * RR).  CTA-uniform: staging synchronises.
    int64_t rows_done = 0;
    auto run_pass = [&](int pass, auto rr_c) {
      constexpr int RR = decltype(rr_c)::value;
      constexpr int KR = RR / 4;
      __syncthreads();
      // stage this pass's profile slice [letter][4-row chunk][lane][4] from the
      // plain [letter][m] profile, rows row0 + pass*32*R + lane*RR ...
      for (int i = threadIdx.x; i < kNL * KR * 32 * 4; i += blockDim.x) {
        const int e4 = i & 3, ln = (i >> 2) & 31, rest = i >> 7;
        const int kk = rest % KR, c = rest / KR;
        const int row = p.row0 + pass * 32 * R + ln * RR + kk * 4 + e4;
        reinterpret_cast<int32_t *>(sq)[i] = row < p.m ? p.qp32[(int64_t)c * p.m + row] : -(1 << 30);
      }
      __syncthreads();
      rows_done += 32 * RR;
      if (!active) return;
      const uint2 *bin = pass == 0 ? nullptr : ((pass & 1) ? buf0 : buf1);
      const uint2 *b16 = (pass == 0 && p.row0 > 0) ? p.bnd16 + col0 : nullptr;
      uint2 *bout = pass == p.passes - 1 ? nullptr : ((pass & 1) ? buf1 : buf0);
      int H[RR], E[RR];
#pragma unroll
      for (int r = 0; r < RR; ++r) { H[r] = 0; E[r] = 0; }
      int S = 0, hout = 0, fout = 0, hprev = 0, code = kNul;
      // Lane 0's column inputs (letter, boundary H and F of the row above) are
      // fetched 32 columns at a time, one column per lane, coalesced and one
      // 32-column block ahead, and handed to lane 0 by shuffle: no dependent
      // global load per column.  Columns >= n read as NUL with a zero boundary.
      auto fetch = [&](int cb, int &r, int &bh, int &bf) {
        const int c = cb + lane;
        r = kNul;
        bh = 0;
        bf = 0;
        if (c < n) {
          r = (int)res[c];
          if (bin) {
            const uint2 b = bin[c];
            bh = (int)b.x;
            bf = (int)b.y;
          } else if (b16) {                 // exact 16-bit boundary, unbiased
            const uint2 b = b16[c];
            bh = (int)((b.x >> (16 * half)) & 0xffffu) - kBias16;
            bf = (int)((b.y >> (16 * half)) & 0xffffu) - kBias16;
          }
        }
      };
      int rcur, hcur, fcur, rnxt, hnxt, fnxt;
      fetch(0, rcur, hcur, fcur);
      fetch(32, rnxt, hnxt, fnxt);
      const int nsteps = (n + 31 + 3) & ~3;
      for (int c0 = 0; c0 < nsteps; c0 += 4) {
        if (c0 > 0 && (c0 & 31) == 0) {    // warp-uniform
          rcur = rnxt;
          hcur = hnxt;
          fcur = fnxt;
          fetch(c0 + 32, rnxt, hnxt, fnxt);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = c0 + u;
          const int code_up = __shfl_up_sync(0xffffffffu, code, 1);
          const int hu_up = __shfl_up_sync(0xffffffffu, hout, 1);
          const int fu_up = __shfl_up_sync(0xffffffffu, fout, 1);
          const int sel = c & 31;
          const int rc = __shfl_sync(0xffffffffu, rcur, sel);
          const int bh = (int)imad((uint32_t)__shfl_sync(0xffffffffu, hcur, sel), 1u - nfirst, 0u);
          const int bf = (int)imad((uint32_t)__shfl_sync(0xffffffffu, fcur, sel), 1u - nfirst, 0u);
          code = first ? rc : code_up;
          const int hu = hu_up * nfirst + bh;
          int F = fu_up * nfirst + bf;
          const uint32_t qa = sbase + (uint32_t)code * (KR * 32 * 16);
          int hd = hprev;
          hprev = hu;
#pragma unroll
          for (int kk = 0; kk < KR; ++kk) {
            const uint4 a = lds128(qa + kk * 32 * 16);
            const int av[4] = {(int)a.x, (int)a.y, (int)a.z, (int)a.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int r = kk * 4 + e;
              // H_diag + SM as an IMAD on the FMA pipe; E, F >= 0 make the 0 of
              // Eq. 1 implicit, so Eq. 1 is one VIMNMX3 (4.5 ALU per cell, not 5.5)
              const int h = __vimax3_s32((int)imad((uint32_t)hd, one, (uint32_t)av[e]), E[r], F);
              hd = H[r];
              H[r] = h;
              const int hg = __viaddmax_s32_relu(h, p.neg_goe, 0);
              E[r] = __viaddmax_s32(E[r], p.neg_ge, hg);
              F = __viaddmax_s32(F, p.neg_ge, hg);
            }
          }
#pragma unroll
          for (int r = 0; r + 1 < RR; r += 2) S = __vimax3_s32(S, H[r], H[r + 1]);
          hout = H[RR - 1];
          fout = F;
          if (last && bout) bout[c - 31] = make_uint2((uint32_t)hout, (uint32_t)fout);
        }
      }
      best = max(best, S);
      __syncwarp();
    };
    for (int pass = 0; pass < p.passes; ++pass) {
      if constexpr (R % 12 == 0) {
        const int left = p.len - p.row0 - pass * 32 * R;   // query rows from this pass on
        if (pass == p.passes - 1 && left <= 32 * (R / 3)) {
          run_pass(pass, std::integral_constant<int, R / 3>{});
          continue;
        }
        if (pass == p.passes - 1 && left <= 32 * (2 * R / 3)) {
          run_pass(pass, std::integral_constant<int, 2 * R / 3>{});
          continue;
        }
      }
      run_pass(pass, std::integral_constant<int, R>{});
    }
    if (active) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
      if (first) {
        p.scores[orig] = best;
        if (p.cells) atomicAdd(reinterpret_cast<unsigned long long *>(p.cells),
                               (unsigned long long)n * (unsigned long long)rows_done);
      }
    }
  }
}

// Per-search zeroing (replaces four memsets; done by the profile launch).  16-B stores for
// the byte arrays' aligned bulk.
__device__ __forceinline__ void zero_bytes(uint8_t *p, int64_t n, int64_t tid, int64_t nth) {
  if (!p || n <= 0) return;
  const int64_t mis = (16 - (int64_t)(reinterpret_cast<uintptr_t>(p) & 15)) & 15;
  const int64_t head = n < mis ? n : mis;
  const int64_t n16 = (n - head) >> 4;
  uint4 *q = reinterpret_cast<uint4 *>(p + head);
  for (int64_t i = tid; i < n16; i += nth) q[i] = make_uint4(0u, 0u, 0u, 0u);
  for (int64_t i = tid; i < head; i += nth) p[i] = 0;
  for (int64_t i = head + 16 * n16 + tid; i < n; i += nth) p[i] = 0;
}
__device__ __forceinline__ void search_init(const SearchInit &z, int64_t tid, int64_t nth) {
  for (int64_t i = tid; i < z.nfc; i += nth) z.fcounters[i] = 0;
  if (tid == 0 && z.cells32) *z.cells32 = 0;
  zero_bytes(z.flagged, z.count, tid, nth);
  zero_bytes(z.flagged2, z.count, tid, nth);
  zero_bytes(z.item_hot, z.nitems, tid, nth);
}

// ---------------------------------------------------------------------------
// Query profile ("auxiliary two-dimensional array of size
// |q| x |Sigma|"), built per query in the layouts the kernels read.
// ---------------------------------------------------------------------------
__global__ void qp_build_kernel(const uint8_t *__restrict__ q, int m, const uint8_t *__restrict__ q2, int m2,
                                const int8_t *__restrict__ M, int G, int R, int P, uint32_t *qp, uint4 *desc,
                                int32_t *qp32, int32_t *qp32b, int goe, int ge, int sp, const SearchInit ini) {
  search_init(ini, blockIdx.x * (int64_t)blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x);
  // q2 == nullptr: one query (QPM 0); q2 != nullptr: query pair (QPM 3).  See
  // the profile-mode notes above the pass kernel for the word formats.
  // slice layout: kernels.cuh (qp_letter_bytes): full chunks, then a narrow tail block
  const int KCF = qp_full_chunks(R);
  const int TW = qp_tail_w(R) == 16 ? 0 : qp_tail_w(R);
  const int LS = qp_letter_bytes(G, R);
  const int LW = LS / 4;                    // 32-bit words per letter
  const int mm = q2 ? max(m, m2) : m;
  // sp: the score profile SP[pair (cA, cB)][query letter c < kSPL] instead
  const int64_t nq = sp ? (int64_t)kSPBytes / 4 : (int64_t)P * kNL * LW;
  const int64_t ndesc = kNL * kNL;
  const int64_t n32 = (int64_t)kNL * mm;   // plain s32 profile(s)
  const int64_t total = nq + ndesc + n32;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < nq && sp) {
      const int pr = (int)(i / kSPL), c = (int)(i % kSPL);
      const int cA = pr / kNL, cB = pr % kNL;
      const int lo = (c < kAlpha && cA < kAlpha) ? M[c * kAlpha + cA] : kDummy16;
      const int hi = (c < kAlpha && cB < kAlpha) ? M[c * kAlpha + cB] : kDummy16;
      qp[i] = (uint32_t)(hi * 65536 + lo);
    } else if (i < nq) {
      const int w = (int)(i % LW);
      const int c = (int)((i / LW) % kNL);
      const int pass = (int)(i / ((int64_t)LW * kNL));
      int t, rloc;
      if (w < KCF * G * 4) {              // full chunk kk: [kk][t][4 rows]
        t = (w >> 2) % G;
        rloc = 4 * (w / (G * 4)) + (w & 3);
      } else {                            // tail block: [copy][t][TW/4 rows]
        const int u = w - KCF * G * 4, tw = TW / 4;
        t = (u / tw) % G;
        rloc = 4 * KCF + u % tw;
      }
      const int64_t row = (int64_t)pass * G * R + (int64_t)t * R + rloc;
      // kDummy16: separator letters and phantom rows
      int lo = kDummy16, hi = kDummy16;
      if (rloc < R && c < kAlpha) {
        if (row < m) lo = M[q[row] * kAlpha + c];
        if (q2 && row < m2) hi = M[q2[row] * kAlpha + c];
      }
      if (kBiased)   // the 32-bit integer hi * 65536 + lo (added to H_diag as one 32-bit add)
        qp[i] = q2 ? (uint32_t)(hi * 65536 + lo) : (uint32_t)lo;
      else               // zero-extended halves
        qp[i] = q2 ? ((uint32_t)(uint16_t)lo | ((uint32_t)(uint16_t)hi << 16)) : (uint32_t)(uint16_t)lo;
    } else if (i < nq + ndesc) {
      const int k = (int)(i - nq);
      const int cA = k / kNL, cB = k % kNL;
      const uint32_t offA = (uint32_t)(cA * LS / 16), offB = (uint32_t)(cB * LS / 16);
      // Per half, built explicitly (a packed add of the two halves would carry
      // when a penalty is 0): -Goe / -Ge, or -32767 in a separator half (zeroes
      // E and F at the column); the S-reset word -32768 after a separator half.
      const bool sA = cA >= kAlpha, sB = cB >= kAlpha;
      const uint32_t pgoe = (uint32_t)(uint16_t)(-(int)min(goe, 32767));
      const uint32_t pge = (uint32_t)(uint16_t)(-(int)min(ge, 32767));
      const uint32_t wgoe = (sA ? 0x8001u : pgoe) | ((sB ? 0x8001u : pgoe) << 16);
      const uint32_t wge = (sA ? 0x8001u : pge) | ((sB ? 0x8001u : pge) << 16);
      const uint32_t wk = (sA ? 0x8000u : 0u) | ((sB ? 0x8000u : 0u) << 16);
      desc[k] = make_uint4(sp ? (uint32_t)(k * kSPL * 4) : (offA | (offB << 16)), wgoe, wge, wk);
    } else {
      // s32 profile(s), plain [letter][m] (the 32-bit kernel stages its slices)
      const int64_t j = i - nq - ndesc;
      const int c = (int)(j / mm), row = (int)(j % mm);
      qp32[j] = (row < m && c < kAlpha) ? (int32_t)M[q[row] * kAlpha + c] : -(1 << 30);
      if (q2) qp32b[j] = (row < m2 && c < kAlpha) ? (int32_t)M[q2[row] * kAlpha + c] : -(1 << 30);
    }
  }
}

// Leading columns of each item that hold only already-flagged sequences in
// both halves (half A and half B each walk their sequences in column order
// until the first unflagged one; a half whose sequences are all flagged is
// dead to the item's end).  Starting a later pass there is exact for every
// unflagged sequence: the column after a sequence's NUL separator starts from
// H = E = F = 0, which is what a fresh item start gives, and a half whose dead
// run is longer only recomputes part of a flagged sequence, whose 16-bit
// results nobody reads again (the gather skips flagged sequences; their s32
// re-scoring was seeded in the pass that flagged them).
__global__ void item_skip_kernel(const Item *__restrict__ items, int nitems, const int32_t *__restrict__ slots,
                                 const int64_t *__restrict__ offs, const uint8_t *__restrict__ flagged,
                                 int32_t *skip) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nitems; i += gridDim.x * blockDim.x) {
    const Item it = items[i];
    int64_t dead[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int32_t s0 = h ? it.seqB : it.seqA, n = h ? it.nB : it.nA;
      int64_t d = 0;
      int k = 0;
      for (; k < n; ++k) {
        const int32_t o = slots[s0 + k];
        if (!flagged[o]) break;
        d += offs[o + 1] - offs[o] + 2;   // residues, END, NUL
      }
      dead[h] = k == n ? (int64_t)it.ncols : d;
    }
    skip[i] = (int32_t)min(min(dead[0], dead[1]), (int64_t)it.ncols);
  }
}


// 16-bit column words -> 32-bit words (device image upload, out-of-core
// chunks as they arrive over the host link).
__global__ void expand_columns_kernel(const uint16_t *__restrict__ in, int64_t n, uint32_t *__restrict__ out) {
  const int64_t n4 = n >> 2;
  const bool vec = ((reinterpret_cast<uintptr_t>(in) & 7) | (reinterpret_cast<uintptr_t>(out) & 15)) == 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (vec ? n4 : 0);
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint2 v = __ldg(reinterpret_cast<const uint2 *>(in) + i);
    reinterpret_cast<uint4 *>(out)[i] = make_uint4(v.x & 0xffffu, v.x >> 16, v.y & 0xffffu, v.y >> 16);
  }
  for (int64_t i = (vec ? 4 * n4 : 0) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

// Per-search inputs (matrix, query, item cursors) read straight from the
// pinned, mapped staging slot: used instead of a copy-engine memcpy when the
// copy engine is busy with a streamed database's chunks (a small H2D copy
// queues behind a chunk copy of several ms).
__global__ void stage_copy_kernel(const uint32_t *__restrict__ host_src, uint32_t *__restrict__ dst, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = host_src[i];
}

__global__ void flag_compact_kernel(const uint8_t *__restrict__ flagged, int64_t count, int32_t *list,
                                    int *n, int want) {
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < count;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const bool f = i < count && (want ? flagged[i] == want : flagged[i] != 0);
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    if (bal) {
      const int lane = threadIdx.x & 31;
      int pos = 0;
      if (lane == 0) pos = atomicAdd(n, __popc(bal));
      pos = __shfl_sync(0xffffffffu, pos, 0);
      if (f) list[pos + __popc(bal & ((1u << lane) - 1u))] = (int32_t)i;
    }
  }
}

// ---------------------------------------------------------------------------
// Sorting stage: keys = (score, -index) packed so that one
// descending order of 64-bit keys is "score descending, index ascending".
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t make_key(int32_t score, uint64_t idx) {
  return ((uint64_t)((uint32_t)score ^ 0x80000000u) << 32) | (uint64_t)(0xffffffffu - (uint32_t)idx);
}

__global__ void make_keys_kernel(const int32_t *scores, const int64_t *index, int64_t n, uint64_t *keys,
                                 int64_t npad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npad;
       i += (int64_t)gridDim.x * blockDim.x)
    keys[i] = i < n ? make_key(scores[i], index ? (uint64_t)index[i] : (uint64_t)i) : 0ull;
}

__global__ void bitonic_step_kernel(uint64_t *keys, int64_t n, int64_t size, int64_t stride) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n / 2;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = (i / stride) * stride * 2 + (i % stride);
    const int64_t hi = lo + stride;
    const bool desc = ((lo & size) == 0);  // descending blocks give a descending result
    const uint64_t a = keys[lo], b = keys[hi];
    if ((a < b) == desc) { keys[lo] = b; keys[hi] = a; }
  }
}

__global__ void bitonic_local_kernel(uint64_t *keys, int64_t size, int64_t stride_hi) {
  // all strides <= stride_hi (<= 1024) of one bitonic merge stage, in shared memory
  __shared__ uint64_t sk[2048];
  const int64_t base = (int64_t)blockIdx.x * 2048;
  sk[threadIdx.x] = keys[base + threadIdx.x];
  sk[threadIdx.x + 1024] = keys[base + threadIdx.x + 1024];
  __syncthreads();
  for (int64_t stride = stride_hi; stride > 0; stride >>= 1) {
    const int i = threadIdx.x;
    const int lo = (int)((i / stride) * stride * 2 + (i % stride));
    const int hi = lo + (int)stride;
    const bool desc = (((base + lo) & size) == 0);
    const uint64_t a = sk[lo], b = sk[hi];
    if ((a < b) == desc) { sk[lo] = b; sk[hi] = a; }
    __syncthreads();
  }
  keys[base + threadIdx.x] = sk[threadIdx.x];
  keys[base + threadIdx.x + 1024] = sk[threadIdx.x + 1024];
}

// Block-level top-k (k <= 32), the sorting stage's fast path: every warp keeps
// a lane-distributed sorted list of the k best keys of a strided slice (lane i
// holds the i-th largest), with the next batch's load issued before the
// current batch is inserted; warp 0 then merges the block's lists from shared
// memory.  Launched twice: a grid over the scores, then one block over the
// grid's lists.
__device__ __forceinline__ void warp_topk_insert(uint64_t key, uint64_t &L, uint64_t &thr, int k, int lane) {
  unsigned cand = __ballot_sync(0xffffffffu, key > thr);
  while (cand) {
    const int src = __ffs(cand) - 1;
    cand &= cand - 1;
    const uint64_t c = __shfl_sync(0xffffffffu, key, src);
    if (c > thr) {
      const int pos = __popc(__ballot_sync(0xffffffffu, L > c));
      const uint64_t up = __shfl_up_sync(0xffffffffu, L, 1);
      if (lane > pos) L = up;
      if (lane == pos) L = c;
      thr = __shfl_sync(0xffffffffu, L, k - 1);
    }
  }
}

__global__ void __launch_bounds__(1024) block_topk_kernel(const int32_t *scores, const int64_t *index,
                                                          const uint64_t *keys_in, int64_t n, int k,
                                                          uint64_t *out) {
  __shared__ uint64_t s_lists[32 * 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * nwarps + warp;
  const int64_t stride = (int64_t)gridDim.x * nwarps * 32;
  auto load = [&](int64_t i) -> uint64_t {
    if (i >= n) return 0ull;
    return keys_in ? keys_in[i] : make_key(scores[i], index ? (uint64_t)index[i] : (uint64_t)i);
  };
  uint64_t L = 0ull, thr = 0ull;
  int64_t i = gw * 32 + lane;
  uint64_t key = load(i);
  for (int64_t base = gw * 32; base < n; base += stride) {
    const uint64_t next = load(i + stride);   // in flight while this batch is inserted
    warp_topk_insert(key, L, thr, k, lane);
    key = next;
    i += stride;
  }
  s_lists[warp * 32 + lane] = lane < k ? L : 0ull;
  __syncthreads();
  if (warp == 0) {
    L = 0ull;
    thr = 0ull;
    for (int w = 0; w < nwarps; ++w) warp_topk_insert(s_lists[w * 32 + lane], L, thr, k, lane);
    if (lane < k) out[(int64_t)blockIdx.x * k + lane] = L;
  }
}

// Sorting stage for k > 32: radix select of the k-th largest
// 64-bit key (score, -index), 8 passes of 8 bits from the most significant
// digit, then compaction of the k keys >= it and a sort of those k only.
// State in device memory, no host round trip: each pass histograms the digit
// of the keys that match the selected prefix so far, and a one-block kernel
// picks the digit where the count from the top reaches the keys still
// needed.  When every key with the new prefix is needed the selection is
// complete (done) and the remaining passes return at once.
struct SelState {
  uint64_t prefix, mask;
  long long need;
  int done;
};

__global__ void __launch_bounds__(512) radix_hist_kernel(const int32_t *__restrict__ scores,
                                                         const int64_t *__restrict__ index, int64_t n,
                                                         const SelState *__restrict__ st, int shift,
                                                         unsigned *hist) {
  __shared__ unsigned sh[256];
  if (st->done) return;
  for (int b = threadIdx.x; b < 256; b += blockDim.x) sh[b] = 0u;
  __syncthreads();
  const uint64_t prefix = st->prefix, mask = st->mask;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = make_key(scores[i], index ? (uint64_t)index[i] : (uint64_t)i);
    if ((key & mask) == prefix) atomicAdd(&sh[(key >> shift) & 255u], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < 256; b += blockDim.x)
    if (sh[b]) atomicAdd(&hist[b], sh[b]);
}

__global__ void radix_select_kernel(SelState *st, unsigned *hist, int shift) {
  __shared__ unsigned sh[256];
  for (int b = threadIdx.x; b < 256; b += blockDim.x) sh[b] = hist[b];
  __syncthreads();
  if (threadIdx.x == 0 && !st->done) {
    long long cum = 0;
    const long long need = st->need;
    for (int d = 255; d >= 0; --d) {
      if (cum + (long long)sh[d] >= need) {
        st->need = need - cum;
        st->prefix |= (uint64_t)d << shift;
        st->mask |= (uint64_t)255u << shift;
        if ((long long)sh[d] == need - cum) st->done = 1;   // every key with this prefix is needed
        break;
      }
      cum += sh[d];
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < 256; b += blockDim.x) hist[b] = 0u;   // for the next pass
}

// The k selected keys ((key & mask) >= prefix), in any order.
__global__ void radix_gather_kernel(const int32_t *__restrict__ scores, const int64_t *__restrict__ index,
                                    int64_t n, const SelState *__restrict__ st, uint64_t *out, unsigned *cnt) {
  const uint64_t prefix = st->prefix, mask = st->mask;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    uint64_t key = 0;
    bool take = false;
    if (i < n) {
      key = make_key(scores[i], index ? (uint64_t)index[i] : (uint64_t)i);
      take = (key & mask) >= prefix;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, take);
    if (bal) {
      const int lane = threadIdx.x & 31;
      unsigned pos = 0;
      if (lane == 0) pos = atomicAdd(cnt, (unsigned)__popc(bal));
      pos = __shfl_sync(0xffffffffu, pos, 0);
      if (take) out[pos + __popc(bal & ((1u << lane) - 1u))] = key;
    }
  }
}

// One-block descending bitonic sort of n <= 4096 keys (padded with 0).
__global__ void __launch_bounds__(1024) block_sort_desc_kernel(uint64_t *keys, int n, int npow2) {
  __shared__ uint64_t sk[4096];
  for (int i = threadIdx.x; i < npow2; i += blockDim.x) sk[i] = i < n ? keys[i] : 0ull;
  __syncthreads();
  for (int size = 2; size <= npow2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < npow2 / 2; i += blockDim.x) {
        const int lo = (i / stride) * stride * 2 + (i % stride);
        const int hi = lo + stride;
        const bool desc = (lo & size) == 0;
        const uint64_t a = sk[lo], b = sk[hi];
        if ((a < b) == desc) { sk[lo] = b; sk[hi] = a; }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) keys[i] = sk[i];
}

// Sorting stage, multi-GPU: scatter the scores gathered
// from every rank's shard back to the original database order on rank 0,
// dst[index[i]] = src[i]; index < 0 marks the gather's padding slots.  Four
// entries per thread with 16-B loads where aligned (the gathered buffer is
// contiguous and padded per rank); stores are scattered 4-B writes.
__global__ void scatter_scores_kernel(const int32_t *__restrict__ src, const int64_t *__restrict__ index, int64_t n,
                                      int32_t *__restrict__ dst, int64_t dst_count) {
  const int64_t n4 = n >> 2;
  const bool vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(index)) & 15) == 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (vec ? n4 : 0);
       i += (int64_t)gridDim.x * blockDim.x) {
    const int4 s = __ldg(reinterpret_cast<const int4 *>(src) + i);
    const longlong2 a = __ldg(reinterpret_cast<const longlong2 *>(index) + 2 * i);
    const longlong2 b = __ldg(reinterpret_cast<const longlong2 *>(index) + 2 * i + 1);
    if (a.x >= 0 && a.x < dst_count) dst[a.x] = s.x;
    if (a.y >= 0 && a.y < dst_count) dst[a.y] = s.y;
    if (b.x >= 0 && b.x < dst_count) dst[b.x] = s.z;
    if (b.y >= 0 && b.y < dst_count) dst[b.y] = s.w;
  }
  for (int64_t i = (vec ? 4 * n4 : 0) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = index[i];
    if (j >= 0 && j < dst_count) dst[j] = src[i];
  }
}

__global__ void decode_keys_kernel(const uint64_t *keys, int64_t k, int64_t *idx, int32_t *score) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = keys[i];
    score[i] = (int32_t)((uint32_t)(key >> 32) ^ 0x80000000u);
    idx[i] = (int64_t)(0xffffffffu - (uint32_t)(key & 0xffffffffull));
  }
}

// ---------------------------------------------------------------------------
// Tile table.
// ---------------------------------------------------------------------------
using PassFn = void (*)(const SW16Params);

template <int R, int G, int QPM>
constexpr int smem_of() {
  return kNL * kNL * 16 + (QPM == 1 ? kSPBytes : kNL * qp_letter_bytes(G, R));
}

// Per (tile, boundary input, profile mode): 1 when the descriptor address from
// lane G-1's s_qp measured faster than from the shared base (both forms are
// the same instructions; the register allocation of the main loop differs).
// From tools/calibrate_tiles.py under SW_DESCADDR=0 and =1 builds, >= 0.5%
// faster (profiles/r02b_descaddr_calibration.jsonl, tools/descaddr_table.py);
// query-profile throughput tiles only.
struct DescPick { int G, R; bool bin; };
constexpr DescPick kDescFromQp[] = {
    {8, 8, false},
    {8, 8, true},
    {8, 12, false},
    {8, 12, true},
    {8, 16, false},
    {8, 16, true},
    {8, 18, false},
    {8, 18, true},
    {8, 20, false},
    {8, 20, true},
    {8, 22, false},
    {8, 22, true},
    {8, 24, false},
    {8, 24, true},
    {8, 26, false},
    {8, 26, true},
    {8, 28, false},
    {8, 28, true},
    {8, 29, true},
    {8, 30, false},
    {8, 30, true},
    {16, 8, false},
    {16, 8, true},
    {16, 12, false},
    {16, 12, true},
    {16, 16, false},
    {16, 16, true},
    {16, 18, false},
    {16, 18, true},
    {16, 20, false},
    {16, 20, true},
    {16, 22, false},
    {16, 22, true},
    {16, 24, false},
    {16, 24, true},
    {16, 26, false},
    {16, 26, true},
    {16, 28, false},
    {16, 28, true},
    {16, 30, false},
    {16, 30, true},
    {32, 8, false},
    {32, 12, false},
    {32, 12, true},
    {32, 15, false},
    {32, 15, true},
    {32, 16, false},
    {32, 16, true},
    {32, 20, false},
    {32, 22, false},
    {32, 22, true},
    {32, 24, false},
    {32, 26, true},
    {32, 28, false},
    {32, 29, true},
    {32, 30, false},
    {32, 32, false},
};
constexpr bool desc_from_qp(int G, int R, bool bin, int qpm) {
  if (qpm != 0) return false;
  for (const DescPick &d : kDescFromQp)
    if (d.G == G && d.R == R && d.bin == bin) return true;
  return false;
}
// Per (tile, boundary input): the plain row order of the biased cell loop
// (the diagonal add after the row) instead of one row ahead, where it measured
// >= 0.5% faster (profiles/r02b_variant_calibration.jsonl).
constexpr DescPick kRowPlain[] = {
    {8, 20, false}, {8, 20, true}, {8, 22, false}, {8, 24, false}, {8, 28, false}, {8, 28, true},
    {8, 32, true}, {16, 20, false}, {16, 20, true}, {16, 22, false}, {16, 24, false}, {16, 28, false},
    {16, 28, true}, {32, 8, true}, {32, 15, false}, {32, 16, false}, {32, 16, true}, {32, 18, true},
    {32, 22, false}, {32, 24, false}, {32, 26, true}, {32, 28, false}, {32, 29, false}, {32, 30, false},
};
constexpr bool row_ahead(int G, int R, bool bin, int qpm) {
  if (qpm != 0) return true;
  for (const DescPick &d : kRowPlain)
    if (d.G == G && d.R == R && d.bin == bin) return false;
  return true;
}

struct TileEntry {
  int G, R, qpm, nt, smem;
  PassFn fn0, fn1;   // pass 0 / passes > 0 (boundary input)
  int ctas;
  PassFn fnw;        // cross-pass wavefront (all passes in one launch), or null
  int ctasw;         // resident CTAs per SM of fnw (its grid must be fully resident)
  int lat;           // 1: latency tile (256 threads, one CTA per SM), for critical-path-bound launches
};

#define SW_TILE_NTU(G_, R_, M_, NT_, U_)                                                          \
  {G_, R_, M_, NT_, smem_of<R_, G_, M_>(),                                                      \
   sw16_pass_kernel<R_, G_, false, M_, NT_, U_, false, desc_from_qp(G_, R_, false, M_),          \
                    row_ahead(G_, R_, false, M_)>,                                              \
   sw16_pass_kernel<R_, G_, true, M_, NT_, U_, false, desc_from_qp(G_, R_, true, M_),            \
                    row_ahead(G_, R_, true, M_)>, 0, nullptr, 0, 0}
// latency tiles (single query): small R, 256 threads, launched
// with one CTA per SM, for passes bounded by one long item's critical path
#define SW_TILE_LAT(G_, R_)                                                                    \
  {G_, R_, 0, 256, smem_of<R_, G_, 0>(), sw16_pass_kernel<R_, G_, false, 0, 256, SW_UNROLL>, \
   sw16_pass_kernel<R_, G_, true, 0, 256, SW_UNROLL>, 0, nullptr, 0, 1}
// tiles that also have a wavefront kernel (single-query mode)
#define SW_TILE_W(G_, R_)                                                                       \
  {G_, R_, 0, 512, smem_of<R_, G_, 0>(),                                                        \
   sw16_pass_kernel<R_, G_, false, 0, 512, SW_UNROLL, false, desc_from_qp(G_, R_, false, 0),     \
                    row_ahead(G_, R_, false, 0)>,                                               \
   sw16_pass_kernel<R_, G_, true, 0, 512, SW_UNROLL, false, desc_from_qp(G_, R_, true, 0),       \
                    row_ahead(G_, R_, true, 0)>, 0,                                             \
   sw16_pass_kernel<R_, G_, true, 0, 512, SW_UNROLL, true>, 0, 0}
#ifndef SW_UNROLL
#define SW_UNROLL 4   // columns per unrolled block = lane G-1's prefetch distance
#endif
#define SW_TILE_NT(G_, R_, M_, NT_) SW_TILE_NTU(G_, R_, M_, NT_, SW_UNROLL)
#define SW_TILE(G_, R_, M_) SW_TILE_NT(G_, R_, M_, 512)
#define SW_TILES_COMMON(M_)                                                                   \
  SW_TILE(8, 8, M_), SW_TILE(8, 12, M_), SW_TILE(8, 16, M_), SW_TILE(8, 18, M_),              \
  SW_TILE(8, 20, M_), SW_TILE(8, 22, M_), SW_TILE(8, 24, M_), SW_TILE(8, 26, M_),             \
  SW_TILE(8, 28, M_), SW_TILE(8, 29, M_), SW_TILE(8, 30, M_), SW_TILE(8, 32, M_),             \
  SW_TILE(16, 8, M_), SW_TILE(16, 12, M_), SW_TILE(16, 18, M_),                               \
  SW_TILE(16, 20, M_), SW_TILE(16, 22, M_), SW_TILE(16, 24, M_), SW_TILE(16, 26, M_),         \
  SW_TILE(16, 28, M_), SW_TILE(16, 30, M_),                                                   \
  SW_TILE(32, 12, M_), SW_TILE(32, 15, M_),                                                   \
  SW_TILE(32, 18, M_), SW_TILE(32, 20, M_), SW_TILE(32, 22, M_), SW_TILE(32, 24, M_),         \
  SW_TILE(32, 26, M_), SW_TILE(32, 28, M_), SW_TILE(32, 30, M_)
TileEntry g_tiles[] = {
    SW_TILES_COMMON(0), SW_TILE_W(16, 16), SW_TILE_W(16, 29), SW_TILE_W(16, 32), SW_TILE_W(32, 8),
    SW_TILE_W(32, 16), SW_TILE_W(32, 29), SW_TILE_W(32, 32),
    SW_TILES_COMMON(3), SW_TILE(16, 16, 3), SW_TILE(16, 29, 3), SW_TILE(16, 32, 3), SW_TILE(32, 8, 3),
    SW_TILE(32, 16, 3), SW_TILE(32, 29, 3), SW_TILE(32, 32, 3),
    SW_TILE_LAT(32, 3), SW_TILE_LAT(32, 4), SW_TILE_LAT(32, 5), SW_TILE_LAT(32, 6), SW_TILE_LAT(32, 8),
    SW_TILE_LAT(16, 9)
#if SW_ARITH >= 1
    // score-profile tiles (NEXT-1): R registers of row-letter offsets cap R
    , SW_TILE(8, 8, 1), SW_TILE(8, 12, 1), SW_TILE(8, 16, 1), SW_TILE(8, 20, 1),
    SW_TILE(16, 8, 1), SW_TILE(16, 12, 1), SW_TILE(16, 16, 1), SW_TILE(16, 20, 1),
    SW_TILE(32, 8, 1), SW_TILE(32, 12, 1), SW_TILE(32, 16, 1), SW_TILE(32, 20, 1)
#endif
};
#undef SW_TILES_COMMON
#undef SW_TILE_W
#undef SW_TILE
#undef SW_TILE_NT
#undef SW_TILE_NTU
#undef SW_TILE_LAT
constexpr int kNumTiles = sizeof(g_tiles) / sizeof(g_tiles[0]);

// Measured full-row throughput (GCUPS) of each tile's pass kernel on one
// B200, biased-unsigned arithmetic, configs[1] at FULL size, in the
// descriptor-address form kDescFromQp picks (round 2, tools/calibrate_tiles.py
// 1.0 under both forms, profiles/r02b_descaddr_calibration.jsonl,
// tools/descaddr_table.py) and the row order kRowPlain picks (the same tool
// under SW_ROWAHEAD=1 / =0 builds, profiles/r02b_variant_calibration.jsonl);
// round 1's table came from a 0.3-scale database and ran 2-5% lower: eff0 =
// first pass (query of G*R), eff1 = a pass reading the previous pass's
// boundary (2*G*R minus G*R).  The tile choice predicts time
// ~ G*R * (1/eff0 + (P-1)/eff1).
struct TileEff { int G, R; float eff0, eff1; };
const TileEff kTileEff[] = {
    {8, 8, 4411.0f, 3628.2f},
    {8, 12, 5202.2f, 4507.4f},
    {8, 16, 5541.1f, 5106.0f},
    {8, 18, 5726.3f, 5238.0f},
    {8, 20, 5804.8f, 5466.5f},
    {8, 22, 5843.1f, 5553.7f},
    {8, 24, 5892.6f, 5561.9f},
    {8, 26, 5919.6f, 5690.1f},
    {8, 28, 5958.2f, 5760.4f},
    {8, 29, 5967.1f, 5699.0f},
    {8, 30, 6021.9f, 5760.6f},
    {8, 32, 5953.8f, 5709.2f},
    {16, 8, 4463.2f, 3861.8f},
    {16, 12, 5214.1f, 4665.8f},
    {16, 16, 5540.1f, 5174.5f},
    {16, 18, 5744.9f, 5308.0f},
    {16, 20, 5806.9f, 5480.4f},
    {16, 22, 5844.3f, 5566.4f},
    {16, 24, 5885.6f, 5563.7f},
    {16, 26, 5915.7f, 5692.7f},
    {16, 28, 5953.1f, 5764.5f},
    {16, 29, 5968.5f, 5674.4f},
    {16, 30, 6022.5f, 5759.0f},
    {16, 32, 5968.2f, 5684.4f},
    {32, 8, 4575.3f, 3969.8f},
    {32, 12, 5296.1f, 4816.8f},
    {32, 15, 5468.5f, 5072.6f},
    {32, 16, 5582.6f, 5170.8f},
    {32, 18, 5628.5f, 5265.4f},
    {32, 20, 5800.9f, 5405.9f},
    {32, 22, 5804.2f, 5542.8f},
    {32, 24, 5912.1f, 5592.2f},
    {32, 26, 5773.9f, 5672.4f},
    {32, 28, 5817.2f, 5631.1f},
    {32, 29, 5888.3f, 5738.4f},
    {32, 30, 5894.1f, 5650.3f},
    {32, 32, 6004.0f, 5672.6f},
};

// Latency tiles (EARLY + LROWS, 256 threads, one CTA per SM;
// tools/lat_calibrate.py, profiles/r02b_lat_calibration.jsonl): SM cycles
// per column step of a group running alone (one 12,000-residue sequence) and
// bulk GCUPS (configs[1] at full size, one pass, solo items off).
struct LatEff { int G, R; float step, bulk; };
const LatEff kLatEff[] = {
    {32, 3, 115.5f, 2432.3f},
    {32, 4, 136.5f, 2933.0f},
    {32, 5, 150.3f, 3066.8f},
    {32, 6, 168.6f, 3354.4f},
    {32, 8, 199.8f, 3723.9f},
    {16, 9, 211.8f, 3839.1f},
};

TileEff tile_eff(int G, int R) {
  for (const TileEff &e : kTileEff)
    if (e.G == G && e.R == R) return e;
  return TileEff{G, R, 4000.f, 3500.f};   // uncalibrated tile: pessimistic
}

int64_t g_launches = 0;   // kernels launched by this library (sw_launch_count)

int grid_for(int64_t total, int threads) {
  int64_t g = (total + threads - 1) / threads;
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace

int64_t launch_count() { return g_launches; }
int num_tiles() { return kNumTiles; }
TileInfo tile(int i) {
  const TileEff e = tile_eff(g_tiles[i].G, g_tiles[i].R);
  TileInfo t{g_tiles[i].G, g_tiles[i].R, g_tiles[i].smem, g_tiles[i].qpm, e.eff0, e.eff1, g_tiles[i].lat, 0.f};
  if (t.lat)
    for (const LatEff &l : kLatEff)
      if (l.G == t.G && l.R == t.R) {
        t.eff0 = t.eff1 = l.bulk;
        t.step = l.step;
      }
  return t;
}
int find_tile_mode(int G, int R, int qpm, int lat) {
  for (int i = 0; i < kNumTiles; ++i)
    if (g_tiles[i].G == G && g_tiles[i].R == R && g_tiles[i].qpm == qpm && g_tiles[i].lat == lat) return i;
  return -1;
}
int find_tile(int G, int R) { return find_tile_mode(G, R, 0); }
int tile_ctas_per_sm(int i) { return g_tiles[i].ctas; }
int tile_threads(int i) { return g_tiles[i].nt; }

cudaError_t init_kernels() {
  for (int i = 0; i < kNumTiles; ++i) {
    for (PassFn fn : {g_tiles[i].fn0, g_tiles[i].fn1, g_tiles[i].fnw}) {
      if (!fn) continue;
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, g_tiles[i].smem);
      if (e != cudaSuccess) return e;
    }
    int n0 = 0, n1 = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n0, g_tiles[i].fn0, g_tiles[i].nt, g_tiles[i].smem);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n1, g_tiles[i].fn1, g_tiles[i].nt, g_tiles[i].smem);
    if (e != cudaSuccess) return e;
    g_tiles[i].ctas = n0 < n1 ? n0 : n1;
    if (g_tiles[i].fnw) {
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_tiles[i].ctasw, g_tiles[i].fnw, g_tiles[i].nt,
                                                        g_tiles[i].smem);
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

size_t qp_bytes(int G, int R, int P, int qpm) {
  return qpm == 1 ? (size_t)kSPBytes : (size_t)P * kNL * qp_letter_bytes(G, R);
}

cudaError_t launch_qp_build(const uint8_t *d_query, int m, const uint8_t *d_query2, int m2, const int8_t *d_matrix,
                            int G, int R, int P, uint8_t *d_qp, uint4 *d_desc, int32_t *d_qp32, int32_t *d_qp32b,
                            int goe, int ge, cudaStream_t st, int sp, const SearchInit &init) {
  const int mm = d_query2 ? (m > m2 ? m : m2) : m;
  const int64_t total = (sp ? (int64_t)kSPBytes / 4 : (int64_t)P * kNL * (qp_letter_bytes(G, R) / 4)) +
                        kNL * kNL + (int64_t)kNL * mm;
  const int64_t zero = std::max<int64_t>(std::max<int64_t>(init.count, init.nitems) / 16, init.nfc) + 1;
  ++g_launches;
  qp_build_kernel<<<grid_for(std::max(total, zero), 256), 256, 0, st>>>(
      d_query, m, d_query2, m2, d_matrix, G, R, P, reinterpret_cast<uint32_t *>(d_qp), d_desc, d_qp32, d_qp32b, goe,
      ge, sp, init);
  return cudaGetLastError();
}

bool tile_has_wave(int i) { return g_tiles[i].fnw != nullptr && g_tiles[i].ctasw > 0; }
int tile_wave_ctas_per_sm(int i) { return g_tiles[i].ctasw; }

cudaError_t launch_sw16_pass(int ti, int grid, const SW16Params &p, cudaStream_t st) {
  PassFn fn = p.npass > 0 ? g_tiles[ti].fnw : (p.bnd_in ? g_tiles[ti].fn1 : g_tiles[ti].fn0);
  if (!fn) return cudaErrorInvalidValue;
  ++g_launches;
  fn<<<grid, g_tiles[ti].nt, g_tiles[ti].smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_sw16_gather(const int64_t *endcol, int64_t count, const uint32_t *sc_out, int32_t *scores,
                               uint8_t *flagged, int32_t *scores2, uint8_t *flagged2, int pass, int thresh,
                               cudaStream_t st, const int32_t *seq_idx, const int32_t *item_of,
                               uint8_t *item_hot, int32_t *list, int *nlist, int32_t *list2, int *nlist2,
                               int want, bool detect) {
  if (count <= 0) return cudaSuccess;
  if (detect) ++g_launches;
  if (detect)
    sw16_detect_kernel<<<grid_for(count, 256), 256, 0, st>>>(endcol, count, sc_out, flagged, flagged2,
                                                            scores2 != nullptr, pass, thresh, seq_idx, item_of,
                                                            item_hot);
  ++g_launches;
  sw16_update_kernel<<<grid_for(count, 256), 256, 0, st>>>(endcol, count, sc_out, scores, flagged, scores2,
                                                            flagged2, pass, seq_idx, item_of, item_hot, list,
                                                            nlist, list2, nlist2, want);
  return cudaGetLastError();
}

cudaError_t launch_item_skip(const Item *items, int nitems, const int32_t *slots, const int64_t *offs,
                             const uint8_t *flagged, int32_t *skip, cudaStream_t st) {
  if (nitems < 1) return cudaSuccess;
  ++g_launches;
  item_skip_kernel<<<grid_for(nitems, 256), 256, 0, st>>>(items, nitems, slots, offs, flagged, skip);
  return cudaGetLastError();
}

cudaError_t launch_flag_compact(const uint8_t *flagged, int64_t count, int32_t *list, int *n, int want,
                                cudaStream_t st) {
  ++g_launches;
  flag_compact_kernel<<<grid_for(count, 256), 256, 0, st>>>(flagged, count, list, n, want);
  return cudaGetLastError();
}

cudaError_t launch_sw32(int grid, const SW32Params &p, cudaStream_t st) {
  constexpr int smem = kNL * (kSW32Rows / 4) * 32 * 16;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(sw32_kernel<kSW32Rows>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  ++g_launches;
  sw32_kernel<kSW32Rows><<<grid, kSW32Threads, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_make_keys(const int32_t *scores, const int64_t *index, int64_t n, uint64_t *keys,
                             int64_t npad, cudaStream_t st) {
  ++g_launches;
  make_keys_kernel<<<grid_for(npad, 256), 256, 0, st>>>(scores, index, n, keys, npad);
  return cudaGetLastError();
}

cudaError_t launch_bitonic_sort_desc(uint64_t *keys, int64_t npow2, cudaStream_t st) {
  for (int64_t size = 2; size <= npow2; size <<= 1) {
    int64_t stride = size >> 1;
    for (; stride > 1024; stride >>= 1) {
      ++g_launches;
      bitonic_step_kernel<<<grid_for(npow2 / 2, 256), 256, 0, st>>>(keys, npow2, size, stride);
    }
    if (npow2 >= 2048) {
      ++g_launches;
      bitonic_local_kernel<<<(unsigned)(npow2 / 2048), 1024, 0, st>>>(keys, size, stride);
    } else {
      for (; stride > 0; stride >>= 1) {
        ++g_launches;
        bitonic_step_kernel<<<grid_for(npow2 / 2, 256), 256, 0, st>>>(keys, npow2, size, stride);
      }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_block_topk(const int32_t *scores, const int64_t *index, const uint64_t *keys_in, int64_t n,
                              int k, uint64_t *out, int blocks, cudaStream_t st) {
  ++g_launches;
  block_topk_kernel<<<blocks, 1024, 0, st>>>(scores, index, keys_in, n, k, out);
  return cudaGetLastError();
}

cudaError_t launch_scatter_scores(const int32_t *src, const int64_t *index, int64_t n, int32_t *dst,
                                  int64_t dst_count, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  ++g_launches;
  scatter_scores_kernel<<<grid_for((n + 3) / 4, 256), 256, 0, st>>>(src, index, n, dst, dst_count);
  return cudaGetLastError();
}

size_t rows_smem_bytes(int ncq) {
  return (size_t)kRowsHeadBytes + (size_t)kRowsWarps * kNL * kRowsLS + (size_t)(kRowsWarps - 1) * kRowsRing * 16 +
         (size_t)(kRowsWarps - 1) * 2 * (kRowsRing / kRowsBatch) * 8 + (2 * kRowsWarps + 4) * sizeof(int) +
         (size_t)((ncq + 15) & ~15);
}

cudaError_t launch_sw16_rows(int grid, const RowsParams &p, cudaStream_t st) {
  const size_t smem = rows_smem_bytes(p.ncq);
  cudaError_t e = cudaFuncSetAttribute(sw16_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  ++g_launches;
  sw16_rows_kernel<<<grid, kRowsWarps * 32, smem, st>>>(p);
  return cudaGetLastError();
}


cudaError_t launch_expand_columns(const uint16_t *in, int64_t n, uint32_t *out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  ++g_launches;
  expand_columns_kernel<<<grid_for((n + 3) / 4, 256), 256, 0, st>>>(in, n, out);
  return cudaGetLastError();
}

cudaError_t launch_stage_copy(const void *host_src_dev, void *dst, size_t bytes, cudaStream_t st) {
  const int n = (int)((bytes + 3) / 4);
  if (n <= 0) return cudaSuccess;
  ++g_launches;
  stage_copy_kernel<<<std::min(8, (n + 255) / 256), 256, 0, st>>>(reinterpret_cast<const uint32_t *>(host_src_dev),
                                                                  reinterpret_cast<uint32_t *>(dst), n);
  return cudaGetLastError();
}

size_t radix_topk_scratch_bytes() { return sizeof(SelState) + 256 * sizeof(unsigned) + 16; }

cudaError_t launch_radix_topk(const int32_t *scores, const int64_t *index, int64_t n, int64_t k, uint64_t *out,
                              void *scratch, cudaStream_t st) {
  SelState *ss = reinterpret_cast<SelState *>(scratch);
  unsigned *hist = reinterpret_cast<unsigned *>(reinterpret_cast<char *>(scratch) + sizeof(SelState));
  unsigned *cnt = hist + 256;
  SelState init{0ull, 0ull, (long long)k, 0};
  cudaError_t e = cudaMemcpyAsync(ss, &init, sizeof(SelState), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(hist, 0, 257 * sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  const int hg = (int)std::min<int64_t>((n + 511) / 512, 148 * 4);
  for (int shift = 56; shift >= 0; shift -= 8) {
    ++g_launches;
    radix_hist_kernel<<<hg, 512, 0, st>>>(scores, index, n, ss, shift, hist);
    ++g_launches;
    radix_select_kernel<<<1, 256, 0, st>>>(ss, hist, shift);
  }
  ++g_launches;
  radix_gather_kernel<<<grid_for(n, 256), 256, 0, st>>>(scores, index, n, ss, out, cnt);
  if (k <= 4096) {
    int np2 = 1;
    while (np2 < k) np2 <<= 1;
    ++g_launches;
    block_sort_desc_kernel<<<1, 1024, 0, st>>>(out, (int)k, np2);
    return cudaGetLastError();
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // k > 4096: the caller sorts out[0, k) padded to a power of two
  return cudaSuccess;
}

cudaError_t launch_decode_keys(const uint64_t *keys, int64_t k, int64_t *idx, int32_t *score, cudaStream_t st) {
  ++g_launches;
  decode_keys_kernel<<<grid_for(k, 256), 256, 0, st>>>(keys, k, idx, score);
  return cudaGetLastError();
}

}  // namespace swdb
