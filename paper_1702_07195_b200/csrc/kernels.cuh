// Kernel launch interface (host side of kernels.cu), used by api.cu.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "swdb_internal.h"

// SW_ARITH selects the 16x2 cell arithmetic of the pass kernel:
//   2 (default): "biased unsigned" form.  Every 16-bit value is stored as
//     x + kBias16 with kBias16 = 32768 in UNSIGNED halves [32768, 65535], so
//     the diagonal add H_diag + SM runs as one 32-bit add on the FMA pipe (no
//     carry between the halves while exact) and Eq. 1 is one VIMNMX3.U16x2 on
//     the ALU pipe: 4.5 ALU + 2 FMA instructions per pair of cells, exact
//     below 65536 - smax - kBias16 (= 32757 for BLOSUM62), the same range as
//     the relu form; above, flagged for 32-bit re-scoring.
//   1: the same with SIGNED halves and kBias16 = 16384 (round 1): exact only
//     below 32768 - smax - 16384 (= 16373).
//   0: the plain relu form, 5.5 DPX per pair of cells, exact below 32768 - smax.
#ifndef SW_ARITH
#define SW_ARITH 2
#endif

namespace swdb {

constexpr int kArith = SW_ARITH;
constexpr bool kBiased = kArith >= 1;               // the diagonal add on the FMA pipe, Eq. 1 one VIMNMX3
constexpr int kBias16 = kArith == 2 ? 32768 : (kArith == 1 ? 16384 : 0);   // stored = value + kBias16 (per half)
constexpr int kDummy16 = kArith == 1 ? -16384 : -32768;   // separator / phantom-row score (-kBias16 when biased)
constexpr int kHalfTop = kArith == 2 ? 65536 : 32768;     // stored halves are < kHalfTop

// Query-profile slice layout of the s16x2 pass kernel (one pass, one letter),
// for a group of G lanes with R rows each:
//   R/4 full chunks [chunk][lane t][4 rows x 4 B] (LDS.128, lane t at t*16:
//   each quarter-warp hits 8 distinct 16-B bank groups), then, when R % 4 is
//   1 or 2, a tail block of W = 4 or 8 B per lane [copy][lane t][W] read with
//   LDS.32 / LDS.64 at lane stride W: contiguous, so conflict-free.  The block
//   holds ncopy copies so that the 32/G groups of a warp read distinct banks
//   (group g reads copy g % ncopy).  R % 4 == 3: the tail is a full-width
//   chunk (LDS.128).  Every letter's slice is a multiple of 128 B.
#ifndef SW_QPTAIL
#define SW_QPTAIL 0   // 1: narrow conflict-free tail block (measured slower); 0: full-width LDS.128 tail chunk
#endif
__host__ __device__ constexpr int qp_tail_w(int R) {
  return R % 4 == 0 ? 0 : ((R % 4 == 3 || !SW_QPTAIL) ? 16 : (R % 4 == 1 ? 4 : 8));
}
__host__ __device__ constexpr int qp_full_chunks(int R) { return qp_tail_w(R) == 16 ? R / 4 + 1 : R / 4; }
__host__ __device__ constexpr int qp_tail_ncopy(int G, int R) {
  return (qp_tail_w(R) == 4 || qp_tail_w(R) == 8) ? (G * qp_tail_w(R) >= 128 ? 1 : 128 / (G * qp_tail_w(R))) : 1;
}
__host__ __device__ constexpr int qp_tail_bytes(int G, int R) {
  return (qp_tail_w(R) == 4 || qp_tail_w(R) == 8) ? qp_tail_ncopy(G, R) * G * qp_tail_w(R) : 0;
}
__host__ __device__ constexpr int qp_letter_bytes(int G, int R) { return qp_full_chunks(R) * G * 16 + qp_tail_bytes(G, R); }

// Score profile (QPM 1): per letter pair (cA, cB) of the stream alphabet, a
// vector over the query letters c < kSPL (24 residue codes + one phantom-row
// letter) of SM(c, cB) * 65536 + SM(c, cA): 676 x 25 words.
constexpr int kSPL = 25;
constexpr int kSPBytes = 26 * 26 * kSPL * 4;
static_assert(kSPBytes % 16 == 0, "bulk copy size");

struct SW16Params {
  const uint32_t *stream;   // column words (descriptor byte offsets)
  const Item *items;
  int num_items;
  int *counter;             // atomic item cursor for this pass (zeroed)
  const uint4 *qp;          // int16 query profile, all passes: [P][kNL][K8][G][8]
  const uint4 *desc;        // descriptor table: [kNL*kNL] uint4
  const uint2 *bnd_in;      // boundary (H,F) per column from the previous pass, or null
  uint2 *bnd_out;           // boundary for the next pass, or null
  uint2 *dummy;             // one 16-B scratch slot per launched thread (idle-lane stores)
  const uint32_t *nul_stream;  // >= 16 NUL column words (groups without items)
  const uint2 *zero_bnd;       // >= 16 zero boundary columns
  int64_t col_lo, col_hi;      // valid column range of stream / bnd / sc_out (SW_DEBUG checks)
  uint32_t *sc_out;         // per column: score chain value at the last lane
  int pass;
  int thresh;               // 32768 - max(1, smax)
  uint32_t zero;            // 0 (passed in so ptxas keeps it in a register)
  uint32_t one;             // 1 (passed in: keeps 32-bit adds on the FMA pipe as IMAD)
  // Cross-pass wavefront (one launch runs every pass): npass
  // passes starting at `pass`, item cursors pcounters[npass], per-(pass, item)
  // finished-column counts progress[npass * num_items] (zeroed), and the two
  // boundary buffers (pass p reads bndbuf[(p-1)&1], writes bndbuf[p&1]).  The
  // score chain is carried from pass to pass through sc_out.  npass == 0: off.
  int npass;
  int *pcounters;
  int *progress;
  uint2 *bndbuf[2];
  // Per item: leading columns to skip in this pass (per-pass launches only),
  // or null.  They hold only sequences already flagged in both halves
  // (item_skip_kernel), whose 16-bit results are no longer used.
  const int32_t *skip;
  // QPM 1 (score profile): the query and its length (each lane's row letters)
  const uint8_t *query;
  int m;
  // Latency tiles (EARLY, G = 32): items [*solo_counter, solo_end) are claimed
  // only by warps 0-3 of a CTA (one per SM sub-partition); a warp 4-7 whose
  // partner's first item is one of them claims nothing (null: off).
  int *solo_counter;
  int solo_end;
  // Wavefront launches with fewer units (items x passes) than lane groups: only
  // the first group_limit groups of a CTA (counted across its warps first)
  // claim, so the units spread over all SMs instead of filling the CTAs that
  // reach the cursor first (0: every group claims).
  int group_limit;
};

// Rows mode (long database sequences along the rows, kernels.cu).
constexpr int kRowsR = 8;                           // rows per lane (one 32-lane group per warp)
constexpr int kRowsWarps = 8;                       // warps per CTA = passes in flight per item
constexpr int kRowsRing = 64;                       // shared-memory ring between consecutive warps (columns)
constexpr int kRowsBatch = 8;                       // columns per ring slot (one full / empty mbarrier each)
constexpr int kRowsPublish = 4;                     // columns between producer-count updates
constexpr int kRowsAhead = 4;                       // lane 31's prefetch distance (columns)
constexpr int kRowsLS = (kRowsR / 4) * 32 * 16;     // profile bytes per query letter of a warp
constexpr int kRowsHeadBytes = 26 * 16 + 26 * 26 * 4 + 16;   // descriptors + matrix (+ pad to 16 B)
constexpr int kRowsRows = 32 * kRowsR;              // database rows per pass
struct RowsParams {
  const uint8_t *query;     // device, m codes
  int m;
  int ncq;                  // columns of the query stream: m letters, END, NUL... (multiple of 4)
  const int8_t *matrix;     // device [24][24], matrix[q*24 + d]
  const uint8_t *res;       // plain database, original order
  const int64_t *offs;
  const Item *items;        // the image's items; the long pairs are items 0 .. n_items-1
  const int32_t *slots;
  int n_items;
  int *counter;             // zeroed: next item
  uint4 *wrap;              // per CTA: ncq entries (warp 7 -> warp 0 hand-over)
  const int64_t *endcol;    // the image's END columns (2 * column + half)
  uint32_t *sc_out;         // the image's per-column chain buffer (the gather reads the END columns)
  int goe, ge;
  uint32_t one;
};

struct SW32Params {
  const int32_t *flag_list;
  const int *flag_count;
  int *cursor;
  const uint8_t *res;       // plain database, original order
  const int64_t *offs;
  const int32_t *qp32;      // plain int32 profile [kNL][m] (-2^30 for separator letters)
  int m;                    // query length (rows of qp32)
  int len;                  // rows of this query (<= m; a pair's shorter query); the last pass
                            // runs R/3 or 2R/3 rows per lane when that covers the rest
  int row0;                 // first query row to compute (rows < row0 were exact in 16 bit)
  int passes;               // ceil((m - row0) / (32 * R))
  int neg_goe, neg_ge;      // -(open+extend), -extend  (>= -2^30)
  // row0 > 0: the exact 16-bit boundary (H, F) of row row0-1, per stream column
  // (pass output of the 16-bit kernel, stored + kBias16 per half), located by
  // endcol (2 * END column + half) and read from half `half` (< 0: endcol's own)
  const uint2 *bnd16;
  const int64_t *endcol;
  int half;
  uint2 *scratch;           // per warp: 2 * stride
  int64_t stride;           // >= max_len + 64
  int32_t *scores;          // row0 > 0: holds the exact max over rows < row0 on entry
  int64_t *cells;           // re-scored cells (statistics), may be null
  uint32_t one;             // 1 (keeps the diagonal add on the FMA pipe)
};

struct TileInfo {
  int G, R;
  int smem_bytes;           // dynamic shared memory of the pass kernel
  int qpm;                  // profile mode (see kernels.cu)
  float eff0, eff1;         // measured full-row GCUPS: first pass / boundary-reading pass
  int lat;                  // latency tile (critical-path-bound launches)
  float step;               // latency tile: measured SM cycles per column step of a lone group (0: model)
};

// Number of kernel launches issued by the library since it was loaded.
int64_t launch_count();

// Compiled (G, R) tiles of the s16x2 pass kernel.
int num_tiles();
TileInfo tile(int i);
int find_tile(int G, int R);                // index or -1 (profile mode 0)
int find_tile_mode(int G, int R, int qpm, int lat = 0);  // index or -1
size_t qp_bytes(int G, int R, int P, int qpm);

// Prepares kernel attributes (max dynamic smem).  Returns cudaError_t.
cudaError_t init_kernels();
// Max resident CTAs per SM of tile i's kernel.
int tile_ctas_per_sm(int i);
// Threads per CTA of tile i's kernel.
int tile_threads(int i);

// Per-search zeroing of the re-scoring counters, the flag bytes, the 32-bit
// cell counter and the per-item carry marks (null / 0 = skip), done by the
// profile launch (one launch fewer per search).
struct SearchInit {
  int *fcounters;
  int nfc;
  uint8_t *flagged, *flagged2;
  int64_t count;
  int64_t *cells32;
  uint8_t *item_hot;
  int64_t nitems;
};
// d_query2 != nullptr: query-pair profile (QPM 3) and a second s32 profile.
cudaError_t launch_qp_build(const uint8_t *d_query, int m, const uint8_t *d_query2, int m2, const int8_t *d_matrix,
                            int G, int R, int P, uint8_t *d_qp, uint4 *d_desc, int32_t *d_qp32, int32_t *d_qp32b,
                            int goe, int ge, cudaStream_t st, int sp, const SearchInit &init);
// sp = 1: d_qp receives the score profile (QPM 1) and the descriptors its pair offsets.
// goe = gap open + extend, ge = gap extend (>= 0; the descriptor penalty words clamp at 32767)
cudaError_t launch_sw16_pass(int tile_index, int grid, const SW16Params &p, cudaStream_t st);
// Whether tile i has a cross-pass wavefront kernel (p.npass > 0 launches it).
bool tile_has_wave(int i);
int tile_wave_ctas_per_sm(int i);
// item_of: per original sequence its work item (sequence-pair image), with
// item_hot[items] zeroed per search: the carry propagation of SW_ARITH 2
// (kernels.cu, R7); null for the query-pair image.
cudaError_t launch_sw16_gather(const int64_t *endcol, int64_t count, const uint32_t *sc_out, int32_t *scores,
                               uint8_t *flagged, int32_t *scores2, uint8_t *flagged2, int pass, int thresh,
                               cudaStream_t st, const int32_t *seq_idx, const int32_t *item_of,
                               uint8_t *item_hot, int32_t *list = nullptr, int *nlist = nullptr,
                               int32_t *list2 = nullptr, int *nlist2 = nullptr, int want = 0,
                               bool detect = true);   // false: no score can reach thresh (no flag pass)
// want > 0: the update launch also compacts the sequences with flag byte ==
// want (those first flagged in this pass) into list / list2 (counts nlist /
// nlist2, zeroed by the caller), as launch_flag_compact would.
// thresh: in stored 16-bit units (32768 - smax); scores are stored - kBias16.
// A sequence already flagged is skipped; one flagged in this pass gets
// flagged = pass + 1 and keeps in scores the exact maximum of the earlier passes
// (pass 0: not written) -- the 32-bit kernel owns its score from then on.
// Compacts the indices i with flagged[i] == want (want == 0: any non-zero).
cudaError_t launch_flag_compact(const uint8_t *flagged, int64_t count, int32_t *list, int *n, int want,
                                cudaStream_t st);
// Per item, the leading columns whose sequences are all flagged (both halves);
// skip[i] = min over the halves.
cudaError_t launch_item_skip(const Item *items, int nitems, const int32_t *slots, const int64_t *offs,
                             const uint8_t *flagged, int32_t *skip, cudaStream_t st);
#ifndef SW_S32ROWS
#define SW_S32ROWS 24
#endif
constexpr int kSW32Rows = SW_S32ROWS;  // rows per lane of the 32-bit kernel
constexpr int kSW32Threads = 256;
cudaError_t launch_sw32(int grid, const SW32Params &p, cudaStream_t st);

// 16-bit column words (host image, streamed chunks) -> the pass kernel's
// 32-bit words: out[i] = in[i] for i < n.
cudaError_t launch_expand_columns(const uint16_t *in, int64_t n, uint32_t *out, cudaStream_t st);
// bytes (rounded up to 4) from a pinned, mapped host buffer (its device pointer) to device memory
cudaError_t launch_stage_copy(const void *host_src_dev, void *dst, size_t bytes, cudaStream_t st);


// Sorting stage.
cudaError_t launch_make_keys(const int32_t *scores, const int64_t *index, int64_t n,
                             uint64_t *keys, int64_t npad, cudaStream_t st);
cudaError_t launch_bitonic_sort_desc(uint64_t *keys, int64_t npow2, cudaStream_t st);
// k <= 32: `blocks` blocks of 1024 threads; out[] holds blocks * k keys, each
// block's k best in descending order.
cudaError_t launch_block_topk(const int32_t *scores, const int64_t *index, const uint64_t *keys_in, int64_t n,
                              int k, uint64_t *out, int blocks, cudaStream_t st);
cudaError_t launch_decode_keys(const uint64_t *keys, int64_t k, int64_t *idx, int32_t *score,
                               cudaStream_t st);
size_t rows_smem_bytes(int ncq);   // head + 8 profiles + 7 rings + counters + the query stream
constexpr int kRowsMaxNcq = 8192;  // rows mode needs the query stream in shared memory
cudaError_t launch_sw16_rows(int grid, const RowsParams &p, cudaStream_t st);
// k > 32: radix select (8 digit passes of the 64-bit key) + compaction of the
// k largest keys into out[0, k); sorted descending when k <= 4096 (otherwise
// unsorted: the caller sorts them).  scratch: radix_topk_scratch_bytes().
size_t radix_topk_scratch_bytes();
cudaError_t launch_radix_topk(const int32_t *scores, const int64_t *index, int64_t n, int64_t k, uint64_t *out,
                              void *scratch, cudaStream_t st);
// dst[index[i]] = src[i] for i < n, skipping index < 0 or >= dst_count.
cudaError_t launch_scatter_scores(const int32_t *src, const int64_t *index, int64_t n, int32_t *dst,
                                  int64_t dst_count, cudaStream_t st);

}  // namespace swdb
