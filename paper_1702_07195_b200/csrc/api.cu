// C-ABI of the B200 Smith-Waterman database search (include/swdb.h).
//
// Pipeline per query:
//   sw_db_load  : pre-processing stage -> device-resident stream image
//   sw_search   : query profile build -> P s16x2 pass kernels
//                 -> flag compaction -> exact s32 re-scoring of flagged
//                 sequences -> scores in original order
//   sw_topk     : sorting stage
// All state lives in one process-wide object (one database per process; one
// process per GPU for multi-GPU runs).  No exception crosses the ABI.
#include "../../include/swdb.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "kernels.cuh"
#include "swdb_internal.h"

using namespace swdb;

namespace {

thread_local std::string t_err;

int fail(int code, const std::string &msg) {
  t_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess) {                                                             \
      return fail(_e == cudaErrorMemoryAllocation ? SW_ENOMEM : SW_ECUDA,                \
                  std::string(#expr) + ": " + cudaGetErrorString(_e));                   \
    }                                                                                    \
  } while (0)

template <class T>
struct DevBuf {
  T *p = nullptr;
  size_t n = 0;  // elements
  cudaError_t ensure(size_t want) {
    if (want <= n && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(want, 1) * sizeof(T));
    if (e == cudaSuccess) n = want;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

// A device-resident stream image.
struct Image {
  DevBuf<uint32_t> stream;  // column words (descriptor byte offsets; host image: 16-bit)
  DevBuf<Item> items;
  DevBuf<int64_t> endcol;   // per sequence: 2 * END column + half
  DevBuf<int32_t> slots;    // slot -> original sequence (items' sequences in column order)
  DevBuf<int32_t> item_of;  // original sequence -> work item (sequence-pair image)
  int64_t total_cols = 0;
  int64_t max_item_cols = 0;  // longest work item (columns)
  int num_items = 0;
  // rows mode (sequence-pair image): the leading n_long items hold one long
  // sequence per half; units (item, pass) of the rows kernel
  int n_long = 0;
  int64_t long_min_len = 0;       // shortest long sequence
  int64_t long_max_len = 0;       // longest long sequence
  int64_t long_cols = 0;          // pair-columns of the long items
  int64_t max_item_cols_rest = 0; // longest item after them
  DevBuf<int2> units;
  int n_units = 0;
  std::vector<int32_t> item_ncols;  // host: columns of each item (claim order, descending)
  void release() {
    stream.release(); items.release(); endcol.release(); slots.release(); item_of.release(); units.release();
    item_ncols.clear();
    total_cols = 0;
    max_item_cols = 0;
    num_items = 0;
    n_long = 0;
    n_units = 0;
    long_min_len = long_max_len = long_cols = max_item_cols_rest = 0;
  }
};

struct State {
  bool loaded = false;
  int device = -1;
  int num_sms = 0;
  cudaStream_t stream = nullptr;
  int64_t count = 0, total_res = 0, max_len = 0;
  // img[0]: two sequences per column (one query); img[1]: one sequence per
  // column (query pairs)
  Image img[2];
  int64_t max_cols = 0;
  DevBuf<uint32_t> sc_out;  // per column: score chain value (one pass)
  DevBuf<uint8_t> res;      // plain copy, original order (for s32 re-scoring)
  DevBuf<int64_t> offs;
  // per search
  DevBuf<int32_t> scores;   // internal scores (sw_search)
  DevBuf<int32_t> bscores;  // internal scores (sw_search_batch)
  DevBuf<uint8_t> flagged, flagged2;
  DevBuf<int32_t> flag_list, flag_list2;
  DevBuf<int> fcounters;    // 32-bit re-scoring: (count, cursor) per (pass, query of a pair)
  const uint8_t *res_dev = nullptr;  // residues for s32 re-scoring (device or mapped host)
  DevBuf<int64_t> cells32;
  // per-search inputs in one device buffer: matrix (576 B), query, query 2
  DevBuf<uint8_t> qin;
  const uint8_t *q_d = nullptr, *q2_d = nullptr;
  const int8_t *mat_d = nullptr;
  DevBuf<uint8_t> qp;
  DevBuf<uint4> desc;
  DevBuf<int32_t> qp32, qp32b;
  DevBuf<uint2> bnd;        // 2 * max_cols
  DevBuf<int32_t> skip;     // per item: dead leading columns for the next pass
  DevBuf<uint8_t> item_hot; // per item: a low-half sequence flagged (carry propagation, R7)
  DevBuf<uint2> dummy;      // scratch for idle-lane stores (16-B slot per thread)
  DevBuf<uint32_t> nulcols; // 16 NUL column words
  DevBuf<uint2> zerocols;   // 16 zero boundary columns
  DevBuf<uint2> scratch32;
  DevBuf<uint64_t> keys;
  DevBuf<uint64_t> keys2;
  DevBuf<int64_t> tk_idx;
  DevBuf<int32_t> tk_score;
  int64_t scratch_stride = 0;
  int sw32_grid = 0;
  // last search
  bool has_search = false;
  const int32_t *last_scores = nullptr;
  cudaStream_t last_stream = nullptr;
  int last_G = 0, last_R = 0, last_P = 0, last_mode = 0;
  int64_t last_flags = -1, last_cells32 = -1, last_thresh = 0;
  // forced tile
  int force_G = 0, force_R = 0;
  int wave_mode = 0;        // cross-pass wavefront: 0 auto, 1 always (multi-pass), -1 never
  int lat_mode = 0;         // latency tiles: 0 auto, 1 always, -1 never
  int rows_mode = 0;        // rows mode for the long items: 0 auto, 1 whenever possible, -1 never
  int64_t last_rows = 0;    // long pairs scored in rows mode by the last search
  DevBuf<uint4> rows_wrap;  // rows mode: per CTA one pass of (H, F, chain) (warp 7 -> warp 0)
  DevBuf<int> rows_prog;    // rows mode: item counter
  int prof_mode = 0;        // substitution scores: 0 auto, 1 query profile, 2 score profile
  int last_prof = 1;
  bool last_lat = false;
  bool last_wave = false;
  DevBuf<int> progress;     // wavefront: finished columns per (pass, item)
  // timing events of the last search
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t tk_ev = nullptr;    // end of the last sw_topk_dev (its key scratch is shared)
  // (start, end) of every pass-kernel launch of the last kHist searches (a
  // batch is one), a ring: slot hslot is the last search's (sw_timing_history)
  static constexpr int kHist = 64;
  std::vector<cudaEvent_t> hpev[kHist];
  int hnpev[kHist] = {};
  int hslot = 0;
  int64_t nsearch = 0;
  std::vector<cudaEvent_t> *pevp = &hpev[0];
  int npev = 0;                   // pairs recorded by the last search (or batch)
  bool batch_cont = false;        // search_core continues a batch: keep ev[0] and the pass events
  // ---- streamed (out-of-core) database, SURVEY 8(f) NEXT-3
  struct Chunk {
    int item_begin, item_end;   // items [begin, end)
    int64_t col_begin, col_end; // image columns [begin, end), padding included
    int64_t seq_begin, seq_end; // entries in cseq_idx / cseq_endcol
  };
  bool streamed = false;
  std::vector<Chunk> chunks;
  int64_t chunk_span = 0;       // max columns of a chunk
  uint16_t *h_stream = nullptr; // pinned host image: 16-bit column words (1 B per residue)
  uint8_t *h_res = nullptr;     // pinned, mapped host copy of the residues (s32 re-scoring)
  DevBuf<uint32_t> cbuf[2];     // device chunk buffers (double-buffered), 32-bit column words
  DevBuf<uint16_t> cbuf16[2];
  // chunk k of a search uses buffer (k + buf_parity) & 1; at the end of a
  // search chunk 0 of the next one is copied into the buffer the last chunk
  // did not use (the database does not change between searches), so its copy
  // overlaps the last chunk's passes instead of opening the next search
  int buf_parity = 0;
  bool chunk0_staged = false;   // their compact copies as they arrive over the host link
  DevBuf<int32_t> cseq_idx;     // sequences grouped by chunk
  DevBuf<int64_t> cseq_endcol;  // their END columns (global image columns)
  cudaStream_t copy_st = nullptr;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr};
  // Resident head: the leading (longest) work items stay on
  // the device and run on a second, high-priority compute stream beside the
  // streamed chunks, so a long sequence's chain is hidden by the whole search
  // instead of bounding the one chunk that holds it.
  bool has_head = false;
  Chunk head{};
  DevBuf<uint32_t> head_buf, head_sc;
  DevBuf<uint2> head_bnd;
  cudaStream_t head_st = nullptr;
  cudaEvent_t ev_head = nullptr;

  void release_streamed() {
    if (h_stream) cudaFreeHost(h_stream);
    if (h_res) cudaFreeHost(h_res);
    h_stream = nullptr;
    h_res = nullptr;
    cbuf[0].release(); cbuf[1].release(); cbuf16[0].release(); cbuf16[1].release();
    cseq_idx.release(); cseq_endcol.release();
    for (int k = 0; k < 2; ++k) {
      if (ev_copied[k]) cudaEventDestroy(ev_copied[k]);
      if (ev_free[k]) cudaEventDestroy(ev_free[k]);
      ev_copied[k] = ev_free[k] = nullptr;
    }
    if (copy_st) cudaStreamDestroy(copy_st);
    copy_st = nullptr;
    if (head_st) cudaStreamDestroy(head_st);
    head_st = nullptr;
    if (ev_head) cudaEventDestroy(ev_head);
    ev_head = nullptr;
    head_buf.release(); head_sc.release(); head_bnd.release();
    has_head = false;
    chunks.clear();
    streamed = false;
    buf_parity = 0;
    chunk0_staged = false;
  }

  void release_all() {
    release_streamed();
    img[0].release(); img[1].release();
    sc_out.release(); res.release(); offs.release();
    scores.release(); bscores.release(); flagged.release(); flagged2.release(); flag_list.release();
    flag_list2.release(); fcounters.release(); cells32.release(); progress.release();
    qin.release(); qp.release(); desc.release(); qp32.release();
    qp32b.release(); bnd.release(); skip.release(); item_hot.release();
    rows_wrap.release(); rows_prog.release();
    scratch32.release(); dummy.release(); nulcols.release(); zerocols.release(); keys.release(); keys2.release(); tk_idx.release(); tk_score.release();
    loaded = false;
    has_search = false;
    last_scores = nullptr;
  }
};

State g;
constexpr int kMaxPass = 4096;

bool solo_enabled() {   // SWDB_SOLO=0 turns solo items off (experiments; read per search)
  const char *e = std::getenv("SWDB_SOLO");
  return !(e && e[0] == '0');
}

// The per-search inputs (matrix, query, query 2) cross the host link in ONE
// copy from a pinned staging slot: a copy from pageable memory may wait for
// the stream (the host could not enqueue a search before the previous one
// ends, and every launch latency would be exposed).  Slots are reused round
// robin, each guarded by the event recorded after its copy.  Independent of
// the loaded database (kept across sw_db_load / sw_db_free).
struct Staging {
  static constexpr int kSlots = 4;
  uint8_t *h[kSlots] = {};
  size_t cap[kSlots] = {};
  cudaEvent_t ev[kSlots] = {};
  int next = 0;
};
Staging g_stage;
bool g_kernels_ready = false;

int ensure_device_ready() {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  if (!g_kernels_ready) {
    CUDA_TRY(init_kernels());
    g_kernels_ready = true;
  }
  return SW_OK;
}

// Choose (G, R) for a query of m residues: minimise the predicted time
// G*R * (1/eff0 + (P-1)/eff1) -- rows computed, incl. the phantom rows of the
// last pass, over the tile's measured full-row throughput of a first pass and
// of a boundary-reading pass -- plus a per-pass constant.
// Tile choice: predicted time per database residue of a query of m rows,
//   rows * (1/eff0 + (P-1)/eff1) / balance + P * const,
// eff0/eff1 the measured full-row throughput of the tile (kernels.cu).  A pass
// lasts at least as long as its longest work item, which one group of G lanes
// processes alone (the intra-task part of the kernel); balance = min(1,
// average columns per group / (1.15 * longest item)) charges tiles with many
// small groups for that tail (cfg4: 5-35 k residue sequences).
int choose_tile(int m, int qpm, const Image &I, bool wave_only = false) {
  if (g.force_G) {
    int ti = find_tile_mode(g.force_G, g.force_R, qpm, 0);
    if (ti >= 0) return ti;
  }
  double best = 1e300;
  int bi = -1;
  for (int i = 0; i < num_tiles(); ++i) {
    const TileInfo ti = tile(i);
    if (ti.qpm != qpm || ti.lat || tile_ctas_per_sm(i) < 1 || (wave_only && !tile_has_wave(i))) continue;
    const int rows = ti.G * ti.R;
    const int P = (m + rows - 1) / rows;
    const double groups = (double)g.num_sms * tile_ctas_per_sm(i) * tile_threads(i) / ti.G;
    const double avg_cols = (double)I.total_cols / groups;
    // (the wavefront overlaps the passes of the longest item: no balance term)
    const double balance = (I.max_item_cols > 0 && !wave_only)
                               ? std::min(1.0, avg_cols / (1.15 * (double)I.max_item_cols)) : 1.0;
    const double cost = (double)rows * (1.0 / ti.eff0 + (P - 1) / ti.eff1) / balance + P * 0.002;
    if (cost < best - 1e-12) {
      best = cost;
      bi = i;
    }
  }
  return bi;
}

// Time model of a pass launch (profiles/r02_lat_calibration.jsonl):
//   bulk  = cells computed (phantom rows included) / the tile's throughput,
//   chain = (longest item + G) columns x the per-column step latency of one
//           group, c0 + c1 * R SM cycles (measured on one 12,000-residue
//           sequence: one warp issues its column's instructions back to back,
//           ~14 cycles per row plus ~145 per column for the lane-to-lane
//           hand-over, the descriptor -> profile load chain and the stores);
// a pass lasts about max(bulk, chain).  Latency tiles (small R, one
// 256-thread CTA per SM) shorten the chain at lower throughput.
constexpr double kStepC0 = 145.0, kStepC1 = 14.0;
// rows kernel (profiles/r02_rows_mode.jsonl, traces): ~850 cycles per column
// step with 8 warps per SM, ~44 steps between consecutive passes
constexpr double kRowsStep = 850.0, kRowsLag = 44.0;
constexpr bool kRowsAuto = false;

// What the pass time model sees of a database (or of one streamed chunk).
struct Shape {
  int64_t total_cols, max_item_cols;
};
Shape shape_of(const Image &I) { return Shape{I.total_cols, I.max_item_cols}; }

double pass_time_model(const TileInfo &T, int m, Shape I, bool lat) {
  const int rows = T.G * T.R;
  const int P = (m + rows - 1) / rows;
  const double f = 1.9e9;   // SM cycles per second
  const double cells = (double)rows * P * 2.0 * (double)I.total_cols;
  // latency tiles: their own measured bulk rate (eff0) and step (kernels.cu kLatEff)
  (void)lat;
  const double bulk = cells / (T.eff0 * 1e9);
  const double step = T.step > 0.f ? (double)T.step : kStepC0 + kStepC1 * T.R;
  const double chain = (double)P * ((double)I.max_item_cols + T.G) * step / f;
  return std::max(bulk, chain);
}

// The latency tile with the smallest modelled time, if it beats the throughput
// tile `ti` by 10% (or the best latency tile when forced); -1 if none.
// single_pass: only latency tiles that hold the query in one pass (rows mode
// runs beside a single pass of the pass kernel)
int choose_lat_tile(int m, Shape I, int ti, bool forced, bool single_pass = false) {
  const double base = pass_time_model(tile(ti), m, I, false);
  double best = forced ? 1e300 : 0.9 * base;
  int bi = -1;
  for (int i = 0; i < num_tiles(); ++i) {
    const TileInfo t = tile(i);
    if (!t.lat || t.qpm != 0 || tile_ctas_per_sm(i) < 1) continue;
    if (single_pass && t.G * t.R < m) continue;
    const double c = pass_time_model(t, m, I, true);
    if (c < best) {
      best = c;
      bi = i;
    }
  }
  return bi;
}

// QP/SP switch by query length (the paper's best profile
// depended on the query length and the lane width).  Measured on B200 in the
// real pass kernel over configs[3]'s 20 query lengths: the query profile is
// faster at every length (profiles/r02_qp_sp_crossover.jsonl), so the switch
// point lies beyond the longest query measured.
constexpr int kSPMinLen = INT_MAX;
bool sp_wins(int m) { return m >= kSPMinLen; }

int validate_query(const uint8_t *query, int32_t qlen, const int8_t *matrix, int32_t gap_open,
                   int32_t gap_extend) {
  if (!query || !matrix) return fail(SW_EINVAL, "query or matrix is NULL");
  if (qlen < 1) return fail(SW_EINVAL, "qlen must be >= 1");
  if (gap_open < 0 || gap_extend < 0) return fail(SW_EINVAL, "gap penalties must be >= 0");
  if ((int64_t)gap_open + gap_extend >= (int64_t(1) << 30))
    return fail(SW_EINVAL, "gap_open + gap_extend must be < 2^30");
  for (int32_t i = 0; i < qlen; ++i)
    if (query[i] >= kAlpha) return fail(SW_EINVAL, "query code >= 24 at position " + std::to_string(i));
  int smax = 0;
  for (int i = 0; i < kAlpha * kAlpha; ++i) smax = std::max(smax, std::abs((int)matrix[i]));
  if ((int64_t)smax * std::min<int64_t>(qlen, std::max<int64_t>(g.max_len, 1)) >= (int64_t(1) << 30))
    return fail(SW_EINVAL, "max|matrix| * min(qlen, longest sequence) must be < 2^30");
  return SW_OK;
}

// One query (q2 == nullptr) against the database image of sequence pairs, or
// a query pair (q, q2) against the image of single sequences.  Stream-ordered
// on st; scores (and scores2) are device arrays in original database order.
int search_core(const uint8_t *q, int32_t m, const uint8_t *q2, int32_t m2, const int8_t *matrix,
                int32_t gap_open, int32_t gap_extend, int32_t *d_scores, int32_t *d_scores2, cudaStream_t st) {
  int rc = validate_query(q, m, matrix, gap_open, gap_extend);
  if (rc) return rc;
  if (q2 && (rc = validate_query(q2, m2, matrix, gap_open, gap_extend))) return rc;
  int dev = -1;
  CUDA_TRY(cudaGetDevice(&dev));
  if (dev != g.device) return fail(SW_EINVAL, "current CUDA device differs from the one sw_db_load used");

  const bool pair = q2 != nullptr;
  if (pair && g.streamed) return fail(SW_EINVAL, "query pairs / batch search need a resident database");
  // Substitution scores: the query profile
  // (QPM 0) or the score profile (QPM 1, sw_set_profile).  Auto: the query
  // profile at every query length (the switch point measured on configs[3]'s
  // 20 lengths, profiles/r02_qp_sp_crossover.jsonl).
  const bool use_sp = !pair && (g.prof_mode == 2 || (g.prof_mode == 0 && sp_wins(pair ? std::max(m, m2) : m)));
  const int mode = pair ? 3 : (use_sp ? 1 : 0);
  const Image &I0 = g.img[pair ? 1 : 0];
  const int mm = pair ? std::max(m, m2) : m;
  // Rows mode: the long pairs (the image's leading items) are
  // scored with the sequence along the rows by sw16_rows_kernel, the pass
  // kernel claims the other items only.  Only on request (sw_set_rows_mode(1)):
  // measured slower than the ordinary path on every database tried
  // (profiles/r02_rows_mode.jsonl) -- the cross-SM progress hand-over between
  // consecutive passes costs more than the shorter chain saves.  Single-pass
  // resident single-query searches without the wavefront.
  const bool rows_possible = !pair && !g.streamed && I0.n_long > 0 && I0.n_units > 0 && g.rows_mode >= 0 &&
                             ((m + 2 + 3) & ~3) <= kRowsMaxNcq;
  bool rows_cand = rows_possible && g.rows_mode == 1;
  // auto (mode 0) is off: measured slower than the ordinary path on every
  // database tried, including one long sequence with a short query
  // (profiles/r02_rows_mode.jsonl); kRowsAuto keeps the model for experiments
  if (kRowsAuto && rows_possible && g.rows_mode == 0 && I0.n_long <= g.num_sms) {
    // auto: the longest sequence's chain in the rows kernel (one CTA per item,
    // warps on consecutive passes) against its chain in the pass kernel, when
    // that chain bounds the search (profiles/r02_rows_mode.jsonl)
    const int tn = choose_tile(mm, 0, I0);
    if (tn >= 0) {
      const TileInfo tt = tile(tn);
      const double f = 1.9e9;
      const double chain_normal = ((double)I0.long_max_len + tt.G) * (kStepC0 + kStepC1 * tt.R) / f;
      const double P = std::ceil((double)I0.long_max_len / kRowsRows);
      const double ncq = (double)((m + 2 + 3) & ~3);
      const double rows_t = kRowsStep * (std::ceil(P / kRowsWarps) * (ncq + 31.0) +
                                         (std::min(P, (double)kRowsWarps) - 1.0) * kRowsLag) / f;
      Image Iv2 = I0;
      Iv2.max_item_cols = I0.max_item_cols_rest;
      Iv2.total_cols = std::max<int64_t>(1, I0.total_cols - I0.long_cols);
      const double t_rest = pass_time_model(tt, mm, shape_of(Iv2), false);
      const double t_all = pass_time_model(tt, mm, shape_of(I0), false);
      rows_cand = chain_normal >= t_all * 0.99 && t_rest + rows_t < 0.8 * t_all;
    }
  }
  const Image &I = I0;
  // the tile model's view of the items the pass kernel runs (rows mode: all
  // but the long pairs); device buffers are shared, only these sizes differ
  Image Iv = I0;
  if (rows_cand) {
    Iv.max_item_cols = I0.max_item_cols_rest;
    Iv.total_cols = std::max<int64_t>(1, I0.total_cols - I0.long_cols);
    Iv.num_items = std::max(1, I0.num_items - I0.n_long);
  }
  auto passes_of = [&](int i) { return (mm + tile(i).G * tile(i).R - 1) / (tile(i).G * tile(i).R); };
  int ti = choose_tile(mm, mode, rows_cand ? Iv : I);
  if (ti < 0) return fail(SW_ECUDA, "no runnable kernel tile");
  // rows mode needs a single pass of the pass kernel; otherwise the ordinary choice
  const bool rows_ok = rows_cand && passes_of(ti) == 1;
  if (rows_cand && !rows_ok) ti = choose_tile(mm, mode, I);
  const Image &Im = rows_ok ? Iv : I;   // what the latency model sees
  // Cross-pass wavefront (one launch runs every pass).  A pass
  // of the per-pass path keeps at most one lane group per work item busy; with
  // far fewer items than groups (a database of few, long sequences) the
  // wavefront runs the query passes of an item on several groups at once.
  // Auto rule, from a tile sweep on databases of 10-4,000 items of 1-35 k
  // residues (profiles/r01b_wavefront_tiles.jsonl): below half as many items
  // as 32-lane groups, 32x8 tiles when the query makes >= 4 passes of them and
  // the units (items x passes) do not overfill the groups 1.5 times, else 32x16
  // tiles when their units exceed half the groups.  Forced mode (1) uses the
  // forced or chosen tile when it has a wavefront kernel, else 32x16 / 32x8.
  bool wave = false;
  if (!pair && !use_sp && !g.streamed && !rows_ok && g.wave_mode >= 0) {
    const int t8 = find_tile_mode(32, 8, 0), t16 = find_tile_mode(32, 16, 0);
    const double items = (double)std::max(1, I.num_items);
    int tw = -1;
    if (g.wave_mode == 1) {
      if (tile_has_wave(ti) && passes_of(ti) > 1) tw = ti;
      else if (!g.force_G && t16 >= 0 && tile_has_wave(t16) && passes_of(t16) > 1) tw = t16;
      else if (!g.force_G && t8 >= 0 && tile_has_wave(t8) && passes_of(t8) > 1) tw = t8;
    } else if (!g.force_G && t8 >= 0 && t16 >= 0 && tile_has_wave(t8) && tile_has_wave(t16)) {
      const double groups32 = (double)g.num_sms * std::max(1, tile_ctas_per_sm(t8)) * 512.0 / 32.0;
      if (items < 0.5 * groups32) {
        // >= 4 passes since the last session of round 2 (tools/wave_small.py, 1-100
        // items of 20-35 k residues: m = 1000 runs 1.3-1.7x faster as 4 chained
        // 32x8 passes than as one 32x32 pass; 2-3 passes are slower or mixed)
        if (passes_of(t8) >= 4 && items * passes_of(t8) <= 1.5 * groups32) tw = t8;
        else if (passes_of(t16) >= 2 && items * passes_of(t16) > 0.5 * groups32) tw = t16;
      }
    }
    if (tw >= 0) {
      ti = tw;
      wave = true;
    }
  }
  // Latency tiles: when one long work item's critical path,
  // not the total work, bounds the pass (a small database with a long
  // sequence, e.g. configs[0]), run a small-R tile on one 256-thread CTA per
  // SM: the per-column step of a group is shorter.
  bool lat = false;
  if (!pair && !use_sp && !wave && g.lat_mode >= 0) {
    int tl = -1;
    if (g.force_G) {   // a forced latency tile: used when forced or when it is latency-only
      const int tf = find_tile_mode(g.force_G, g.force_R, 0, 1);
      if (tf >= 0 && (g.lat_mode == 1 || find_tile_mode(g.force_G, g.force_R, 0, 0) < 0)) tl = tf;
      else if (g.lat_mode == 1) tl = choose_lat_tile(mm, shape_of(Im), ti, true, rows_ok);
    } else {
      tl = choose_lat_tile(mm, shape_of(Im), ti, g.lat_mode == 1, rows_ok);
    }
    if (tl >= 0) {
      ti = tl;
      lat = true;
    }
  }
  const TileInfo T = tile(ti);
  const int rows = T.G * T.R;
  const int P = (mm + rows - 1) / rows;
  if (P > kMaxPass) return fail(SW_EINVAL, "query too long");
  const bool rowsm = rows_ok && !wave && P == 1;   // (a forced multi-pass latency tile turns it off)
  int smax = 1;
  for (int i = 0; i < kAlpha * kAlpha; ++i) smax = std::max(smax, (int)matrix[i]);
  const int thresh = kHalfTop - smax;   // stored 16-bit units (R7)
  g.last_thresh = thresh - kBias16;  // in score units
  // A local alignment pairs at most min(m, n) residues, each scoring <= smax,
  // so no score reaches the flag threshold when smax * min(m, longest
  // sequence) is below it (configs[0-3]): the search then launches no flag
  // detection, no flag compaction, no item skipping and no 32-bit re-scoring.
  const bool can_flag = (int64_t)smax * std::min<int64_t>(mm, std::max<int64_t>(g.max_len, 1)) >=
                        (int64_t)g.last_thresh;
  const int goe = gap_open + gap_extend, ge = gap_extend;

  // Item cursors per (chunk, pass), then the solo cursors: the leading,
  // chain-bound items of a chunk (the whole resident image is one chunk) are
  // claimed only by the first group of warps 0-3 of a CTA, one per SM
  // sub-partition, whose partner warps then claim nothing, so the long item
  // streams without competing for issue slots.  Latency tiles
  // only (the model chose them because a chain bounds the pass; in the
  // throughput tiles the claim code alone measured 1.7-2.3% slower: register
  // allocation of the main loop).  Rows mode: the pass kernel starts claiming
  // after the long items.
  // streamed: the chunks, then the resident head (cursor index nchk - 1)
  const int nchk = g.streamed ? (int)g.chunks.size() + (g.has_head ? 1 : 0) : 1;
  auto chunk_at = [&](int k) -> const State::Chunk & { return k < (int)g.chunks.size() ? g.chunks[k] : g.head; };
  const int first = rowsm ? I0.n_long : 0;
  std::vector<int> solo_n((size_t)nchk, 0);
  if (solo_enabled() && lat && T.G == 32 && !pair && !use_sp && !wave) {
    for (int k = 0; k < nchk; ++k) {
      const int ib = g.streamed ? chunk_at(k).item_begin : first;
      const int ie = g.streamed ? chunk_at(k).item_end : I0.num_items;
      if (ie <= ib) continue;
      const int64_t thr = std::max<int64_t>(512, I0.item_ncols[ib] / 2);   // half the chunk's longest item
      int n = 0;
      // at most one per SM: each idles the other warps of its sub-partition
      while (ib + n < ie && n < g.num_sms && I0.item_ncols[ib + n] >= thr) ++n;
      solo_n[k] = n;
    }
  }

  // pc[k * P + pass]: item cursor, pc[nchk * P + k * P + pass]: solo cursor
  // (item indices relative to the chunk's first item); copied with the inputs
  const size_t pc_off = ((size_t)kAlpha * kAlpha + (size_t)m + (pair ? (size_t)m2 : 0) + 15) & ~(size_t)15;
  const size_t npc = (size_t)2 * nchk * P;
  const size_t in_bytes = pc_off + npc * sizeof(int);
  CUDA_TRY(g.qin.ensure(in_bytes));
  const int slot = g_stage.next;
  g_stage.next = (slot + 1) % Staging::kSlots;
  if (g_stage.ev[slot]) CUDA_TRY(cudaEventSynchronize(g_stage.ev[slot]));   // its previous copy is done
  else CUDA_TRY(cudaEventCreateWithFlags(&g_stage.ev[slot], cudaEventDisableTiming));
  if (g_stage.cap[slot] < in_bytes) {
    if (g_stage.h[slot]) cudaFreeHost(g_stage.h[slot]);
    g_stage.h[slot] = nullptr;
    g_stage.cap[slot] = 0;
    const size_t cap = std::max<size_t>(in_bytes, 64 * 1024);
    CUDA_TRY(cudaHostAlloc(&g_stage.h[slot], cap, cudaHostAllocDefault));
    g_stage.cap[slot] = cap;
  }
  std::memcpy(g_stage.h[slot], matrix, (size_t)kAlpha * kAlpha);
  std::memcpy(g_stage.h[slot] + kAlpha * kAlpha, q, (size_t)m);
  if (pair) std::memcpy(g_stage.h[slot] + kAlpha * kAlpha + m, q2, (size_t)m2);
  {
    int *hpc = reinterpret_cast<int *>(g_stage.h[slot] + pc_off);
    for (int k = 0; k < nchk; ++k) {
      const int start = g.streamed ? 0 : first;
      for (int pass = 0; pass < P; ++pass) {
        hpc[(size_t)k * P + pass] = start + solo_n[(size_t)k];
        hpc[(size_t)nchk * P + (size_t)k * P + pass] = start;
      }
    }
  }
  int *const pc = reinterpret_cast<int *>(g.qin.p + pc_off);
  g.mat_d = reinterpret_cast<const int8_t *>(g.qin.p);
  g.q_d = g.qin.p + kAlpha * kAlpha;
  g.q2_d = pair ? g.q_d + m : nullptr;
  CUDA_TRY(g.qp.ensure(qp_bytes(T.G, T.R, P, T.qpm)));
  CUDA_TRY(g.desc.ensure((size_t)kNL * kNL));
  CUDA_TRY(g.qp32.ensure((size_t)kNL * mm));
  if (pair) CUDA_TRY(g.qp32b.ensure((size_t)kNL * mm));

  // The per-search scratch (profile, flags, counters, sc_out, boundaries, ...)
  // is shared by every search: order this search's device work after the
  // previous one's, whatever stream that ran on (ev[3] marks its end).
  if (g.has_search && g.ev[3]) CUDA_TRY(cudaStreamWaitEvent(st, g.ev[3], 0));
  // Streamed database: the copy engine is busy with chunk copies of several
  // ms each, and a small copy queues behind them (measured: ~5 ms between
  // back-to-back searches on cfg2 with 1 GiB chunks), so a kernel reads the
  // pinned slot over the link instead.  SWDB_STAGE_KERNEL=0/1 forces either.
  static const int stage_kernel_env = [] {
    const char *e = std::getenv("SWDB_STAGE_KERNEL");
    return e ? (e[0] == '0' ? 0 : 1) : -1;
  }();
  if (stage_kernel_env == 1 || (stage_kernel_env < 0 && g.streamed)) {
    void *hdev = nullptr;
    CUDA_TRY(cudaHostGetDevicePointer(&hdev, g_stage.h[slot], 0));
    CUDA_TRY(launch_stage_copy(hdev, g.qin.p, in_bytes, st));
  } else {
    CUDA_TRY(cudaMemcpyAsync(g.qin.p, g_stage.h[slot], in_bytes, cudaMemcpyHostToDevice, st));
  }
  CUDA_TRY(cudaEventRecord(g_stage.ev[slot], st));
  // 32-bit re-scoring counters: (count, cursor) per (pass, query of the pair),
  // plus one set for the end-of-search launch; flags; carry marks
  CUDA_TRY(g.fcounters.ensure((size_t)4 * (P + 1)));
  const int32_t *item_of = pair ? nullptr : g.img[0].item_of.p;
  if (!pair) CUDA_TRY(g.item_hot.ensure((size_t)std::max(1, g.img[0].num_items)));
  // zeroed by the profile launch below
  const SearchInit zinit{g.fcounters.p, 4 * (P + 1), g.flagged.p, pair ? g.flagged2.p : nullptr, g.count,
                         g.cells32.p, pair ? nullptr : g.item_hot.p, pair ? 0 : std::max(1, g.img[0].num_items)};
  if (!g.ev[0])
    for (int i = 0; i < 4; ++i) CUDA_TRY(cudaEventCreate(&g.ev[i]));
  // a batch's timing spans all of its searches (sw_last_timing)
  if (!g.batch_cont) {
    CUDA_TRY(cudaEventRecord(g.ev[0], st));
    g.hslot = (g.hslot + 1) % State::kHist;
    g.pevp = &g.hpev[g.hslot];
    g.hnpev[g.hslot] = 0;
    ++g.nsearch;
    g.npev = 0;
  }
  std::vector<cudaEvent_t> &pev = *g.pevp;
  auto pass_event = [&](int idx) -> cudaError_t {   // event slot idx of this search's launches
    while (pev.size() < (size_t)idx + 1) {
      cudaEvent_t e;
      cudaError_t er = cudaEventCreate(&e);
      if (er != cudaSuccess) return er;
      pev.push_back(e);
    }
    return cudaSuccess;
  };
  const int pev0 = 2 * g.npev;
  CUDA_TRY(launch_qp_build(g.q_d, m, pair ? g.q2_d : nullptr, m2, g.mat_d, T.G, T.R, P, g.qp.p,
                           g.desc.p, g.qp32.p, pair ? g.qp32b.p : nullptr,
                           goe, ge, st, use_sp ? 1 : 0, zinit));

  const int grid = g.num_sms * (lat ? 1 : std::max(1, tile_ctas_per_sm(ti)));
  // Exact s32 re-scoring ("recalculated using the next wider
  // integer range").  Resident database: right after the gather of pass p, the
  // sequences first flagged in pass p are re-scored from row p*rows on, seeded
  // with that pass's input boundary (exact: no earlier pass flagged them) and
  // with the exact maximum of the earlier passes.  Streamed database: once at
  // the end, from row 0.
  // The flag byte is min(pass + 1, 255): passes >= 254 share the value 255 and
  // are re-scored at the end, from row 0.
  // compacted: the flag list of (pass, k) was already written by the update launch
  auto rescore = [&](int k, int pass, const uint2 *bnd16, bool compacted = false) -> cudaError_t {
    const bool early = pass >= 0 && pass + 1 < 255;
    const int slot = early ? pass : P;
    int *cnt = g.fcounters.p + 4 * slot + 2 * k;
    const int row0 = early ? pass * rows : 0;
    const int want = pass < 0 ? 0 : (early ? pass + 1 : 255);
    const int len = k ? m2 : m;
    cudaError_t e = compacted ? cudaSuccess
                              : launch_flag_compact(k ? g.flagged2.p : g.flagged.p, g.count,
                                                    k ? g.flag_list2.p : g.flag_list.p, cnt, want, st);
    if (e != cudaSuccess || row0 >= len) return e;
    SW32Params q{};
    q.flag_list = k ? g.flag_list2.p : g.flag_list.p;
    q.flag_count = cnt;
    q.cursor = cnt + 1;
    q.res = g.res_dev;
    q.offs = g.offs.p;
    q.qp32 = k ? g.qp32b.p : g.qp32.p;
    q.m = mm;
    q.len = len;
    q.row0 = row0;
    q.passes = (len - row0 + 32 * kSW32Rows - 1) / (32 * kSW32Rows);
    q.neg_goe = -goe;
    q.neg_ge = -ge;
    q.bnd16 = row0 > 0 ? bnd16 : nullptr;
    q.endcol = I.endcol.p;
    q.half = pair ? k : -1;
    q.scratch = g.scratch32.p;
    q.stride = g.scratch_stride;
    q.scores = k ? d_scores2 : d_scores;
    q.cells = g.cells32.p;
    q.one = 1u;
    return launch_sw32(g.sw32_grid, q, st);
  };
  // resident database: one "chunk" (the whole image); streamed database: the
  // image's chunks are copied host->device on copy_st into two buffers,
  // overlapping the passes of the previous chunk
  const bool strm = g.streamed;
  const int nch = strm ? (int)g.chunks.size() : 1;
  const int64_t span = strm ? g.chunk_span : I.total_cols;
  const int ncq = (m + 2 + 3) & ~3;   // rows mode: the query stream (m letters, END, NUL, padding)
  if (rowsm) {
    CUDA_TRY(g.rows_wrap.ensure((size_t)g.num_sms * ncq));
    CUDA_TRY(g.rows_prog.ensure(1));
    CUDA_TRY(cudaMemsetAsync(g.rows_prog.p, 0, sizeof(int), st));
  }
  if (P > 1 && g.bnd.n < (size_t)span * 2) CUDA_TRY(g.bnd.ensure((size_t)span * 2));
  if (!strm && !pair && P > 1) CUDA_TRY(g.skip.ensure((size_t)std::max(1, I.num_items)));
  CUDA_TRY(cudaEventRecord(g.ev[1], st));
  if (wave) {
    CUDA_TRY(g.progress.ensure((size_t)P * std::max(1, I.num_items)));
    CUDA_TRY(cudaMemsetAsync(g.progress.p, 0, sizeof(int) * (size_t)P * std::max(1, I.num_items), st));
    SW16Params p{};
    p.stream = I.stream.p;
    p.items = I.items.p;
    p.num_items = I.num_items;
    p.counter = pc;
    p.qp = reinterpret_cast<const uint4 *>(g.qp.p);
    p.desc = g.desc.p;
    p.bnd_in = nullptr;
    p.bnd_out = nullptr;
    p.dummy = g.dummy.p;
    p.nul_stream = g.nulcols.p;
    p.zero_bnd = g.zerocols.p;
    p.col_lo = 0;
    p.col_hi = I.total_cols;
    p.sc_out = g.sc_out.p;
    p.pass = 0;
    p.thresh = thresh;
    p.zero = 0u;
    p.one = 1u;
    p.npass = P;
    p.pcounters = pc;
    p.progress = g.progress.p;
    p.bndbuf[0] = g.bnd.p;
    p.bndbuf[1] = g.bnd.p + span;
    CUDA_TRY(pass_event(pev0 + 1));
    CUDA_TRY(cudaEventRecord(pev[pev0], st));
    // every CTA must be resident: a wavefront CTA may wait on another's progress
    const int wgrid = g.num_sms * tile_wave_ctas_per_sm(ti);
    {
      // few units: spread them, at most ceil(units / CTAs) groups per CTA claim
      // (all units are still claimed at once: the limit times the grid covers them)
      const int64_t units = (int64_t)std::max(1, I.num_items) * P;
      const int64_t lim = (units + wgrid - 1) / wgrid;
      // measured (tools/wave_small.py, 1-100 items of 20-35 k residues): up to 4
      // groups per CTA the spread is 1.2-1.3x faster (100 items x 4 passes 12.9 ->
      // 10.4 ms, 10-30 items 10.9 -> 8.3-8.5), at 6 (100 items x 8 passes) slower
      // (13.3 -> 15.8 ms), so it is used up to 4
      p.group_limit = (lim <= 4 && lim < 512 / T.G) ? (int)lim : 0;
      if (const char *e = std::getenv("SWDB_WAVE_SPREAD")) if (e[0] == '0') p.group_limit = 0;
    }
    CUDA_TRY(launch_sw16_pass(ti, wgrid, p, st));
    CUDA_TRY(cudaEventRecord(pev[pev0 + 1], st));
    g.npev = pev0 / 2 + 1;
    g.hnpev[g.hslot] = g.npev;
    // the score chain was carried through the passes: one gather of the maxima
    CUDA_TRY(launch_sw16_gather(I.endcol.p, g.count, g.sc_out.p, d_scores, g.flagged.p, nullptr, nullptr, 0,
                                thresh, st, nullptr, item_of, g.item_hot.p, nullptr, nullptr, nullptr, nullptr, 0,
                                can_flag));
  }
  int npl = 0;   // pass launches so far (per-pass path)
  // Streamed database with a resident head: its passes and gathers run on
  // head_st (high priority: its CTAs take the first SMs that free up) beside
  // the chunks below; the search stream joins it after the last chunk.
  const bool head = strm && !wave && g.has_head;
  if (head) {
    const State::Chunk &c = g.head;
    const int kh = nch;   // cursor index of the head
    const int64_t hc = c.col_end - c.col_begin, base = c.col_begin;
    if (P > 1) CUDA_TRY(g.head_bnd.ensure((size_t)hc * 2));
    CUDA_TRY(cudaStreamWaitEvent(g.head_st, g.ev[1], 0));   // the profile and the cursors are ready
    for (int pass = 0; pass < P; ++pass) {
      SW16Params p{};
      p.stream = g.head_buf.p - base;
      p.items = I.items.p + c.item_begin;
      p.num_items = c.item_end - c.item_begin;
      p.counter = pc + (size_t)kh * P + pass;
      p.qp = reinterpret_cast<const uint4 *>(g.qp.p);
      p.desc = g.desc.p;
      p.bnd_in = pass == 0 ? nullptr : g.head_bnd.p + (size_t)((pass - 1) & 1) * hc - base;
      p.bnd_out = pass == P - 1 ? nullptr : g.head_bnd.p + (size_t)(pass & 1) * hc - base;
      p.dummy = g.dummy.p;
      p.nul_stream = g.nulcols.p;
      p.col_lo = base;
      p.col_hi = c.col_end;
      p.zero_bnd = g.zerocols.p;
      p.sc_out = g.head_sc.p - base;
      p.pass = pass;
      p.thresh = thresh;
      p.zero = 0u;
      p.one = 1u;
      p.skip = nullptr;
      p.query = g.q_d;
      p.m = m;
      p.solo_counter = solo_n[(size_t)kh] ? pc + (size_t)nchk * P + (size_t)kh * P + pass : nullptr;
      p.solo_end = solo_n[(size_t)kh];
      const int pe = pev0 + 2 * npl++;
      CUDA_TRY(pass_event(pe + 1));
      CUDA_TRY(cudaEventRecord(pev[pe], g.head_st));
      CUDA_TRY(launch_sw16_pass(ti, grid, p, g.head_st));
      CUDA_TRY(cudaEventRecord(pev[pe + 1], g.head_st));
      g.npev = pe / 2 + 1;
      g.hnpev[g.hslot] = g.npev;
      CUDA_TRY(launch_sw16_gather(g.cseq_endcol.p + c.seq_begin, c.seq_end - c.seq_begin, g.head_sc.p - base,
                                  d_scores, g.flagged.p, nullptr, nullptr, pass, thresh, g.head_st,
                                  g.cseq_idx.p + c.seq_begin, item_of, g.item_hot.p, nullptr, nullptr, nullptr,
                                  nullptr, 0, can_flag));
    }
    CUDA_TRY(cudaEventRecord(g.ev_head, g.head_st));
  }
  for (int k = 0; k < (wave ? 0 : nch); ++k) {
    const uint32_t *stream_base = I.stream.p;
    const Item *items = I.items.p;
    int nitems = I.num_items;
    int64_t base = 0;
    const int b = (k + (strm ? g.buf_parity : 0)) & 1;
    if (strm) {
      const State::Chunk &c = g.chunks[k];
      if (k > 0 || !g.chunk0_staged) {
        // the buffer is free once the passes of the chunk that used it last are done
        CUDA_TRY(cudaStreamWaitEvent(g.copy_st, g.ev_free[b], 0));
        // the 16-bit image crosses the host link (2 B per column, 1 B per
        // residue) and is expanded to 32-bit column words on the device
        CUDA_TRY(cudaMemcpyAsync(g.cbuf16[b].p, g.h_stream + c.col_begin, (size_t)(c.col_end - c.col_begin) * 2,
                                 cudaMemcpyHostToDevice, g.copy_st));
        CUDA_TRY(cudaEventRecord(g.ev_copied[b], g.copy_st));
      }
      CUDA_TRY(cudaStreamWaitEvent(st, g.ev_copied[b], 0));
      CUDA_TRY(launch_expand_columns(g.cbuf16[b].p, c.col_end - c.col_begin, g.cbuf[b].p, st));
      base = c.col_begin;
      stream_base = g.cbuf[b].p - base;     // so that item.col_begin indexes the buffer
      items = I.items.p + c.item_begin;
      nitems = c.item_end - c.item_begin;
    }
    for (int pass = 0; pass < P; ++pass) {
      SW16Params p{};   // npass = 0: one pass per launch
      p.stream = stream_base;
      p.items = items;
      p.num_items = nitems;
      p.counter = pc + (size_t)k * P + pass;
      p.qp = reinterpret_cast<const uint4 *>(g.qp.p);
      p.desc = g.desc.p;
      p.bnd_in = pass == 0 ? nullptr : g.bnd.p + (size_t)((pass - 1) & 1) * span - base;
      p.bnd_out = pass == P - 1 ? nullptr : g.bnd.p + (size_t)(pass & 1) * span - base;
      p.dummy = g.dummy.p;
      p.nul_stream = g.nulcols.p;
      p.col_lo = base;
      p.col_hi = strm ? g.chunks[k].col_end : I.total_cols;
      p.zero_bnd = g.zerocols.p;
      p.sc_out = g.sc_out.p - base;
      p.pass = pass;
      p.thresh = thresh;
      p.zero = 0u;
      p.one = 1u;
      // resident single-query passes after the first start each item behind
      // its leading run of flagged sequences (item_skip_kernel below)
      const bool skipping = !strm && !pair && P > 1 && can_flag;
      p.skip = (skipping && pass > 0) ? g.skip.p : nullptr;
      p.query = g.q_d;
      p.m = m;
      // the chunk's solo items (SWDB_SOLO=0 turns them off for experiments)
      p.solo_counter = solo_n[(size_t)k] ? pc + (size_t)nchk * P + (size_t)k * P + pass : nullptr;
      p.solo_end = (strm ? 0 : first) + solo_n[(size_t)k];
      const int pe = pev0 + 2 * npl++;   // event slots: this search's pass launches in order
      CUDA_TRY(pass_event(pe + 1));
      CUDA_TRY(cudaEventRecord(pev[pe], st));
      CUDA_TRY(launch_sw16_pass(ti, grid, p, st));
      if (rowsm) {   // the long pairs, rows along the database sequence (before the gather reads sc_out)
        RowsParams r{};
        r.query = g.q_d;
        r.m = m;
        r.ncq = ncq;
        r.matrix = g.mat_d;
        r.res = g.res.p;
        r.offs = g.offs.p;
        r.items = I0.items.p;
        r.slots = I0.slots.p;
        r.n_items = I0.n_long;
        r.counter = g.rows_prog.p;
        r.wrap = g.rows_wrap.p;
        r.endcol = I0.endcol.p;
        r.sc_out = g.sc_out.p;
        r.goe = goe;
        r.ge = ge;
        r.one = 1u;
        CUDA_TRY(launch_sw16_rows(g.num_sms, r, st));
      }
      CUDA_TRY(cudaEventRecord(pev[pe + 1], st));
      g.npev = pe / 2 + 1;
      g.hnpev[g.hslot] = g.npev;
      if (strm) {
        const State::Chunk &c = g.chunks[k];
        CUDA_TRY(launch_sw16_gather(g.cseq_endcol.p + c.seq_begin, c.seq_end - c.seq_begin, g.sc_out.p - base,
                                    d_scores, g.flagged.p, nullptr, nullptr, pass, thresh, st,
                                    g.cseq_idx.p + c.seq_begin, item_of, g.item_hot.p, nullptr, nullptr, nullptr,
                                    nullptr, 0, can_flag));
      } else {
        // the update launch also compacts the sequences first flagged in this
        // pass for the 32-bit kernel (passes < 254; flag byte pass + 1)
        const bool fuse = pass + 1 < 255 && can_flag;
        CUDA_TRY(launch_sw16_gather(I.endcol.p, g.count, g.sc_out.p, d_scores, g.flagged.p,
                                    pair ? d_scores2 : nullptr, pair ? g.flagged2.p : nullptr, pass, thresh, st,
                                    nullptr, item_of, pair ? nullptr : g.item_hot.p, g.flag_list.p,
                                    g.fcounters.p + 4 * pass, pair ? g.flag_list2.p : nullptr,
                                    g.fcounters.p + 4 * pass + 2, fuse ? pass + 1 : 0, can_flag));
        if (fuse)
          for (int k = 0; k < (pair ? 2 : 1); ++k) CUDA_TRY(rescore(k, pass, p.bnd_in, true));
        if (skipping && pass + 1 < P)
          CUDA_TRY(launch_item_skip(I.items.p, I.num_items, I.slots.p, g.offs.p, g.flagged.p, g.skip.p, st));
      }
    }
    if (strm) CUDA_TRY(cudaEventRecord(g.ev_free[b], st));
  }
  if (head) CUDA_TRY(cudaStreamWaitEvent(st, g.ev_head, 0));
  if (strm && !wave) {
    // the next search's chunk 0 into the buffer this search's last chunk did not use
    g.chunk0_staged = false;
    const int nb = (g.buf_parity + nch) & 1;
    const State::Chunk &c0 = g.chunks[0];
    CUDA_TRY(cudaStreamWaitEvent(g.copy_st, g.ev_free[nb], 0));
    CUDA_TRY(cudaMemcpyAsync(g.cbuf16[nb].p, g.h_stream + c0.col_begin, (size_t)(c0.col_end - c0.col_begin) * 2,
                             cudaMemcpyHostToDevice, g.copy_st));
    CUDA_TRY(cudaEventRecord(g.ev_copied[nb], g.copy_st));
    g.buf_parity = nb;
    g.chunk0_staged = true;
  }
  CUDA_TRY(cudaEventRecord(g.ev[2], st));
  if ((strm || wave || P >= 255) && can_flag)
    for (int k = 0; k < (pair ? 2 : 1); ++k) CUDA_TRY(rescore(k, (strm || wave) ? -1 : 254, nullptr));
  CUDA_TRY(cudaEventRecord(g.ev[3], st));

  g.has_search = true;
  g.last_scores = d_scores;
  g.last_stream = st;
  g.last_G = T.G;
  g.last_R = T.R;
  g.last_P = P;
  g.last_mode = mode;
  g.last_wave = wave;
  g.last_lat = lat;
  g.last_prof = use_sp ? 2 : 1;
  g.last_rows = rowsm ? I0.n_long : 0;
  g.last_flags = -1;
  g.last_cells32 = -1;
  return SW_OK;
}

int search_impl(const uint8_t *query, int32_t qlen, const int8_t *matrix, int32_t gap_open,
                int32_t gap_extend, int32_t *d_scores, cudaStream_t st) {
  return search_core(query, qlen, nullptr, 0, matrix, gap_open, gap_extend, d_scores, nullptr, st);
}

int validate_batch(const uint8_t *queries, const int64_t *qoffsets, int32_t nq) {
  if (!queries || !qoffsets) return fail(SW_EINVAL, "queries or qoffsets is NULL");
  if (nq < 1) return fail(SW_EINVAL, "nq must be >= 1");
  if (qoffsets[0] != 0) return fail(SW_EINVAL, "qoffsets[0] must be 0");
  for (int32_t k = 0; k < nq; ++k)
    if (qoffsets[k + 1] - qoffsets[k] < 1 || qoffsets[k + 1] - qoffsets[k] >= (int64_t(1) << 31))
      return fail(SW_EINVAL, "query " + std::to_string(k) + " has length < 1 or >= 2^31");
  return SW_OK;
}

// Batch: queries sorted by length, consecutive ones paired into the two 16-bit
// halves (one pass over the single-sequence image serves both); an odd one
// left over runs alone.
int batch_impl(const uint8_t *queries, const int64_t *qoffsets, int32_t nq, const int8_t *matrix,
               int32_t gap_open, int32_t gap_extend, int32_t *d_scores, cudaStream_t st) {
  int rc = validate_batch(queries, qoffsets, nq);
  if (rc) return rc;
  std::vector<int32_t> order(nq);
  for (int32_t k = 0; k < nq; ++k) order[k] = k;
  std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
    return qoffsets[x + 1] - qoffsets[x] > qoffsets[y + 1] - qoffsets[y];
  });
  struct BatchGuard {   // the batch's searches share one timing window
    ~BatchGuard() { g.batch_cont = false; }
  } guard;
  for (int32_t k = 0; k < nq; k += 2) {
    g.batch_cont = k > 0;
    const int32_t a = order[k];
    const uint8_t *qa = queries + qoffsets[a];
    const int32_t ma = (int32_t)(qoffsets[a + 1] - qoffsets[a]);
    if (k + 1 < nq) {
      const int32_t b = order[k + 1];
      rc = search_core(qa, ma, queries + qoffsets[b], (int32_t)(qoffsets[b + 1] - qoffsets[b]), matrix, gap_open,
                       gap_extend, d_scores + (size_t)a * g.count, d_scores + (size_t)b * g.count, st);
    } else {
      rc = search_core(qa, ma, nullptr, 0, matrix, gap_open, gap_extend, d_scores + (size_t)a * g.count, nullptr, st);
    }
    if (rc) return rc;
  }
  g.last_scores = d_scores;   // sw_topk after a batch ranks query 0
  return SW_OK;
}

}  // namespace

extern "C" {

const char *sw_last_error(void) { return t_err.c_str(); }
const char *sw_version(void) { return "swdb-b200 0.1 (sm_100a)"; }

void sw_db_free(void) {
  if (g.loaded || g.stream) {
    g.release_all();
    if (g.stream) cudaStreamDestroy(g.stream);
    g.stream = nullptr;
  }
  g.loaded = false;
}

int64_t sw_db_count(void) { return g.loaded ? g.count : 0; }
int64_t sw_launch_count(void) { return launch_count(); }
int64_t sw_db_residues(void) { return g.loaded ? g.total_res : 0; }

}  // extern "C"

namespace {

// chunk_bytes == 0: resident database (both images on the device).
// chunk_bytes  > 0: streamed database: the sequence-pair image stays in
// pinned host memory, split into chunks of at most chunk_bytes of stream,
// copied to the device during every search.
int load_impl_body(const uint8_t *residues, const int64_t *offsets, int64_t count, int64_t chunk_bytes) {
  t_err.clear();
  std::string err;
  if (validate_db(residues, offsets, count, err)) return fail(SW_EINVAL, err);
  if (chunk_bytes < 0) return fail(SW_EINVAL, "chunk_bytes must be >= 0");
  const bool strm = chunk_bytes > 0;
  int rc = ensure_device_ready();
  if (rc) return rc;
  int dev = 0, nsm = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  // Items are sized for the number of lane groups that run concurrently with
  // the widest-occupancy tile (4 groups per warp at G = 8, 16 warps per SM).
  const int64_t target_groups = (int64_t)nsm * 16 * 2;
  HostImage himg[2];
  const int nimg = strm ? 1 : 2;
  // the two images are independent: build them on two host threads
  {
    std::string errs[2];
    int rcs[2] = {0, 0};
    auto build_one = [&](int k) {
      try {
        // streamed: items of at most a quarter of a chunk's share per group,
        // so each chunk's launch keeps the 8-lane tiles' 2 x target_groups busy
        // streamed: at least 4 items per group per chunk, and at most 4,096
        // columns per item: a chunk is one launch, whose drain is about one
        // item long (measured on cfg2, m = 144, 1 GiB chunks: cap 14,170 ->
        // 4,096 takes the three pass kernels from 36.6 to 34.0 ms)
        const int64_t cap = strm ? std::max<int64_t>(256, std::min<int64_t>(4096, (chunk_bytes / 4) / (4 * target_groups))) : 0;
        // rows mode (resident pair image): sequences longer than 4x the
        // average columns per lane group are the long pairs
        const int64_t avg = (offsets[count] + 2 * count) / 2 / std::max<int64_t>(1, target_groups);
        const int64_t long_min = (!strm && k == 0) ? std::max<int64_t>(512, 4 * avg) : 0;
        rcs[k] = build_image(residues, offsets, count, target_groups, k == 1, himg[k], errs[k], cap, long_min)
                     ? SW_EINVAL : 0;
      } catch (const std::bad_alloc &) {
        rcs[k] = SW_ENOMEM;
        errs[k] = "host allocation failed in the pre-processor";
      } catch (const std::exception &e) {
        rcs[k] = SW_EINVAL;
        errs[k] = e.what();
      }
    };
    std::thread second;
    if (nimg == 2) second = std::thread(build_one, 1);
    build_one(0);
    if (second.joinable()) second.join();
    for (int k = 0; k < nimg; ++k)
      if (rcs[k]) return fail(rcs[k], errs[k]);
  }
  for (int k = 0; k < nimg; ++k)
    if (himg[k].items.size() >= (size_t)INT_MAX) return fail(SW_EINVAL, "too many work items");
  // replace the previous database
  sw_db_free();
  g.device = dev;
  g.num_sms = nsm;
  CUDA_TRY(cudaStreamCreateWithFlags(&g.stream, cudaStreamNonBlocking));
  g.count = count;
  g.total_res = offsets[count];
  g.max_len = himg[0].max_len;
  g.max_cols = std::max(himg[0].total_cols, himg[1].total_cols);
  for (int k = 0; k < nimg; ++k) {
    Image &I = g.img[k];
    const HostImage &H = himg[k];
    I.total_cols = H.total_cols;
    I.num_items = (int)H.items.size();
    I.item_ncols.resize(H.items.size());
    for (size_t i = 0; i < H.items.size(); ++i) I.item_ncols[i] = H.items[i].ncols;
    I.max_item_cols = 0;
    for (const Item &it : H.items) I.max_item_cols = std::max<int64_t>(I.max_item_cols, it.ncols);
    I.n_long = H.n_long_items;
    I.max_item_cols_rest = 0;
    I.long_cols = 0;
    I.long_min_len = INT64_MAX;
    std::vector<int2> units;
    for (size_t i = 0; i < H.items.size(); ++i) {
      const Item &it = H.items[i];
      if ((int)i >= I.n_long) {
        I.max_item_cols_rest = std::max<int64_t>(I.max_item_cols_rest, it.ncols);
        continue;
      }
      I.long_cols += it.ncols;
      int64_t nmax = 0;
      for (int h = 0; h < it.nA + it.nB; ++h) {
        const int32_t sq = H.slots[it.seqA + h];
        const int64_t n = offsets[sq + 1] - offsets[sq];
        I.long_min_len = std::min(I.long_min_len, n);
        I.long_max_len = std::max(I.long_max_len, n);
        nmax = std::max(nmax, n);
      }
      for (int64_t ps = 0; ps < (nmax + kRowsRows - 1) / kRowsRows; ++ps) units.push_back(make_int2((int)i, (int)ps));
    }
    if (I.n_long == 0) I.long_min_len = 0;
    I.n_units = (int)units.size();
    if (!units.empty()) {
      CUDA_TRY(I.units.ensure(units.size()));
      CUDA_TRY(cudaMemcpy(I.units.p, units.data(), units.size() * sizeof(int2), cudaMemcpyHostToDevice));
    }
    CUDA_TRY(I.items.ensure(H.items.size()));
    CUDA_TRY(cudaMemcpy(I.items.p, H.items.data(), H.items.size() * sizeof(Item), cudaMemcpyHostToDevice));
    if (k == 0) {
      CUDA_TRY(I.item_of.ensure(H.item_of.size()));
      CUDA_TRY(cudaMemcpy(I.item_of.p, H.item_of.data(), H.item_of.size() * sizeof(int32_t),
                          cudaMemcpyHostToDevice));
    }
    if (strm) continue;
    CUDA_TRY(I.stream.ensure(H.stream.size()));
    CUDA_TRY(I.endcol.ensure(H.endcol.size()));
    {   // the 16-bit host image crosses the link, expanded to 32-bit words on the device
      DevBuf<uint16_t> tmp;
      cudaError_t e = tmp.ensure(H.stream.size() + 8);
      if (e == cudaSuccess)
        e = cudaMemcpy(tmp.p, H.stream.data(), H.stream.size() * sizeof(uint16_t), cudaMemcpyHostToDevice);
      if (e == cudaSuccess) e = launch_expand_columns(tmp.p, (int64_t)H.stream.size(), I.stream.p, nullptr);
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
      tmp.release();
      CUDA_TRY(e);
    }
    CUDA_TRY(cudaMemcpy(I.endcol.p, H.endcol.data(), H.endcol.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    CUDA_TRY(I.slots.ensure(H.slots.size()));
    CUDA_TRY(cudaMemcpy(I.slots.p, H.slots.data(), H.slots.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  }
  if (strm) {
    const HostImage &H = himg[0];
    const int64_t chunk_cols = std::max<int64_t>(chunk_bytes / 4, 1);   // device buffer of 32-bit words
    // chunks: maximal runs of consecutive items whose columns (with the NUL
    // padding on both sides) fit chunk_cols; an item longer than that is a
    // chunk of its own
    std::vector<int32_t> item_chunk(H.items.size());
    int64_t span = 0;
    // Balanced chunks: the greedy split fixes the chunk count; the limit is
    // then lowered to the smallest one that still gives that count, so the
    // last chunk is not a short one (a short last chunk cannot hide the copy
    // of the next search's first chunk, and the copy before it idles).
    // Resident head: the leading items within a quarter of a chunk (at least
    // the first item), when at least two chunks' worth of items follow.
    size_t head_end = 0;
    {
      const char *e = std::getenv("SWDB_STREAM_HEAD");
      if (!(e && e[0] == '0') && H.items.size() > 1) {
        const int64_t c0 = H.items[0].col_begin - kItemPad;
        size_t e1 = 1;
        while (e1 < H.items.size() && H.items[e1].col_begin + H.items[e1].ncols + kItemPad - c0 <= chunk_cols / 4) ++e1;
        const int64_t rest = e1 < H.items.size()
                                 ? H.items.back().col_begin + H.items.back().ncols - H.items[e1].col_begin : 0;
        if (rest > chunk_cols) head_end = e1;
      }
    }
    std::vector<State::Chunk> all;
    if (head_end > 0) {
      State::Chunk c;
      c.item_begin = 0;
      c.item_end = (int)head_end;
      c.col_begin = H.items[0].col_begin - kItemPad;
      c.col_end = H.items[head_end - 1].col_begin + H.items[head_end - 1].ncols + kItemPad;
      for (size_t i = 0; i < head_end; ++i) item_chunk[i] = 0;
      all.push_back(c);
    }
    auto count_chunks = [&](int64_t limit) {
      int64_t n = 0;
      for (size_t b = head_end; b < H.items.size(); ++n) {
        const int64_t c0 = H.items[b].col_begin - kItemPad;
        size_t e = b + 1;
        while (e < H.items.size() && H.items[e].col_begin + H.items[e].ncols + kItemPad - c0 <= limit) ++e;
        b = e;
      }
      return n;
    };
    int64_t limit = chunk_cols;
    {
      const int64_t n0 = count_chunks(chunk_cols);
      int64_t lo_l = 1, hi_l = chunk_cols;   // count_chunks(hi_l) == n0; find the smallest such limit
      while (lo_l < hi_l) {
        const int64_t mid = lo_l + (hi_l - lo_l) / 2;
        if (count_chunks(mid) <= n0) hi_l = mid; else lo_l = mid + 1;
      }
      limit = hi_l;
    }
    for (size_t b = head_end; b < H.items.size();) {
      State::Chunk c;
      c.item_begin = (int)b;
      c.col_begin = H.items[b].col_begin - kItemPad;
      size_t e = b + 1;
      while (e < H.items.size() &&
             H.items[e].col_begin + H.items[e].ncols + kItemPad - c.col_begin <= limit)
        ++e;
      c.item_end = (int)e;
      c.col_end = H.items[e - 1].col_begin + H.items[e - 1].ncols + kItemPad;
      for (size_t i = b; i < e; ++i) item_chunk[i] = (int32_t)all.size();
      span = std::max(span, c.col_end - c.col_begin);
      all.push_back(c);
      b = e;
    }
    g.chunk_span = span;
    // per chunk (the head first): its sequences (original index) and their END columns
    std::vector<int64_t> cnt(all.size() + 1, 0);
    for (size_t i = 0; i < H.items.size(); ++i) cnt[item_chunk[i] + 1] += H.items[i].nA + H.items[i].nB;
    for (size_t k = 0; k < all.size(); ++k) cnt[k + 1] += cnt[k];
    std::vector<int32_t> idx((size_t)count);
    std::vector<int64_t> ecol((size_t)count);
    std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
    for (size_t i = 0; i < H.items.size(); ++i) {
      const Item &it = H.items[i];
      for (int32_t s = 0; s < it.nA + it.nB; ++s) {
        const int32_t orig = H.slots[it.seqA + s];
        const int64_t pos = fill[item_chunk[i]]++;
        idx[pos] = orig;
        ecol[pos] = H.endcol[orig];
      }
    }
    for (size_t k = 0; k < all.size(); ++k) {
      all[k].seq_begin = cnt[k];
      all[k].seq_end = cnt[k + 1];
    }
    g.has_head = head_end > 0;
    if (g.has_head) g.head = all[0];
    g.chunks.assign(all.begin() + (g.has_head ? 1 : 0), all.end());
    CUDA_TRY(g.cseq_idx.ensure((size_t)count));
    CUDA_TRY(g.cseq_endcol.ensure((size_t)count));
    CUDA_TRY(cudaMemcpy(g.cseq_idx.p, idx.data(), idx.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(g.cseq_endcol.p, ecol.data(), ecol.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaHostAlloc(&g.h_stream, H.stream.size() * sizeof(uint16_t), cudaHostAllocDefault));
    std::memcpy(g.h_stream, H.stream.data(), H.stream.size() * sizeof(uint16_t));
    for (int k = 0; k < 2; ++k) {
      CUDA_TRY(g.cbuf[k].ensure((size_t)span));
      CUDA_TRY(g.cbuf16[k].ensure((size_t)span + 8));
      CUDA_TRY(cudaEventCreateWithFlags(&g.ev_copied[k], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&g.ev_free[k], cudaEventDisableTiming));
    }
    CUDA_TRY(cudaStreamCreateWithFlags(&g.copy_st, cudaStreamNonBlocking));
    CUDA_TRY(g.sc_out.ensure((size_t)span));
    if (g.has_head) {   // the head's columns, expanded once
      const int64_t hc = g.head.col_end - g.head.col_begin;
      int lo_p = 0, hi_p = 0;
      CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo_p, &hi_p));
      CUDA_TRY(cudaStreamCreateWithPriority(&g.head_st, cudaStreamNonBlocking, hi_p));
      CUDA_TRY(cudaEventCreateWithFlags(&g.ev_head, cudaEventDisableTiming));
      CUDA_TRY(g.head_buf.ensure((size_t)hc));
      CUDA_TRY(g.head_sc.ensure((size_t)hc));
      DevBuf<uint16_t> tmp;
      cudaError_t e = tmp.ensure((size_t)hc + 8);
      if (e == cudaSuccess)
        e = cudaMemcpy(tmp.p, g.h_stream + g.head.col_begin, (size_t)hc * 2, cudaMemcpyHostToDevice);
      if (e == cudaSuccess) e = launch_expand_columns(tmp.p, hc, g.head_buf.p, nullptr);
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
      tmp.release();
      CUDA_TRY(e);
    }
    // residues for the (rare) s32 re-scoring: read over the host link
    CUDA_TRY(cudaHostAlloc(&g.h_res, std::max<size_t>((size_t)g.total_res, 1), cudaHostAllocMapped));
    if (g.total_res > 0) std::memcpy(g.h_res, residues, (size_t)g.total_res);
    uint8_t *dres = nullptr;
    CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void **>(&dres), g.h_res, 0));
    g.res_dev = dres;
    g.streamed = true;
  } else {
    CUDA_TRY(g.sc_out.ensure((size_t)g.max_cols));
    CUDA_TRY(g.res.ensure((size_t)g.total_res));
    if (g.total_res > 0)
      CUDA_TRY(cudaMemcpy(g.res.p, residues, (size_t)g.total_res, cudaMemcpyHostToDevice));
    g.res_dev = g.res.p;
  }
  CUDA_TRY(g.offs.ensure((size_t)count + 1));
  CUDA_TRY(g.scores.ensure((size_t)count));
  CUDA_TRY(g.flagged.ensure((size_t)count));
  CUDA_TRY(g.flagged2.ensure((size_t)count));
  CUDA_TRY(g.flag_list.ensure((size_t)count));
  CUDA_TRY(g.flag_list2.ensure((size_t)count));
  CUDA_TRY(g.cells32.ensure(1));
  CUDA_TRY(g.dummy.ensure((size_t)nsm * 4 * 1024));   // one 16-B slot per resident thread
  {
    CUDA_TRY(g.nulcols.ensure(16));
    CUDA_TRY(g.zerocols.ensure(16));
    std::vector<uint32_t> nw(16, column_word(kNul, kNul));
    CUDA_TRY(cudaMemcpy(g.nulcols.p, nw.data(), 16 * sizeof(uint32_t), cudaMemcpyHostToDevice));
    {
      std::vector<uint2> zc(16, make_uint2((uint32_t)kBias16 * 0x10001u, (uint32_t)kBias16 * 0x10001u));
      CUDA_TRY(cudaMemcpy(g.zerocols.p, zc.data(), 16 * sizeof(uint2), cudaMemcpyHostToDevice));
    }
  }
  CUDA_TRY(cudaMemcpy(g.offs.p, offsets, ((size_t)count + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
  // s32 re-scoring scratch: 2 boundary rows of the longest sequence per warp,
  // 2 CTAs x 8 warps per SM -- capped at 4 GiB (or an eighth of the free
  // device memory): with a very long sequence the 32-bit kernel runs on fewer
  // CTAs instead of failing the load (it claims flagged sequences in a loop)
  g.scratch_stride = g.max_len + 64;
  {
    size_t free_b = 0, total_b = 0;
    CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
    const double budget = std::min<double>(4.0 * (1ull << 30), (double)free_b / 8.0);
    const double per_cta = (double)(kSW32Threads / 32) * 2.0 * (double)g.scratch_stride * sizeof(uint2);
    g.sw32_grid = (int)std::max<double>(1.0, std::min<double>(nsm * 2.0, std::floor(budget / per_cta)));
  }
  const int64_t nwarps32 = (int64_t)g.sw32_grid * (kSW32Threads / 32);
  CUDA_TRY(g.scratch32.ensure((size_t)(nwarps32 * 2 * g.scratch_stride)));
  CUDA_TRY(cudaDeviceSynchronize());
  g.loaded = true;
  return SW_OK;
}

// No C++ exception crosses the ABI: host allocation failures (pre-processor
// vectors, pinned buffers) and thread-creation errors become status codes.
int load_impl(const uint8_t *residues, const int64_t *offsets, int64_t count, int64_t chunk_bytes) {
  try {
    return load_impl_body(residues, offsets, count, chunk_bytes);
  } catch (const std::bad_alloc &) {
    return fail(SW_ENOMEM, "host allocation failed while loading the database");
  } catch (const std::exception &e) {
    return fail(SW_ECUDA, std::string("sw_db_load: ") + e.what());
  } catch (...) {
    return fail(SW_ECUDA, "sw_db_load: unknown exception");
  }
}

}  // namespace

extern "C" {

int sw_db_load(const uint8_t *residues, const int64_t *offsets, int64_t count) {
  return load_impl(residues, offsets, count, 0);
}

int sw_db_load_streamed(const uint8_t *residues, const int64_t *offsets, int64_t count, int64_t chunk_bytes) {
  if (chunk_bytes < 1) {
    t_err = "chunk_bytes must be >= 1";
    return SW_EINVAL;
  }
  return load_impl(residues, offsets, count, chunk_bytes);
}

int64_t sw_db_chunks(void) { return g.loaded && g.streamed ? (int64_t)g.chunks.size() : 0; }

int64_t sw_db_head_columns(void) {
  return g.loaded && g.streamed && g.has_head ? g.head.col_end - g.head.col_begin : 0;
}

int sw_search_dev(const uint8_t *query, int32_t qlen, const int8_t *matrix, int32_t gap_open,
                  int32_t gap_extend, int32_t *d_scores, void *cuda_stream) {
  t_err.clear();
  if (!g.loaded) return fail(SW_ENODB, "no database loaded");
  if (!d_scores) return fail(SW_EINVAL, "d_scores is NULL");
  return search_impl(query, qlen, matrix, gap_open, gap_extend, d_scores, (cudaStream_t)cuda_stream);
}

int sw_search(const uint8_t *query, int32_t qlen, const int8_t *matrix, int32_t gap_open,
              int32_t gap_extend, int32_t *scores_out) {
  t_err.clear();
  if (!g.loaded) return fail(SW_ENODB, "no database loaded");
  if (!scores_out) return fail(SW_EINVAL, "scores_out is NULL");
  int rc = search_impl(query, qlen, matrix, gap_open, gap_extend, g.scores.p, g.stream);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(scores_out, g.scores.p, (size_t)g.count * sizeof(int32_t),
                           cudaMemcpyDeviceToHost, g.stream));
  CUDA_TRY(cudaStreamSynchronize(g.stream));
  return SW_OK;
}

int64_t sw_topk_dev(const int32_t *d_scores, const int64_t *d_index, int64_t n, int64_t k,
                    int64_t *d_idx_out, int32_t *d_score_out, void *cuda_stream) {
  t_err.clear();
  if (!d_scores || n < 0 || k < 0) return fail(SW_EINVAL, "bad arguments");
  if (n >= (int64_t(1) << 32)) return fail(SW_EINVAL, "n must be < 2^32");
  const int64_t kk = std::min(k, n);
  if (kk == 0) return 0;
  if (!d_idx_out || !d_score_out) return fail(SW_EINVAL, "output pointers are NULL");
  int rc = ensure_device_ready();
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  // stream-ordered: the key scratch is shared by every call, so this call's
  // work waits for the previous call's (whatever stream that ran on)
  if (!g.tk_ev) CUDA_TRY(cudaEventCreateWithFlags(&g.tk_ev, cudaEventDisableTiming));
  else CUDA_TRY(cudaStreamWaitEvent(st, g.tk_ev, 0));
  if (kk <= 32) {
    // one block per SM (at most), each warp >= 4 batches of 32 scores
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>((n + 4095) / 4096, g.num_sms > 0 ? g.num_sms : 148));
    CUDA_TRY(g.keys.ensure((size_t)nb * kk));
    CUDA_TRY(g.keys2.ensure((size_t)kk));
    CUDA_TRY(launch_block_topk(d_scores, d_index, nullptr, n, (int)kk, g.keys.p, nb, st));
    CUDA_TRY(launch_block_topk(nullptr, nullptr, g.keys.p, (int64_t)nb * kk, (int)kk, g.keys2.p, 1, st));
    CUDA_TRY(launch_decode_keys(g.keys2.p, kk, d_idx_out, d_score_out, st));
  } else if (kk * 4 <= n) {
    // radix select of the kk-th largest key, then a sort of the kk keys only
    // (DESIGN.md 4.4); the full sort below when kk is a large part of n
    int64_t np2 = 1;
    while (np2 < kk) np2 <<= 1;
    if (np2 < 2) np2 = 2;
    CUDA_TRY(g.keys.ensure((size_t)np2));
    CUDA_TRY(g.keys2.ensure((radix_topk_scratch_bytes() + 7) / 8));
    CUDA_TRY(launch_radix_topk(d_scores, d_index, n, kk, g.keys.p, g.keys2.p, st));
    if (kk > 4096) {
      CUDA_TRY(cudaMemsetAsync(g.keys.p + kk, 0, (size_t)(np2 - kk) * sizeof(uint64_t), st));
      CUDA_TRY(launch_bitonic_sort_desc(g.keys.p, np2, st));
    }
    CUDA_TRY(launch_decode_keys(g.keys.p, kk, d_idx_out, d_score_out, st));
  } else {
    int64_t np2 = 1;
    while (np2 < n) np2 <<= 1;
    if (np2 < 2) np2 = 2;
    CUDA_TRY(g.keys.ensure((size_t)np2));
    CUDA_TRY(launch_make_keys(d_scores, d_index, n, g.keys.p, np2, st));
    CUDA_TRY(launch_bitonic_sort_desc(g.keys.p, np2, st));
    CUDA_TRY(launch_decode_keys(g.keys.p, kk, d_idx_out, d_score_out, st));
  }
  CUDA_TRY(cudaEventRecord(g.tk_ev, st));
  return kk;
}

int sw_scatter_dev(const int32_t *d_src, const int64_t *d_index, int64_t n, int32_t *d_dst, int64_t dst_count,
                   void *cuda_stream) {
  t_err.clear();
  if (n < 0 || dst_count < 0) return fail(SW_EINVAL, "n and dst_count must be >= 0");
  if (n == 0) return SW_OK;
  if (!d_src || !d_index || !d_dst) return fail(SW_EINVAL, "NULL device pointer");
  int rc = ensure_device_ready();
  if (rc) return rc;
  CUDA_TRY(launch_scatter_scores(d_src, d_index, n, d_dst, dst_count, (cudaStream_t)cuda_stream));
  return SW_OK;
}

int64_t sw_topk(int64_t k, int64_t *idx_out, int32_t *score_out) {
  t_err.clear();
  if (k < 0) return fail(SW_EINVAL, "k must be >= 0");
  if (!g.loaded || !g.has_search) return fail(SW_ESTATE, "no completed search");
  const int64_t kk = std::min(k, g.count);
  if (kk == 0) return 0;
  if (!idx_out || !score_out) return fail(SW_EINVAL, "output pointers are NULL");
  CUDA_TRY(g.tk_idx.ensure((size_t)kk));
  CUDA_TRY(g.tk_score.ensure((size_t)kk));
  int64_t r = sw_topk_dev(g.last_scores, nullptr, g.count, kk, g.tk_idx.p, g.tk_score.p, g.last_stream);
  if (r < 0) return r;
  CUDA_TRY(cudaMemcpyAsync(idx_out, g.tk_idx.p, (size_t)kk * sizeof(int64_t), cudaMemcpyDeviceToHost,
                           g.last_stream));
  CUDA_TRY(cudaMemcpyAsync(score_out, g.tk_score.p, (size_t)kk * sizeof(int32_t), cudaMemcpyDeviceToHost,
                           g.last_stream));
  CUDA_TRY(cudaStreamSynchronize(g.last_stream));
  return kk;
}

int sw_last_stats(int64_t *stats, int n) {
  t_err.clear();
  if (!stats || n < 0) return fail(SW_EINVAL, "bad arguments");
  if (g.has_search && g.last_flags < 0) {
    int fc = 0;
    int64_t cells = 0;
    CUDA_TRY(cudaStreamSynchronize(g.last_stream));
    std::vector<int> fcs((size_t)4 * (g.last_P + 1));
    CUDA_TRY(cudaMemcpy(fcs.data(), g.fcounters.p, fcs.size() * sizeof(int), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < fcs.size(); i += 2) fc += fcs[i];
    CUDA_TRY(cudaMemcpy(&cells, g.cells32.p, sizeof(int64_t), cudaMemcpyDeviceToHost));
    g.last_flags = fc;
    g.last_cells32 = cells;
  }
  const Image &I = g.img[g.last_mode == 3 ? 1 : 0];
  const int64_t v[14] = {(int64_t)g.last_G * g.last_R, g.last_P, g.last_G, g.last_R,
                         g.last_flags, g.last_cells32, I.total_cols, I.num_items, g.last_thresh, kArith,
                         g.last_wave ? 1 : 0, g.last_lat ? 1 : 0, g.last_prof, g.last_rows};
  const int m = std::min(n, 14);
  for (int i = 0; i < m; ++i) stats[i] = v[i];
  return m;
}

int sw_last_timing(float *ms, int n) {
  t_err.clear();
  if (!ms || n < 0) return fail(SW_EINVAL, "bad arguments");
  if (!g.has_search || !g.ev[0]) return fail(SW_ESTATE, "no completed search");
  CUDA_TRY(cudaEventSynchronize(g.ev[3]));
  float a = 0.f, b = 0.f;
  for (int i = 0; i < g.npev; ++i) {   // sum of the pass-kernel launches only
    float x = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&x, (*g.pevp)[2 * i], (*g.pevp)[2 * i + 1]));
    a += x;
  }
  CUDA_TRY(cudaEventElapsedTime(&b, g.ev[0], g.ev[3]));
  const float v[2] = {a, b};
  const int m = std::min(n, 2);
  for (int i = 0; i < m; ++i) ms[i] = v[i];
  return m;
}

int sw_timing_history(float *ms, int n) {
  t_err.clear();
  if (!ms || n < 0) return fail(SW_EINVAL, "bad arguments");
  if (!g.has_search || !g.ev[0]) return fail(SW_ESTATE, "no completed search");
  // every search waits for the previous one's end (ev[3]): the last search's
  // end orders all of them
  CUDA_TRY(cudaEventSynchronize(g.ev[3]));
  const int avail = (int)std::min<int64_t>(g.nsearch, State::kHist);
  const int m = std::min(n, avail);
  for (int i = 0; i < m; ++i) {   // oldest first
    const int slot = ((g.hslot - (m - 1 - i)) % State::kHist + State::kHist) % State::kHist;
    float a = 0.f;
    for (int j = 0; j < g.hnpev[slot]; ++j) {
      float x = 0.f;
      CUDA_TRY(cudaEventElapsedTime(&x, g.hpev[slot][2 * j], g.hpev[slot][2 * j + 1]));
      a += x;
    }
    ms[i] = a;
  }
  return m;
}

int sw_set_tile(int32_t G, int32_t R) {
  t_err.clear();
  if (G == 0) {
    g.force_G = g.force_R = 0;
    return SW_OK;
  }
  if ((find_tile_mode(G, R, 0) < 0 || find_tile_mode(G, R, 3) < 0) && find_tile_mode(G, R, 0, 1) < 0 &&
      find_tile_mode(G, R, 1) < 0)
    return fail(SW_EINVAL, "tile not compiled");
  g.force_G = G;
  g.force_R = R;
  return SW_OK;
}

int sw_tile_supported(int32_t G, int32_t R) {
  return (find_tile_mode(G, R, 0) >= 0 ? 1 : 0) | (find_tile_mode(G, R, 0, 1) >= 0 ? 2 : 0) |
         (find_tile_mode(G, R, 1) >= 0 ? 4 : 0);
}

int sw_set_rows_mode(int32_t mode) {
  t_err.clear();
  if (mode < -1 || mode > 1) return fail(SW_EINVAL, "mode must be -1, 0 or 1");
  g.rows_mode = mode;
  return SW_OK;
}

int sw_set_profile(int32_t mode) {
  t_err.clear();
  if (mode < 0 || mode > 2) return fail(SW_EINVAL, "mode must be 0, 1 or 2");
  if (mode == 2 && !kBiased) return fail(SW_EINVAL, "the score profile needs the biased arithmetic build");
  g.prof_mode = mode;
  return SW_OK;
}

int sw_set_latency_mode(int32_t mode) {
  t_err.clear();
  if (mode < -1 || mode > 1) return fail(SW_EINVAL, "mode must be -1, 0 or 1");
  g.lat_mode = mode;
  return SW_OK;
}

int sw_set_wave(int32_t mode) {
  t_err.clear();
  if (mode < -1 || mode > 1) return fail(SW_EINVAL, "mode must be -1, 0 or 1");
  g.wave_mode = mode;
  return SW_OK;
}

int sw_search_batch_dev(const uint8_t *queries, const int64_t *qoffsets, int32_t nq, const int8_t *matrix,
                        int32_t gap_open, int32_t gap_extend, int32_t *d_scores, void *cuda_stream) {
  t_err.clear();
  if (!g.loaded) return fail(SW_ENODB, "no database loaded");
  if (!d_scores) return fail(SW_EINVAL, "d_scores is NULL");
  return batch_impl(queries, qoffsets, nq, matrix, gap_open, gap_extend, d_scores, (cudaStream_t)cuda_stream);
}

int sw_search_batch(const uint8_t *queries, const int64_t *qoffsets, int32_t nq, const int8_t *matrix,
                    int32_t gap_open, int32_t gap_extend, int32_t *scores_out) {
  t_err.clear();
  if (!g.loaded) return fail(SW_ENODB, "no database loaded");
  if (!scores_out) return fail(SW_EINVAL, "scores_out is NULL");
  if (nq < 1) return fail(SW_EINVAL, "nq must be >= 1");
  CUDA_TRY(g.bscores.ensure((size_t)nq * g.count));
  int rc = batch_impl(queries, qoffsets, nq, matrix, gap_open, gap_extend, g.bscores.p, g.stream);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(scores_out, g.bscores.p, (size_t)nq * g.count * sizeof(int32_t), cudaMemcpyDeviceToHost,
                           g.stream));
  CUDA_TRY(cudaStreamSynchronize(g.stream));
  return SW_OK;
}

}  // extern "C"
