/*
 * swdb.h -- C-ABI of the B200-native inter-task Smith-Waterman database search.
 *
 * The problem, as the paper states it (Section 4):
 *   1. "Pre-processing stage: database sequences are pre-processed to allow
 *      subsequent parallel computation."                       -> sw_db_load
 *   2. "SW stage: alignments are carried out."                 -> sw_search
 *   3. "Sorting stage: alignment scores are sorted in descending order."
 *                                                              -> sw_topk
 * Each alignment score is the Smith-Waterman local alignment score with
 * affine gaps of PAPER.md:49-66 (Eqs. 1-3): the maximum over the H matrix of
 *   H_ij = max{0, H_{i-1,j-1} + SM(q_i, d_j), E_ij, F_ij}
 *   E_ij = max{H_{i,j-1} - Goe, E_{i,j-1} - Ge}
 *   F_ij = max{H_{i-1,j} - Goe, F_{i-1,j} - Ge}
 * with H, E, F = 0 when i = 0 or j = 0, Goe = gap_open + gap_extend and
 * Ge = gap_extend, so a gap of length k costs gap_open + k*gap_extend
 * (PAPER.md:66, 179).  The query is S1 (rows i), the database sequence S2
 * (columns j).
 *
 * Conventions shared by every entry point
 *   - Residue codes are uint8 in 0..23, alphabet "ARNDCQEGHILKMFPSTWYVBZX*"
 *     (NCBI matrix order).  Codes >= 24 are rejected (SW_EINVAL).
 *   - The substitution matrix is int8[24*24], row-major, indexed
 *     matrix[query_code*24 + db_code].  It need not be symmetric.
 *   - All functions return SW_OK (0) or a negative status; no C++ exception
 *     or abort crosses this boundary.  sw_last_error() returns a message for
 *     the most recent failing call of the calling thread.
 *   - One database per process, held on the CUDA device that is current for
 *     the calling thread at sw_db_load time.  Multi-GPU = one process per GPU,
 *     each loading its own shard (the Python harness shards and merges).
 *   - The library is not reentrant: calls must be serialised by the caller.
 *     Searches may be enqueued on different streams: each search's device
 *     work waits (cudaStreamWaitEvent) for the previous search's work, whose
 *     per-search scratch buffers it reuses, so no synchronisation is needed
 *     between them.
 *   - Host pointers are only read during the call (inputs are copied); the
 *     caller keeps ownership of every buffer it passes.
 */
#ifndef SWDB_H
#define SWDB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SW_OK = 0,
  SW_EINVAL = -1,  /* bad argument: NULL pointer, bad size, code >= 24, ... */
  SW_ENOMEM = -2,  /* host or device allocation failed                    */
  SW_ECUDA = -3,   /* CUDA runtime error (no device, launch failure, ...)  */
  SW_ENODB = -4,   /* sw_search* called before a successful sw_db_load     */
  SW_ESTATE = -5   /* sw_topk called before a successful search            */
};

#define SW_ALPHA 24

/*
 * sw_db_load -- pre-processing stage.
 *   residues : host, uint8[offsets[count]]; sequence i is
 *              residues[offsets[i] .. offsets[i+1]).  Codes < 24.
 *   offsets  : host, int64[count+1], offsets[0] == 0, non-decreasing.
 *              Zero-length sequences are accepted (they score 0).
 *   count    : number of sequences, >= 1, < 2^31.
 * Builds the device-resident, length-balanced, residue-interleaved stream
 * image on the current CUDA device.  Replaces any
 * previously loaded database.  On SW_EINVAL (validation, before any device
 * work) the previous database is kept; the previous database's device memory
 * is released before the new one is uploaded (so a database of nearly the
 * device's size can replace another), hence after SW_ENOMEM / SW_ECUDA no
 * database is loaded (sw_db_count() == 0).
 * Device memory: about 4 B per residue for the two stream images, 1 B per
 * residue for the plain copy, 4 B per image column for the score chain, and
 * for 32-bit re-scoring 2 x 8 B x (longest sequence + 64) per re-scoring
 * warp, capped at 4 GiB (fewer re-scoring warps for very long sequences).
 * Not part of the timed search.
 * Errors: SW_EINVAL (NULL, count < 1, bad offsets, code >= 24),
 *         SW_ENOMEM, SW_ECUDA.
 */
int sw_db_load(const uint8_t *residues, const int64_t *offsets, int64_t count);

/*
 * sw_db_load_streamed -- pre-processing stage for a database that need not fit
 * in device memory ("larger genomic
 * databases that do not fit in MCDRAM").  Same arguments and validation as
 * sw_db_load, plus
 *   chunk_bytes : >= 1, the device memory budget of one chunk of the stream
 *                 image (two chunk buffers are allocated).
 * The sequence-pair image is kept in pinned HOST memory (16-bit column words,
 * 1 B per residue on the link) and split into chunks of consecutive work
 * items (as few chunks as chunk_bytes allows, then equal in size: the column
 * limit is lowered to the smallest one giving that count); every search
 * copies chunk k+1 host->device on a separate stream while
 * the pass kernels run on chunk k (expanded to 32-bit words on the device),
 * and at its end copies the next search's chunk 0 while its last chunk runs.
 * Device memory: 2 x chunk_bytes of 32-bit words + 2 x chunk_bytes / 2 of
 * 16-bit copies, plus the per-column score chain of one chunk.  Residues for 32-bit
 * re-scoring are read from mapped host memory.  sw_search / sw_search_dev /
 * sw_topk work unchanged; sw_search_batch(_dev) returns SW_EINVAL (it needs a
 * resident database).  Per-sequence arrays (scores, offsets) stay on the
 * device.
 */
int sw_db_load_streamed(const uint8_t *residues, const int64_t *offsets, int64_t count, int64_t chunk_bytes);

/* Number of chunks of a streamed database (0 for a resident one). */
int64_t sw_db_chunks(void);

/* Columns of a streamed database's resident head (0: none, or a resident
 * database).  The head is the run of leading -- longest -- work items within a
 * quarter of chunk_bytes (at least the first item), kept on the device when
 * more than one chunk of items follows it: every search scores it on a second,
 * high-priority stream beside the streamed chunks, so that a very long
 * sequence's chain of column steps is hidden by the whole search instead of
 * bounding the chunk that would hold it ("minimize workload
 * imbalances").  It is not counted by sw_db_chunks and costs
 * 8 B per column of device memory (+ 16 B per column for multi-pass queries).
 * SWDB_STREAM_HEAD=0 in the environment at load time turns it off. */
int64_t sw_db_head_columns(void);

/* Frees the database and all device buffers.  Safe to call at any time. */
void sw_db_free(void);

/* Number of sequences / total residues of the loaded database (0 if none). */
int64_t sw_db_count(void);
int64_t sw_db_residues(void);

/*
 * sw_search -- SW stage, synchronous, host buffers.
 *   query      : host, uint8[qlen], codes < 24, qlen >= 1.
 *   matrix     : host, int8[24*24], matrix[q*24 + d].
 *   gap_open   : >= 0.   gap_extend : >= 0.   gap_open + gap_extend < 2^30.
 *   scores_out : host, int32[count]; scores_out[i] = optimal local alignment
 *                score of the query against database sequence i (original
 *                load order), exact (saturated 16-bit lanes are re-scored in
 *                32-bit).
 * Copies the query and matrix to the device, runs the kernels on the
 * library's stream and copies the scores back before returning.
 * Errors: SW_ENODB, SW_EINVAL (NULL, qlen < 1, code >= 24, negative or too
 *         large penalties, max|matrix| * min(qlen, longest) >= 2^30),
 *         SW_ENOMEM, SW_ECUDA.
 */
int sw_search(const uint8_t *query, int32_t qlen, const int8_t *matrix, int32_t gap_open,
              int32_t gap_extend, int32_t *scores_out);

/*
 * sw_search_dev -- same as sw_search but stream-ordered and device-resident:
 *   query, matrix : host pointers, read during the call (copied into a pinned
 *                   staging slot and sent to the device in one copy together
 *                   with the search's item cursors; the host does not wait
 *                   for the stream unless all 4 staging slots are in flight).
 *   d_scores      : DEVICE pointer, int32[count], written in original order.
 *   cuda_stream   : cudaStream_t to order the work on (NULL = legacy default).
 * Returns once all work is enqueued; results are final when the stream
 * reaches them.  sw_topk after sw_search_dev reads d_scores, which must stay
 * allocated until then.
 */
int sw_search_dev(const uint8_t *query, int32_t qlen, const int8_t *matrix, int32_t gap_open,
                  int32_t gap_extend, int32_t *d_scores, void *cuda_stream);

/*
 * sw_search_batch -- several queries against the database (SW stage for each).
 *   queries   : host, uint8, the nq queries concatenated; query k is
 *               queries[qoffsets[k] .. qoffsets[k+1]).
 *   qoffsets  : host, int64[nq+1], qoffsets[0] == 0, every query length >= 1.
 *   nq        : >= 1.
 *   matrix, gap_open, gap_extend : as for sw_search.
 *   scores_out: host, int32[nq * count]; scores_out[k*count + i] = score of
 *               query k against database sequence i.
 * Queries are sorted by length and paired: each pair is scored in ONE pass
 * over a one-sequence-per-column image, query 1 in the low and query 2 in
 * the high 16-bit half of every register (multi-query packing, SURVEY.md
 * 8(f) NEXT-2); results are identical to nq calls of sw_search.
 * sw_topk afterwards ranks query 0.  Errors as for sw_search.
 */
int sw_search_batch(const uint8_t *queries, const int64_t *qoffsets, int32_t nq, const int8_t *matrix,
                    int32_t gap_open, int32_t gap_extend, int32_t *scores_out);

/* Stream-ordered batch search into a DEVICE array d_scores[nq * count]. */
int sw_search_batch_dev(const uint8_t *queries, const int64_t *qoffsets, int32_t nq, const int8_t *matrix,
                        int32_t gap_open, int32_t gap_extend, int32_t *d_scores, void *cuda_stream);

/*
 * sw_topk -- sorting stage over the last search's scores.
 *   k         : >= 0; min(k, count) results are written.
 *   idx_out   : host, int64[k]: original database indices.
 *   score_out : host, int32[k]: their scores.
 * Order: score descending, ties by ascending index (reading R5).
 * k >= count gives the complete sorted order.
 * Returns the number of results written (>= 0) or a negative status
 * (SW_EINVAL, SW_ESTATE, SW_ENOMEM, SW_ECUDA).
 */
int64_t sw_topk(int64_t k, int64_t *idx_out, int32_t *score_out);

/*
 * sw_topk_dev -- sorting stage on caller-provided DEVICE arrays (used to merge
 * per-GPU candidates after the NCCL gather).
 *   d_scores : device int32[n];  d_index : device int64[n] (distinct indices,
 *              0 <= index < 2^32), or NULL meaning index = position.
 *   k        : results wanted; d_idx_out int64[min(k,n)], d_score_out
 *              int32[min(k,n)] are DEVICE pointers.
 *   cuda_stream : stream to enqueue on (NULL = legacy default).  Stream-
 *              ordered: returns once the work is enqueued; the outputs are
 *              ready when the stream reaches this point.  Calls are ordered
 *              among themselves whatever their streams (shared scratch).
 * Returns min(k, n) or a negative status.
 */
int64_t sw_topk_dev(const int32_t *d_scores, const int64_t *d_index, int64_t n, int64_t k,
                    int64_t *d_idx_out, int32_t *d_score_out, void *cuda_stream);

/*
 * sw_scatter_dev -- sorting stage, multi-GPU assembly ("alignment
 * scores are sorted"): rank 0 puts the score vectors gathered
 * from every rank's database shard back into the original database order.
 *   d_src     : device int32[n], the gathered per-rank score vectors (padded).
 *   d_index   : device int64[n], original database index of each entry, or a
 *               negative value for a padding slot (skipped).
 *   n         : >= 0 entries.
 *   d_dst     : device int32[dst_count]; d_dst[d_index[i]] = d_src[i] for
 *               every i with 0 <= d_index[i] < dst_count.  Entries not named
 *               by any index are left unchanged.  Indices must be distinct
 *               (otherwise which of the duplicates lands is unspecified).
 *   cuda_stream : stream to enqueue on (NULL = legacy default); asynchronous.
 * Returns SW_OK, SW_EINVAL (NULL pointer with n > 0, n < 0, dst_count < 0) or
 * SW_ECUDA.
 */
int sw_scatter_dev(const int32_t *d_src, const int64_t *d_index, int64_t n, int32_t *d_dst, int64_t dst_count,
                   void *cuda_stream);

/*
 * Statistics of the last search (for the benchmark report):
 *   stats[0] = rows per query pass (G*R), stats[1] = passes,
 *   stats[2] = G (lanes per group), stats[3] = R (rows per lane),
 *   stats[4] = sequences flagged by the 16-bit saturation test and re-scored
 *              in 32 bit, stats[5] = cells re-scored in 32 bit,
 *   stats[6] = pair-columns streamed per pass, stats[7] = items,
 *   stats[8] = the 16-bit flag threshold T in score units: a sequence is
 *              re-scored in 32 bit iff its 16-bit score is >= T, and every
 *              sequence whose exact score is >= T is (R7),
 *   stats[9] = cell arithmetic of the 16-bit kernel: 1 = biased (4.5 ALU +
 *              2 FMA instructions per pair of cells), 0 = relu form (5.5 ALU
 *              + 1 FMA),
 *   stats[10] = 1 if the last search ran as a cross-pass wavefront,
 *   stats[11] = 1 if it ran a latency tile (sw_set_latency_mode),
 *   stats[12] = substitution scores of the 16-bit kernel: 1 = query profile,
 *              2 = score profile (sw_set_profile),
 *   stats[13] = long-sequence pairs scored in rows mode (sw_set_rows_mode).
 * Returns the number of entries written (<= n).
 */
int sw_last_stats(int64_t *stats, int n);

/*
 * Device timing of the last search (or of all searches of the last batch),
 * from CUDA events recorded on the search stream (synchronises with it):
 *   ms[0] = s16x2 pass kernels (sum of the pass-kernel launches),
 *   ms[1] = whole search on the device (query-profile build .. end of the
 *           32-bit re-scoring kernel).
 * Returns the number of entries written (<= n) or a negative status.
 */
int sw_last_timing(float *ms, int n);

/*
 * sw_timing_history -- the s16x2 pass-kernel device time (ms, sum of its
 * pass-kernel launches, from the same CUDA events as sw_last_timing) of each
 * of the last n searches, a batch counting as one search, oldest first, so
 * that a caller can time a run of back-to-back searches without a
 * synchronisation per search.  At most the last 64 searches are kept (their
 * events are reused after that).  Synchronises with the last search.
 *   ms : host, float[n], written.
 * Returns the number of entries written (min(n, searches kept)) or a
 * negative status (SW_EINVAL: NULL or n < 0; SW_ESTATE: no search yet).
 */
int sw_timing_history(float *ms, int n);

/*
 * sw_set_tile -- override the (G, R) tile choice for subsequent searches
 * (tests of tile invariance).  G in {8,16,32}; R must be
 * one of the compiled row counts (sw_tile_supported).  G = 0 restores the
 * automatic choice.  Returns SW_OK or SW_EINVAL.
 */
int sw_set_tile(int32_t G, int32_t R);
/* Bit 0: (G, R) is a compiled throughput tile; bit 1: a compiled latency
 * tile; bit 2: a compiled score-profile tile. */
int sw_tile_supported(int32_t G, int32_t R);

/*
 * sw_set_profile -- where the 16-bit kernel takes its substitution scores
 * from (Section 4.3 "Substitution scores"):
 *   1: query profile QP[letter][query row], built per query;
 *      a lane reads 4 rows per 16-B load for each of the column's two
 *      database letters and packs the two halves with one IMAD per row;
 *   2: score profile SP[database letter pair][query letter],
 *      one word SM(c, dB) * 65536 + SM(c, dA) per pair and query letter,
 *      built per scoring matrix (not per database group: on B200 every pair
 *      fits in shared memory); a lane reads one word per row at its row's
 *      query letter (no packing);
 *   0 (default): chosen by query length from the measured QP/SP crossover
 *      (DESIGN.md 4.6).
 * Single-query searches only (query pairs always use their paired profile).
 * Returns SW_OK or SW_EINVAL.
 */
int sw_set_profile(int32_t mode);

/*
 * sw_set_rows_mode -- rows mode for the long sequences of a database
 * (intra-task parallelism for long alignments).
 * sw_db_load gives every sequence longer than 4x the average columns per
 * lane group (at least 512 residues) a work item of its own, paired with the
 * next long one.  In rows mode those pairs are scored with the database
 * sequence along the rows and the query as the column stream (the same
 * recurrence on the transposed matrix; scores are identical), one CTA per
 * pair with its 8 warps on consecutive passes over the sequence (hand-over
 * through shared memory), so the pair's critical path is about
 * ceil(n / 2048) x (m + 31) + 7 x 44 column steps instead of n.  mode 1:
 * whenever possible; 0 (default) and -1: never -- measured slower than the
 * ordinary path on every database tried.  Resident single-query
 * searches whose pass kernel makes one pass, without the cross-pass
 * wavefront, queries of at most 8,188 residues.
 * Returns SW_OK or SW_EINVAL.
 */
int sw_set_rows_mode(int32_t mode);



/*
 * sw_set_latency_mode -- latency tiles for searches whose time is one long
 * work item's critical path rather than the total work (small databases with
 * a long sequence): a small number of rows per lane (shorter
 * per-column step of a lane group) on one 256-thread CTA per SM.  mode 0
 * (default): chosen by the pass time model; 1: always (the forced tile if it
 * is a latency tile, else the model's best latency tile); -1: never.
 * Single-query searches of a resident database without the cross-pass
 * wavefront only.  Returns SW_OK or SW_EINVAL.
 */
int sw_set_latency_mode(int32_t mode);

/*
 * sw_set_wave -- cross-pass wavefront for multi-pass single-query searches of
 * a resident database: one launch runs every query pass, an
 * item's pass p trailing its pass p-1 through the boundary buffer, so several
 * lane groups work on one long sequence at once (intra-task parallelism,
 * PAPER.md:32).  mode 0 (default): used when a pass has fewer than half as many
 * work items as lane groups and the query makes at least 4 passes of the 32x8
 * tile (or 2 of the 32x16 tile with enough units); with few units only as many
 * lane groups per CTA claim as spreads them over all SMs; 1: always (when the
 * query needs more than one pass); -1: never.
 * In wavefront mode flagged sequences are re-scored in 32 bit from row 0.
 * Returns SW_OK or SW_EINVAL.
 */
int sw_set_wave(int32_t mode);

/* Number of CUDA kernels the library has launched since it was loaded (every
 * entry point counts its own launches; for the benchmark's launch report). */
int64_t sw_launch_count(void);

/* Message for the most recent failing call on this thread ("" if none). */
const char *sw_last_error(void);

/* Library version string. */
const char *sw_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SWDB_H */
