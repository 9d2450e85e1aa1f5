// Internal definitions shared by the host preprocessor (prep.cpp), the
// kernels (kernels.cu) and the C-ABI (api.cu).  Not part of the public ABI.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace swdb {

// Letters of the stream alphabet: 24 residue codes (SW_ALPHA), then two
// separator letters used to concatenate many database sequences into one
// lane stream:
//   END  closes a sequence: substitution -32768 in every row and the gap
//        penalties of the column forced to 32767, which zeroes E and F; the
//        lane's running score S is emitted down the group and reset.
//   NUL  follows END (and pads streams): substitution -32768, penalties
//        32767; after it H, E and F are all 0, i.e. the column-0 boundary of
//        PAPER.md:66 for the next sequence.
constexpr int kAlpha = 24;
constexpr int kEnd = 24;
constexpr int kNul = 25;
constexpr int kNL = 26;             // letters in the query profile / descriptor table
constexpr int kDescBytes = 16;      // bytes per descriptor table entry
constexpr int kColAlign = 4;        // item column counts are multiples of this
// Columns of NUL padding after every item in the stream image (and before the
// first): lets lane 0 prefetch past an item's end and lane G-1 store its
// pipeline-fill columns without bounds predicates.  >= (32 - 1) + 2U + 1;
// a multiple of 4.
constexpr int kItemPad = 40;

// Column word of the s16x2 stream: byte offset of the descriptor of the
// letter pair (cA, cB) = (cA * kNL + cB) * kDescBytes.  cA is the low 16-bit
// lane ("half A"), cB the high lane ("half B").  The host image (and the
// out-of-core chunks on the host link) hold 16 bits per column, 1 B per
// residue; the device image the same offsets as 32-bit words (expanded on
// upload: the pass kernel's 16-bit-load variant measured 1.6% slower on the
// bench tile).
static_assert(kNL * kNL * kDescBytes <= 65536, "column words are 16-bit");
inline uint16_t column_word(int cA, int cB) { return (uint16_t)((cA * kNL + cB) * kDescBytes); }

// A work item: two lane streams ("halves") of equal column count, each the
// concatenation [seq, END, NUL, seq, END, NUL, ...] padded with NUL.
struct Item {
  int64_t col_begin;  // first column in the stream image
  int32_t ncols;      // columns (multiple of kColAlign)
  int32_t seqA;       // first slot of half A's sequences in the slot array
  int32_t seqB;       // first slot of half B's sequences
  int32_t nA;         // sequences in half A
  int32_t nB;         // sequences in half B
  int32_t pad;
};
static_assert(sizeof(Item) == 32, "Item layout");

struct HostImage {
  std::vector<uint16_t> stream;   // column words, total_cols
  std::vector<Item> items;        // sorted by ncols descending (claim order)
  std::vector<int32_t> slots;     // slot -> original sequence index
  std::vector<int64_t> endcol;    // per original sequence: 2 * (END column) + half (0 = A, 1 = B)
  std::vector<int32_t> item_of;   // per original sequence: its work item
  int64_t total_cols = 0;
  int64_t max_len = 0;
  int32_t n_long_items = 0;       // leading items holding one long sequence per half (rows mode)
};

// Pre-processing stage: validated input -> stream image.
// target_groups: number of concurrently running lane groups to size items for.
// Returns 0 or -1 (err set).
// single = false: two sequences per column (halves A/B, one query);
// single = true: one sequence per column in both halves (query pairs).
// item_cap > 0: upper bound on the columns of a work item (streamed databases:
// a chunk is processed per launch and must hold several items per group).
// long_min > 0 (sequence-pair image): sequences of >= long_min residues get
// items of one sequence per half, first in the claim order (n_long_items).
int build_image(const uint8_t *residues, const int64_t *offsets, int64_t count,
                int64_t target_groups, bool single, HostImage &out, std::string &err, int64_t item_cap = 0,
                int64_t long_min = 0);

// Validation of the raw database (codes < 24, offsets monotone).
int validate_db(const uint8_t *residues, const int64_t *offsets, int64_t count, std::string &err);

}  // namespace swdb
