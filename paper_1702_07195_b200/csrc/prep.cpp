// Database pre-processor (host C++): "database sequences are
// pre-processed to allow subsequent parallel computation" and PAPER.md:114
// "database sequences are sorted by their lengths ... and padded with dummy
// symbols.  This is done to favor memory pattern access and minimize workload
// imbalances".
//
// B200 design: instead of padding every group of L
// sequences to its longest member, each s16x2 lane half is a *stream* of
// whole sequences separated by two separator columns (END, NUL); a work item
// is a pair of such streams of equal length.  Items are filled
// longest-sequence-first with a two-pointer pass over the length-sorted order
// (longest remaining first, then shortest remaining to fill the tail), so the
// padding per item is below the length of the shortest remaining sequence,
// and item capacities shrink geometrically ("guided") so the dynamic
// longest-first claim ("dynamically distributed ... as soon as
// the threads become idle") ends with small items.
#include <cstdlib>
#include "swdb_internal.h"

#include <algorithm>
#include <cstring>
#include <numeric>
#include <thread>

namespace swdb {

int validate_db(const uint8_t *residues, const int64_t *offsets, int64_t count, std::string &err) {
  if (!offsets) { err = "offsets is NULL"; return -1; }
  if (count < 1) { err = "count must be >= 1"; return -1; }
  if (count >= (int64_t(1) << 31) - 1) { err = "count must be < 2^31 - 1"; return -1; }
  if (offsets[0] != 0) { err = "offsets[0] must be 0"; return -1; }
  for (int64_t i = 0; i < count; ++i)
    if (offsets[i + 1] < offsets[i]) {
      err = "offsets must be non-decreasing (at index " + std::to_string(i) + ")";
      return -1;
    }
  const int64_t total = offsets[count];
  if (total > 0 && !residues) { err = "residues is NULL"; return -1; }
  if (total >= (int64_t(1) << 40)) { err = "database too large"; return -1; }
  // residue codes < 24, checked in parallel chunks
  unsigned nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::vector<int64_t> bad(nth, -1);
  std::vector<std::thread> th;
  const int64_t chunk = (total + nth - 1) / nth;
  for (unsigned k = 0; k < nth; ++k)
    th.emplace_back([&, k] {
      const int64_t b = k * chunk, e = std::min(total, b + chunk);
      for (int64_t i = b; i < e; ++i)
        if (residues[i] >= kAlpha) { bad[k] = i; return; }
    });
  for (auto &t : th) t.join();
  for (unsigned k = 0; k < nth; ++k)
    if (bad[k] >= 0) {
      err = "residue code >= 24 at position " + std::to_string(bad[k]);
      return -1;
    }
  return 0;
}

namespace {
inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }
}  // namespace

int build_image(const uint8_t *residues, const int64_t *offsets, int64_t count,
                int64_t target_groups, bool single, HostImage &out, std::string &err, int64_t item_cap,
                int64_t long_min) {
  out = HostImage();
  std::vector<int64_t> len(count);
  int64_t total_stream = 0;
  for (int64_t i = 0; i < count; ++i) {
    len[i] = offsets[i + 1] - offsets[i];
    out.max_len = std::max(out.max_len, len[i]);
    total_stream += len[i] + 2;  // residues, END, NUL
  }
  // Stable sort by length, descending (ties by original index).  The paper
  // sorts ascending and processes groups in that order; we claim longest
  // first to bound the tail of the dynamic schedule.
  std::vector<int32_t> order(count);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int32_t a, int32_t b) { return len[a] > len[b]; });

  if (target_groups < 1) target_groups = 1;
  // Guided item sizes: capacity = remaining columns / (item_div * groups),
  // clipped to [256, item_max].  Measured on one B200: fewer,
  // longer items pay the group's pipeline fill/drain less often, but the first
  // items must stay below one group's share of the work for the 8-lane tiles
  // (twice as many groups as target_groups): item_div 1 is 0.2-0.3% faster on
  // cfg1/cfg2/cfg4 than 2 but loses 35% with 8-lane tiles on cfg1; item_div 2
  // and item_max 16384 beat 3 / 8192 by 0.1-0.5%; the floor 256 beats
  // 128/512/1024.  SW_ITEM_DIV / SW_ITEM_MAX / SW_ITEM_MIN override them for
  // experiments.
  double item_div = 2.0;
  if (const char *e = std::getenv("SW_ITEM_DIV")) item_div = std::max(0.25, std::atof(e));
  int64_t item_max = 16384, item_min = 256;
  if (const char *e = std::getenv("SW_ITEM_MAX")) item_max = std::max<int64_t>(256, std::atoll(e));
  if (const char *e = std::getenv("SW_ITEM_MIN")) item_min = std::max<int64_t>(16, std::atoll(e));
  // a streamed database processes one chunk per launch: its items must stay
  // small enough that every chunk keeps every group busy (item_cap)
  if (item_cap > 0) item_max = std::max(item_min, std::min(item_max, item_cap));
  // columns still to place (pair columns: two sequences per column)
  int64_t remaining = single ? total_stream : (total_stream + 1) / 2;
  int64_t lo = 0, hi = count - 1;
  std::vector<int32_t> halfA, halfB;
  struct Tmp { int64_t ncols; int64_t slot0; int32_t nA, nB; };
  std::vector<Tmp> tmp;
  out.slots.reserve(count);
  // Long sequences (>= long_min residues, sequence-pair image only): items of
  // exactly one sequence per half, consecutive in length order, first in the
  // claim order.  They are the rows-mode pairs: a search may
  // score them with the sequence along the rows and skip their items.
  if (!single && long_min > 0) {
    while (lo <= hi && len[order[lo]] >= long_min) {
      halfA.assign(1, order[lo++]);
      halfB.clear();
      if (lo <= hi && len[order[lo]] >= long_min) halfB.push_back(order[lo++]);
      const int64_t lA = len[halfA[0]] + 2, lB = halfB.empty() ? 0 : len[halfB[0]] + 2;
      const int64_t ncols = round_up(std::max(lA, lB), kColAlign);
      tmp.push_back(Tmp{ncols, (int64_t)out.slots.size(), 1, (int32_t)halfB.size()});
      for (int32_t s : halfA) out.slots.push_back(s);
      for (int32_t s : halfB) out.slots.push_back(s);
      remaining = std::max<int64_t>(0, remaining - (lA + lB + 1) / 2);
      ++out.n_long_items;
    }
  }
  while (lo <= hi) {
    int64_t cap = (int64_t)((double)remaining / ((double)target_groups * item_div));
    cap = std::max<int64_t>(item_min, std::min<int64_t>(item_max, cap));
    halfA.clear();
    halfB.clear();
    int64_t lA = 0, lB = 0;
    {
      int32_t s = order[lo++];
      halfA.push_back(s);
      lA = len[s] + 2;
      cap = std::max(cap, lA);
    }
    for (;;) {
      const bool toA = single || lA <= lB;
      int64_t &l = toA ? lA : lB;
      std::vector<int32_t> &h = toA ? halfA : halfB;
      if (lo <= hi && l + len[order[lo]] + 2 <= cap) {
        int32_t s = order[lo++];
        h.push_back(s);
        l += len[s] + 2;
      } else if (lo <= hi && l + len[order[hi]] + 2 <= cap) {
        int32_t s = order[hi--];
        h.push_back(s);
        l += len[s] + 2;
      } else {
        break;
      }
    }
    const int64_t ncols = round_up(std::max(lA, lB), kColAlign);
    Tmp t{ncols, (int64_t)out.slots.size(), (int32_t)halfA.size(), (int32_t)halfB.size()};
    for (int32_t s : halfA) out.slots.push_back(s);
    for (int32_t s : halfB) out.slots.push_back(s);
    tmp.push_back(t);
    remaining -= single ? lA : (lA + lB + 1) / 2;
    if (remaining < 0) remaining = 0;
  }
  // claim order: longest item first (stable)
  std::vector<int32_t> iorder(tmp.size());
  std::iota(iorder.begin(), iorder.end(), 0);
  // the long items stay first (and in length order); the rest longest first
  std::stable_sort(iorder.begin() + out.n_long_items, iorder.end(),
                   [&](int32_t a, int32_t b) { return tmp[a].ncols > tmp[b].ncols; });
  int64_t col = kItemPad;
  out.items.resize(tmp.size());
  for (size_t k = 0; k < iorder.size(); ++k) {
    const Tmp &t = tmp[iorder[k]];
    Item &it = out.items[k];
    it.col_begin = col;
    it.ncols = (int32_t)t.ncols;
    it.seqA = (int32_t)t.slot0;
    it.nA = t.nA;
    it.seqB = (int32_t)(t.slot0 + t.nA);
    it.nB = t.nB;
    it.pad = 0;
    col += t.ncols + kItemPad;
    if (t.ncols >= (int64_t(1) << 31)) { err = "sequence too long"; return -1; }
  }
  out.total_cols = col;
  // Write the stream: column word per pair column.
  out.stream.assign((size_t)col, column_word(kNul, kNul));
  out.endcol.assign((size_t)count, -1);
  out.item_of.assign((size_t)count, -1);
  // half: 0 = A (low 16 bits), 1 = B (high), 2 = both (single-sequence image)
  auto write_half = [&](const Item &it, int32_t item, int32_t slot0, int32_t n, int half) {
    int64_t c = it.col_begin;
    auto put = [&](int64_t col, int letter) {
      uint32_t w = out.stream[col];
      int cA = (int)(w / kDescBytes) / kNL, cB = (int)(w / kDescBytes) % kNL;
      if (half != 1) cA = letter;
      if (half != 0) cB = letter;
      out.stream[col] = column_word(cA, cB);
    };
    for (int32_t k = 0; k < n; ++k) {
      const int32_t s = out.slots[slot0 + k];
      const uint8_t *r = residues + offsets[s];
      for (int64_t j = 0; j < len[s]; ++j, ++c) put(c, r[j]);
      out.endcol[s] = 2 * c + (half == 1 ? 1 : 0);   // the END column of sequence s
      out.item_of[s] = item;
      put(c++, kEnd);
      put(c++, kNul);
    }
  };
  {
    unsigned nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    const size_t ni = out.items.size();
    for (unsigned k = 0; k < nth; ++k)
      th.emplace_back([&, k] {
        for (size_t i = k; i < ni; i += nth) {
          const Item &it = out.items[i];
          if (single) {
            write_half(it, (int32_t)i, it.seqA, it.nA, 2);
          } else {
            write_half(it, (int32_t)i, it.seqA, it.nA, 0);
            write_half(it, (int32_t)i, it.seqB, it.nB, 1);
          }
        }
      });
    for (auto &t : th) t.join();
  }
  return 0;
}

}  // namespace swdb
