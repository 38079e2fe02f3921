// Host plan builder: block grid, pattern masks, head grouping and the
// kernel's work schedule.  Everything integer here is bit-exact with the
// reference (svdit 0.1.0):
//   layout.py:26-80    TokenLayout validation, total_tokens, frame_of
//   layout.py:135-158  block_grid (bounds / has_text / mixed / frame_index)
//   patterns.py:176-181 frame_period (Python round(): half-to-even)
//   patterns.py:219-259 build_mask (5 modes, forced rows/cols, empty-row error)
//   attention.py:164-183 group_heads (first-occurrence order, ascending heads,
//                         keyed on full PatternSpec equality)
// and then lowers each group's block mask to the kernel schedule: 64-token
// query segments clustered four to a CTA, each cluster with one ascending
// list of 128-key tiles (pairs of key segments) plus per-tile activity bits.
#include <algorithm>
#include <functional>
#include <queue>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>

#include "svd_plan.h"

namespace svd {

static thread_local std::string g_last_error = "";

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}

bool NormSpec::operator<(const NormSpec& o) const {
  auto key = [](const NormSpec& s) {
    return std::make_tuple(s.mode, s.halfwidth, s.period, s.md_halfwidth, s.stripe_count,
                           s.include_diagonal, s.stripes_none, s.stripes);
  };
  return key(*this) < key(o);
}

bool NormSpec::operator==(const NormSpec& o) const { return !(*this < o) && !(o < *this); }

// ---------------------------------------------------------------- layout
// layout.py:33-43 TokenLayout.__post_init__
static int check_layout(const svd_layout* L) {
  if (!L) return fail(SVD_ERR_CONFIG, "layout is NULL");
  if (L->text_tokens < 0)
    return fail(SVD_ERR_CONFIG, "text_tokens must be >= 0, got " + std::to_string(L->text_tokens));
  if (L->frames < 0 || L->tokens_per_frame < 0)
    return fail(SVD_ERR_CONFIG, "frames and tokens_per_frame must be >= 0");
  if (L->frames > 0 && L->tokens_per_frame == 0)
    return fail(SVD_ERR_CONFIG, "frames > 0 requires tokens_per_frame > 0");
  if (L->block_size < 1)
    return fail(SVD_ERR_CONFIG, "block_size must be >= 1, got " + std::to_string(L->block_size));
  if (L->text_tokens + L->frames * L->tokens_per_frame < 1)
    return fail(SVD_ERR_CONFIG, "layout has no tokens");
  return SVD_OK;
}

// layout.py:57-63 frame_of (token already range-checked by callers)
static inline int64_t frame_of(const svd_layout* L, int64_t token) {
  if (token < L->text_tokens) return -1;
  return (token - L->text_tokens) / L->tokens_per_frame;
}

// layout.py:135-158 block_grid
static int make_grid(const svd_layout* L, Grid* g) {
  int st = check_layout(L);
  if (st) return st;
  const int64_t n = L->text_tokens + L->frames * L->tokens_per_frame;
  const int64_t size = L->block_size;
  const int64_t nb = (n + size - 1) / size;
  g->n = n;
  g->nb = nb;
  g->bs = size;
  g->bounds.resize(nb + 1);
  for (int64_t b = 0; b <= nb; ++b) g->bounds[b] = std::min(b * size, n);
  g->has_text.assign(nb, 0);
  g->mixed.assign(nb, 0);
  g->frame_index.assign(nb, -1);
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t t0 = g->bounds[b], t1 = g->bounds[b + 1];
    g->has_text[b] = t0 < L->text_tokens;
    const int64_t first_video = std::max(t0, L->text_tokens);
    if (first_video < t1) {
      g->frame_index[b] = frame_of(L, first_video);
      const bool straddles = t0 < L->text_tokens;
      const bool spans = frame_of(L, t1 - 1) != g->frame_index[b];
      g->mixed[b] = straddles || spans;
    }
  }
  return SVD_OK;
}

// patterns.py:176-181 frame_period: max(1, round(tpf / size)), banker's rounding
static int64_t frame_period(const svd_layout* L) {
  const double ratio = double(L->tokens_per_frame) / double(L->block_size);
  const int64_t r = int64_t(std::nearbyint(ratio));  // FE_TONEAREST = half-to-even
  return std::max<int64_t>(1, r);
}

// ---------------------------------------------------------------- specs
// patterns.py:67-75 PatternSpec.__post_init__ (validation + stripe normalisation)
static int normalise_spec(const svd_spec* s, NormSpec* out) {
  if (!s) return fail(SVD_ERR_CONFIG, "spec is NULL");
  if (s->mode < 0 || s->mode > 4)
    return fail(SVD_ERR_CONFIG, "mode code must be in 0..4, got " + std::to_string(s->mode));
  if (s->halfwidth < 0 || s->md_halfwidth < 0) return fail(SVD_ERR_CONFIG, "halfwidth must be >= 0");
  if (s->stripe_count < 1)
    return fail(SVD_ERR_CONFIG, "stripe_count must be >= 1, got " + std::to_string(s->stripe_count));
  out->mode = s->mode;
  out->halfwidth = s->halfwidth;
  out->period = s->period > 0 ? s->period : -1;
  out->md_halfwidth = s->md_halfwidth;
  out->stripe_count = s->stripe_count;
  out->include_diagonal = s->include_diagonal ? 1 : 0;
  out->stripes_none = s->n_stripes < 0;
  out->stripes.clear();
  if (!out->stripes_none) {
    if (s->n_stripes > 0 && !s->stripes) return fail(SVD_ERR_CONFIG, "stripes pointer is NULL");
    out->stripes.assign(s->stripes, s->stripes + s->n_stripes);
    std::sort(out->stripes.begin(), out->stripes.end());
    out->stripes.erase(std::unique(out->stripes.begin(), out->stripes.end()), out->stripes.end());
  }
  return SVD_OK;
}

// patterns.py:219-259 build_mask.  active must hold nb*nb bytes.
static int build_mask(const NormSpec& spec, const Grid& g, const svd_layout* L, uint8_t* active,
                      bool* is_skip) {
  const int64_t nb = g.nb;
  *is_skip = false;
  if (spec.mode == SVD_SKIP) {
    *is_skip = true;
    return SVD_OK;
  }
  if (spec.mode == SVD_FULL) {
    std::memset(active, 1, size_t(nb * nb));
    return SVD_OK;
  }
  if (spec.mode == SVD_DIAGONAL) {
    // |i - j| <= hw: a band
    const int64_t hw = spec.halfwidth;
    std::memset(active, 0, size_t(nb * nb));
    for (int64_t i = 0; i < nb; ++i) {
      const int64_t j0 = std::max<int64_t>(0, i - hw), j1 = std::min<int64_t>(nb - 1, i + hw);
      if (j0 <= j1) std::memset(active + i * nb + j0, 1, size_t(j1 - j0 + 1));
    }
  } else if (spec.mode == SVD_MULTI_DIAGONAL) {
    // f = |i - j| mod P; active when f <= hw or P - f <= hw: the pattern of
    // row i is the distance pattern of one period, repeated
    const int64_t period = spec.period > 0 ? spec.period : frame_period(L);
    const int64_t hw = spec.md_halfwidth;
    std::vector<uint8_t> by_dist(static_cast<size_t>(nb));
    for (int64_t dist = 0; dist < nb; ++dist) {
      const int64_t folded = dist % period;
      by_dist[dist] = (folded <= hw) || (period - folded <= hw);
    }
    for (int64_t i = 0; i < nb; ++i) {
      uint8_t* row = active + i * nb;
      std::reverse_copy(by_dist.begin() + 1, by_dist.begin() + i + 1, row);  // row[j] = by_dist[i - j]
      std::memcpy(row + i, by_dist.data(), size_t(nb - i));
    }
  } else {  // VERTICAL_STRIPE
    if (spec.stripes_none)
      return fail(SVD_ERR_CONFIG,
                  "vertical-stripe spec has no resolved stripe columns; pass stripes=... or let the "
                  "search pick them");
    std::memset(active, 0, size_t(nb * nb));
    for (int64_t col : spec.stripes) {
      if (!(0 <= col && col < nb))
        return fail(SVD_ERR_CONFIG, "stripe column " + std::to_string(col) + " outside grid of " +
                                        std::to_string(nb) + " blocks");
      for (int64_t i = 0; i < nb; ++i) active[i * nb + col] = 1;
    }
    if (spec.include_diagonal)
      for (int64_t i = 0; i < nb; ++i) active[i * nb + i] = 1;
  }
  // layout.py:119-122 forced = has_text | mixed; patterns.py:253-255
  for (int64_t b = 0; b < nb; ++b) {
    if (!(g.has_text[b] || g.mixed[b])) continue;
    std::memset(active + b * nb, 1, size_t(nb));
    for (int64_t i = 0; i < nb; ++i) active[i * nb + b] = 1;
  }
  // patterns.py:256-258
  for (int64_t i = 0; i < nb; ++i) {
    bool any = false;
    for (int64_t j = 0; j < nb && !any; ++j) any = active[i * nb + j];
    if (!any)
      return fail(SVD_ERR_DEGENERATE_MASK,
                  "query block " + std::to_string(i) + " has no active key blocks");
  }
  return SVD_OK;
}

// ---------------------------------------------------------------- schedule
// Segment-level key sets of one group: keyset[s] bit ks is set when any
// active (qb, kb) pair touches query segment s and key segment ks.
// fullset (FINE grids only, block_size % 64 != 0): bit ks set when EVERY
// (qb, kb) pair overlapping segments (s, ks) is active — such tiles need no
// per-element mask in the kernel.
static void segment_keysets(const Group& grp, const Grid& g, int64_t nseg,
                            std::vector<std::vector<uint64_t>>* keyset,
                            std::vector<std::vector<uint64_t>>* fullset) {
  const int64_t nb = g.nb, bs = g.bs, n = g.n;
  const int64_t words = (nseg + 63) / 64;
  keyset->assign(nseg, std::vector<uint64_t>(words, 0));
  if (bs % kSeg == 0) {
    // block-aligned segments (block_size 64, 128, ...): segment s lies in block
    // s / r and key segment ks in block ks / r — bits straight from the mask row
    const int64_t r = bs / kSeg;
    std::vector<uint64_t> bits(words);
    for (int64_t b = 0; b < nb; ++b) {
      const uint8_t* row = grp.active.data() + b * nb;
      std::fill(bits.begin(), bits.end(), 0);
      if (r == 1) {
        int64_t j = 0;
        for (; j + 8 <= nb; j += 8) {  // eight 0/1 bytes -> eight bits
          uint64_t x;
          std::memcpy(&x, row + j, 8);
          bits[j >> 6] |= ((x * 0x0102040810204080ull) >> 56) << (j & 63);
        }
        for (; j < nb; ++j) bits[j >> 6] |= uint64_t(row[j] != 0) << (j & 63);
      } else {
        for (int64_t j = 0; j < nb; ++j)
          if (row[j])
            for (int64_t ks = j * r; ks < std::min((j + 1) * r, nseg); ++ks) bits[ks >> 6] |= 1ull << (ks & 63);
      }
      for (int64_t s = b * r; s < std::min((b + 1) * r, nseg); ++s) (*keyset)[s] = bits;
    }
    return;
  }
  fullset->assign(nseg, std::vector<uint64_t>(words, 0));
  std::vector<uint8_t> row(nb), row_all(nb);
  std::vector<int64_t> prefix(nb + 1), prefix_all(nb + 1);
  for (int64_t s = 0; s < nseg; ++s) {
    const int64_t t0 = s * kSeg, t1 = std::min(t0 + kSeg, n);
    const int64_t b0 = t0 / bs, b1 = (t1 - 1) / bs;
    std::fill(row.begin(), row.end(), 0);
    std::fill(row_all.begin(), row_all.end(), 1);
    for (int64_t b = b0; b <= b1; ++b)
      for (int64_t j = 0; j < nb; ++j) {
        row[j] |= grp.active[b * nb + j];
        row_all[j] &= grp.active[b * nb + j] != 0;
      }
    prefix[0] = prefix_all[0] = 0;
    for (int64_t j = 0; j < nb; ++j) {
      prefix[j + 1] = prefix[j] + row[j];
      prefix_all[j + 1] = prefix_all[j] + row_all[j];
    }
    auto& ks_bits = (*keyset)[s];
    auto& full_bits = (*fullset)[s];
    for (int64_t ks = 0; ks < nseg; ++ks) {
      const int64_t c0 = ks * kSeg, c1 = std::min(c0 + kSeg, n);
      const int64_t k0 = c0 / bs, k1 = (c1 - 1) / bs;
      if (prefix[k1 + 1] - prefix[k0] > 0) ks_bits[ks >> 6] |= 1ull << (ks & 63);
      if (prefix_all[k1 + 1] - prefix_all[k0] == k1 - k0 + 1) full_bits[ks >> 6] |= 1ull << (ks & 63);
    }
  }
}

static inline bool bit_of(const std::vector<uint64_t>& bits, int64_t i) {
  return (bits[i >> 6] >> (i & 63)) & 1ull;
}

// Cluster query segments four to a CTA so that the four share (nearly) one key
// set: identical key sets first (forced rows, FULL heads, multi-diagonal
// residue classes), then the remainder in index order (diagonal bands and
// stripes, whose neighbouring rows overlap).
static std::vector<std::array<int32_t, kSlotsPerItem>> cluster_segments(
    const std::vector<std::vector<uint64_t>>& keyset, int64_t nseg, int csize) {
  std::map<std::vector<uint64_t>, std::vector<int32_t>> buckets;
  std::vector<const std::vector<uint64_t>*> order;
  for (int64_t s = 0; s < nseg; ++s) {
    auto it = buckets.find(keyset[s]);
    if (it == buckets.end()) {
      it = buckets.emplace(keyset[s], std::vector<int32_t>()).first;
      order.push_back(&it->first);
    }
    it->second.push_back(int32_t(s));
  }
  std::vector<std::array<int32_t, kSlotsPerItem>> out;
  std::vector<int32_t> rest;
  for (auto* key : order) {
    const auto& members = buckets[*key];
    size_t full = members.size() / csize * csize;
    for (size_t i = 0; i < full; i += csize) {
      std::array<int32_t, kSlotsPerItem> q;
      for (int k = 0; k < kSlotsPerItem; ++k) q[k] = k < csize ? members[i + k] : -1;
      out.push_back(q);
    }
    for (size_t i = full; i < members.size(); ++i) rest.push_back(members[i]);
  }
  std::sort(rest.begin(), rest.end());
  for (size_t i = 0; i < rest.size(); i += csize) {
    std::array<int32_t, kSlotsPerItem> q;
    for (int k = 0; k < kSlotsPerItem; ++k)
      q[k] = (k < csize && i + k < rest.size()) ? rest[i + k] : -1;
    out.push_back(q);
  }
  return out;
}

static void build_group_schedule(svd_plan* P, Group& grp) {
  const int64_t nseg = P->nseg;
  grp.qgroups.clear();
  grp.qgroup_kv_begin.clear();
  grp.qgroup_kv_count.clear();
  if (grp.skip) {
    for (int64_t s = 0; s < nseg; s += P->cluster) {
      std::array<int32_t, kSlotsPerItem> q;
      for (int k = 0; k < kSlotsPerItem; ++k)
        q[k] = (k < P->cluster && s + k < nseg) ? int32_t(s + k) : -1;
      grp.qgroups.push_back(q);
      grp.qgroup_kv_begin.push_back(0);
      grp.qgroup_kv_count.push_back(0);
    }
    return;
  }
  std::vector<std::vector<uint64_t>> keyset, fullset;
  segment_keysets(grp, P->grid, nseg, &keyset, &fullset);
  // segment-grain grids: an active segment pair is one active block pair
  const auto& full = P->fine ? fullset : keyset;
  grp.qgroups = cluster_segments(keyset, nseg, P->cluster);
  const bool tail_partial = (P->grid.n % kSeg) != 0;
  const int64_t words = (nseg + 63) / 64;
  std::vector<uint64_t> uni(words);
  std::vector<int32_t> keys;
  keys.reserve(size_t(nseg));
  for (auto& q : grp.qgroups) {
    std::fill(uni.begin(), uni.end(), 0);
    for (int k = 0; k < kSlotsPerItem; ++k)
      if (q[k] >= 0)
        for (int64_t w = 0; w < words; ++w) uni[w] |= keyset[q[k]][w];
    keys.clear();
    for (int64_t w = 0; w < words; ++w)
      for (uint64_t m = uni[w]; m; m &= m - 1) keys.push_back(int32_t(w * 64 + __builtin_ctzll(m)));
    grp.qgroup_kv_begin.push_back(int32_t(P->kv.size()));
    for (size_t i = 0; i < keys.size(); i += 2) {
      KvEntry e{};
      e.kseg0 = keys[i];
      e.kseg1 = i + 1 < keys.size() ? keys[i + 1] : -1;
      uint32_t bits = 0;
      bool all = e.kseg1 >= 0;
      for (int slot = 0; slot < kSlotsPerItem; ++slot) {
        for (int kslot = 0; kslot < 2; ++kslot) {
          const int32_t ks = kslot == 0 ? e.kseg0 : e.kseg1;
          bool on;
          if (q[slot] < 0) on = true;  // empty q slot: never stored
          else on = ks >= 0 && bit_of(keyset[q[slot]], ks);
          if (on) bits |= 1u << (2 * slot + kslot);
          // FINE: "all" also needs every block pair under the segment pair active
          if (!on || (q[slot] >= 0 && !bit_of(full[q[slot]], ks))) all = false;
        }
      }
      const bool tail = tail_partial && (e.kseg0 == nseg - 1 || e.kseg1 == nseg - 1);
      if (tail) all = false;
      e.flags = bits | (all ? kFlagAll : 0u) | (tail ? kFlagTail : 0u) | (P->fine ? kFlagFine : 0u);
      P->kv.push_back(e);
    }
    grp.qgroup_kv_count.push_back(int32_t(P->kv.size()) - grp.qgroup_kv_begin.back());
  }
}

static double group_active_pairs(const Group& grp, const Grid& g) {
  if (grp.skip) return 0.0;
  const int64_t nb = g.nb;
  // every block holds bs tokens except the last: cols = bs * count - short(last)
  const int64_t last_short = g.bs - (g.bounds[nb] - g.bounds[nb - 1]);
  double total = 0.0;
  for (int64_t i = 0; i < nb; ++i) {
    const uint8_t* row = grp.active.data() + i * nb;
    int64_t count = 0;
    for (int64_t j = 0; j < nb; ++j) count += row[j] != 0;
    const int64_t cols = g.bs * count - (row[nb - 1] ? last_short : 0);
    total += double(g.bounds[i + 1] - g.bounds[i]) * double(cols);
  }
  return total;
}


static void build_items(svd_plan* P);

static void finalize_plan(svd_plan* P) {
  // query segments per CTA: two 128-row tiles ping-ponging in the kernel
  if (P->cluster == 0) P->cluster = kDefaultCluster;
  P->nseg = (P->grid.n + kSeg - 1) / kSeg;
  P->fine = (P->grid.bs % kSeg) != 0;
  P->kv.clear();
  for (auto& grp : P->groups) build_group_schedule(P, grp);
  // fine-mask bit tables (per element lookups when block_size % 64 != 0)
  P->fine_bits.clear();
  P->fine_bit_off.assign(P->groups.size(), -1);
  if (P->fine) {
    const int64_t nb = P->grid.nb, wpr = (nb + 31) / 32;
    for (size_t gi = 0; gi < P->groups.size(); ++gi) {
      const Group& grp = P->groups[gi];
      if (grp.skip) continue;
      P->fine_bit_off[gi] = int64_t(P->fine_bits.size());
      P->fine_bits.resize(P->fine_bits.size() + size_t(nb * wpr), 0u);
      uint32_t* base = P->fine_bits.data() + P->fine_bit_off[gi];
      for (int64_t i = 0; i < nb; ++i)
        for (int64_t j = 0; j < nb; ++j)
          if (grp.active[i * nb + j]) base[i * wpr + (j >> 5)] |= 1u << (j & 31);
    }
  }
  for (auto& grp : P->groups) grp.pairs = group_active_pairs(grp, P->grid);
  build_items(P);
}

// Work items of every (group, head, query-segment cluster), heaviest first.
static void build_items(svd_plan* P) {
  P->items.clear();
  P->active_pairs = 0.0;
  for (size_t gi = 0; gi < P->groups.size(); ++gi) {
    const Group& grp = P->groups[gi];
    P->active_pairs += double(grp.heads.size()) * grp.pairs;
    for (int32_t h : grp.heads) {
      for (size_t qi = 0; qi < grp.qgroups.size(); ++qi) {
        WorkItem it{};
        it.head = h;
        it.group = int32_t(gi);
        it.kv_begin = grp.qgroup_kv_begin[qi];
        it.kv_count = grp.qgroup_kv_count[qi];
        for (int k = 0; k < kSlotsPerItem; ++k) it.qseg[k] = grp.qgroups[qi][k];
        it.out_base = -1;
        it.split_group = -1;
        it.split_part = 0;
        it.split_parts = 1;
        P->items.push_back(it);
      }
    }
  }
  // heaviest first: the hardware block scheduler then behaves like LPT
  std::stable_sort(P->items.begin(), P->items.end(),
                   [](const WorkItem& a, const WorkItem& b) { return a.kv_count > b.kv_count; });
  P->computed_tiles = 0;
  for (const auto& it : P->items) P->computed_tiles += 2 * int64_t(it.kv_count);
}

// Split-KV for SM balance inside a shard: an item whose KV list exceeds
// `cap` tiles is cut into ceil(kv / cap) contiguous parts (at most
// kMaxSplitParts); the kernel merges the parts' partial softmax states in
// the epilogue of whichever part finishes last.  Re-sorted heaviest-first.
constexpr int kMaxSplitParts = 8;
constexpr double kItemOverhead = 4.0;  // per-CTA fixed cost, in KV tile steps
static void split_items(svd_plan* S, int64_t cap) {
  S->n_split_groups = 0;
  S->max_split_parts = 1;
  if (cap <= 0) return;
  std::vector<WorkItem> out;
  out.reserve(S->items.size());
  for (const auto& it : S->items) {
    const int64_t parts = std::min<int64_t>(kMaxSplitParts, (int64_t(it.kv_count) + cap - 1) / cap);
    if (it.kv_count <= cap || parts < 2) {
      out.push_back(it);
      continue;
    }
    const int32_t gid = S->n_split_groups++;
    S->max_split_parts = std::max<int32_t>(S->max_split_parts, int32_t(parts));
    for (int64_t p = 0; p < parts; ++p) {
      WorkItem w = it;
      const int64_t b0 = int64_t(it.kv_count) * p / parts, b1 = int64_t(it.kv_count) * (p + 1) / parts;
      w.kv_begin = it.kv_begin + int32_t(b0);
      w.kv_count = int32_t(b1 - b0);
      w.split_group = gid;
      w.split_part = int32_t(p);
      w.split_parts = int32_t(parts);
      out.push_back(w);
    }
  }
  std::stable_sort(out.begin(), out.end(),
                   [](const WorkItem& a, const WorkItem& b) { return a.kv_count > b.kv_count; });
  S->items.swap(out);
}

}  // namespace svd

using namespace svd;

extern "C" {

const char* svd_last_error(void) { return g_last_error.c_str(); }

int svd_grid_size(const svd_layout* layout, int64_t* n_tokens, int64_t* n_blocks) {
  int st = check_layout(layout);
  if (st) return st;
  const int64_t n = layout->text_tokens + layout->frames * layout->tokens_per_frame;
  if (n_tokens) *n_tokens = n;
  if (n_blocks) *n_blocks = (n + layout->block_size - 1) / layout->block_size;
  return SVD_OK;
}

int svd_grid_arrays(const svd_layout* layout, int64_t* bounds, uint8_t* has_text, uint8_t* mixed,
                    int64_t* frame_index) {
  Grid g;
  int st = make_grid(layout, &g);
  if (st) return st;
  if (bounds) std::copy(g.bounds.begin(), g.bounds.end(), bounds);
  if (has_text) std::copy(g.has_text.begin(), g.has_text.end(), has_text);
  if (mixed) std::copy(g.mixed.begin(), g.mixed.end(), mixed);
  if (frame_index) std::copy(g.frame_index.begin(), g.frame_index.end(), frame_index);
  return SVD_OK;
}

int svd_frame_period(const svd_layout* layout, int64_t* period) {
  int st = check_layout(layout);
  if (st) return st;
  *period = frame_period(layout);
  return SVD_OK;
}

int svd_mask_build(const svd_layout* layout, const svd_spec* spec, uint8_t* active,
                   int32_t* is_skip) {
  Grid g;
  int st = make_grid(layout, &g);
  if (st) return st;
  NormSpec ns;
  st = normalise_spec(spec, &ns);
  if (st) return st;
  bool skip = false;
  if (ns.mode == SVD_SKIP) {
    if (is_skip) *is_skip = 1;
    return SVD_OK;
  }
  if (!active) return fail(SVD_ERR_CONFIG, "active buffer is NULL");
  st = build_mask(ns, g, layout, active, &skip);
  if (is_skip) *is_skip = skip ? 1 : 0;
  return st;
}

int svd_plan_create(const svd_layout* layout, const svd_spec* specs, int32_t n_heads,
                    svd_plan** plan) {
  if (!plan) return fail(SVD_ERR_CONFIG, "plan out-pointer is NULL");
  *plan = nullptr;
  if (n_heads < 1) return fail(SVD_ERR_CONFIG, "need at least one head");
  if (!specs) return fail(SVD_ERR_CONFIG, "specs is NULL");
  auto* P = new svd_plan();
  P->layout = *layout;
  int st = make_grid(layout, &P->grid);
  if (st) {
    delete P;
    return st;
  }
  P->n_heads = n_heads;
  // attention.py:170-176: first-occurrence order, members ascending
  std::vector<NormSpec> norm(n_heads);
  for (int32_t h = 0; h < n_heads; ++h) {
    st = normalise_spec(&specs[h], &norm[h]);
    if (st) {
      delete P;
      return st;
    }
  }
  std::map<NormSpec, int32_t> index;
  P->head_group.resize(n_heads);
  for (int32_t h = 0; h < n_heads; ++h) {
    auto it = index.find(norm[h]);
    if (it == index.end()) {
      it = index.emplace(norm[h], int32_t(P->groups.size())).first;
      Group grp;
      grp.spec = norm[h];
      P->groups.push_back(std::move(grp));
    }
    P->groups[it->second].heads.push_back(h);
    P->head_group[h] = it->second;
  }
  // attention.py:177-182: one mask per non-FULL/SKIP group, built in group order
  const int64_t nb = P->grid.nb;
  for (auto& grp : P->groups) {
    grp.skip = grp.spec.mode == SVD_SKIP;
    if (grp.skip) continue;
    grp.active.assign(size_t(nb * nb), 0);
    bool skip = false;
    st = build_mask(grp.spec, P->grid, layout, grp.active.data(), &skip);
    if (st) {
      delete P;
      return st;
    }
  }
  finalize_plan(P);
  *plan = P;
  return SVD_OK;
}

int svd_plan_create_from_masks(const svd_layout* layout, int32_t n_groups, const int32_t* group_skip,
                               const uint8_t* masks, const int32_t* head_group, int32_t n_heads,
                               svd_plan** plan) {
  if (!plan) return fail(SVD_ERR_CONFIG, "plan out-pointer is NULL");
  *plan = nullptr;
  if (n_heads < 1 || n_groups < 1) return fail(SVD_ERR_CONFIG, "need at least one head and group");
  if (!masks || !head_group) return fail(SVD_ERR_CONFIG, "NULL masks or head_group");
  auto* P = new svd_plan();
  P->layout = *layout;
  int st = make_grid(layout, &P->grid);
  if (st) {
    delete P;
    return st;
  }
  const int64_t nb = P->grid.nb;
  P->n_heads = n_heads;
  P->groups.resize(n_groups);
  for (int32_t g = 0; g < n_groups; ++g) {
    Group& grp = P->groups[g];
    grp.skip = group_skip && group_skip[g];
    grp.spec.mode = grp.skip ? SVD_SKIP : SVD_FULL;  // explicit masks carry no spec
    if (!grp.skip) {
      grp.active.assign(masks + size_t(g) * nb * nb, masks + size_t(g + 1) * nb * nb);
      // attention.py:72-73 sparse_attention rejects an empty query row
      for (int64_t i = 0; i < nb; ++i) {
        bool any = false;
        for (int64_t j = 0; j < nb && !any; ++j) any = grp.active[i * nb + j] != 0;
        if (!any) {
          delete P;
          return fail(SVD_ERR_DEGENERATE_ROW, "mask has a query row with no active key blocks");
        }
      }
    }
  }
  P->head_group.assign(head_group, head_group + n_heads);
  for (int32_t h = 0; h < n_heads; ++h) {
    if (P->head_group[h] < 0 || P->head_group[h] >= n_groups) {
      delete P;
      return fail(SVD_ERR_CONFIG, "head_group out of range");
    }
    P->groups[P->head_group[h]].heads.push_back(h);
  }
  finalize_plan(P);
  *plan = P;
  return SVD_OK;
}

void svd_plan_destroy(svd_plan* plan) {
  if (!plan) return;
  release_device_tables(plan);
  delete plan;
}

int svd_plan_get_info(const svd_plan* P, svd_plan_info* info) {
  if (!P || !info) return fail(SVD_ERR_CONFIG, "NULL argument");
  info->n_tokens = P->grid.n;
  info->n_blocks = P->grid.nb;
  info->n_segments = P->nseg;
  info->n_heads = P->n_heads;
  info->n_groups = int32_t(P->groups.size());
  info->fine_mask = P->fine ? 1 : 0;
  info->sharded = P->sharded ? 1 : 0;
  info->n_work_items = int64_t(P->items.size());
  info->n_kv_entries = int64_t(P->kv.size());
  info->computed_tiles = P->computed_tiles;
  info->active_pairs = P->active_pairs;
  info->dense_pairs = double(P->grid.n) * double(P->grid.n) * double(P->n_heads);
  info->n_split_groups = P->n_split_groups;
  info->max_split_parts = P->max_split_parts;
  return SVD_OK;
}

int svd_plan_group_heads(const svd_plan* P, int32_t g, int32_t* heads, int32_t* n_heads,
                         int32_t* is_skip) {
  if (!P || g < 0 || g >= int32_t(P->groups.size())) return fail(SVD_ERR_CONFIG, "bad group index");
  const Group& grp = P->groups[g];
  if (n_heads) *n_heads = int32_t(grp.heads.size());
  if (heads) std::copy(grp.heads.begin(), grp.heads.end(), heads);
  if (is_skip) *is_skip = grp.skip ? 1 : 0;
  return SVD_OK;
}

int svd_plan_group_mask(const svd_plan* P, int32_t g, uint8_t* active) {
  if (!P || g < 0 || g >= int32_t(P->groups.size())) return fail(SVD_ERR_CONFIG, "bad group index");
  const Group& grp = P->groups[g];
  if (grp.skip) return fail(SVD_ERR_CONFIG, "SKIP group has no mask");
  std::copy(grp.active.begin(), grp.active.end(), active);
  return SVD_OK;
}

int svd_plan_group_nnz(const svd_plan* P, int32_t g, int64_t* nnz) {
  if (!P || g < 0 || g >= int32_t(P->groups.size())) return fail(SVD_ERR_CONFIG, "bad group index");
  const Group& grp = P->groups[g];
  int64_t c = 0;
  for (uint8_t a : grp.active) c += a != 0;
  *nnz = c;
  return SVD_OK;
}

// patterns.py:205-208 active_key_blocks(qb) = flatnonzero(active[qb]), per row
int svd_plan_group_csr(const svd_plan* P, int32_t g, int64_t* row_ptr, int64_t* col_idx) {
  if (!P || g < 0 || g >= int32_t(P->groups.size())) return fail(SVD_ERR_CONFIG, "bad group index");
  const Group& grp = P->groups[g];
  const int64_t nb = P->grid.nb;
  row_ptr[0] = 0;
  int64_t c = 0;
  for (int64_t i = 0; i < nb; ++i) {
    if (!grp.skip)
      for (int64_t j = 0; j < nb; ++j)
        if (grp.active[i * nb + j]) col_idx[c++] = j;
    row_ptr[i + 1] = c;
  }
  return SVD_OK;
}

int svd_plan_schedule(const svd_plan* P, int32_t* items, int32_t* kv) {
  if (!P) return fail(SVD_ERR_CONFIG, "plan is NULL");
  if (items) std::memcpy(items, P->items.data(), P->items.size() * sizeof(WorkItem));
  if (kv) std::memcpy(kv, P->kv.data(), P->kv.size() * sizeof(KvEntry));
  return SVD_OK;
}

int svd_plan_subset(const svd_plan* P, const int32_t* heads, int32_t n_heads, svd_plan** out) {
  if (!P || !heads || !out) return fail(SVD_ERR_CONFIG, "NULL argument");
  *out = nullptr;
  if (P->sharded) return fail(SVD_ERR_CONFIG, "a shard plan cannot be subset by heads");
  if (n_heads < 1) return fail(SVD_ERR_CONFIG, "need at least one head");
  std::vector<uint8_t> seen(P->n_heads, 0);
  for (int32_t i = 0; i < n_heads; ++i) {
    if (heads[i] < 0 || heads[i] >= P->n_heads) return fail(SVD_ERR_CONFIG, "head out of range");
    if (seen[heads[i]]++) return fail(SVD_ERR_CONFIG, "duplicate head");
  }
  auto* S = new svd_plan();
  S->layout = P->layout;
  S->grid = P->grid;
  S->nseg = P->nseg;
  S->fine = P->fine;
  S->cluster = P->cluster;
  S->n_heads = n_heads;
  S->head_group.resize(n_heads);
  // the parent's groups in first-occurrence order of the listed heads, each
  // with its mask, schedule and KV list copied (nothing is rebuilt)
  std::vector<int32_t> remap(P->groups.size(), -1);
  const int64_t wpr = (P->grid.nb + 31) / 32;
  for (int32_t i = 0; i < n_heads; ++i) {
    const int32_t pg = P->head_group[heads[i]];
    if (remap[pg] < 0) {
      remap[pg] = int32_t(S->groups.size());
      const Group& src = P->groups[pg];
      Group g;
      g.spec = src.spec;
      g.skip = src.skip;
      g.active = src.active;
      g.qgroups = src.qgroups;
      g.qgroup_kv_count = src.qgroup_kv_count;
      g.pairs = src.pairs;
      int64_t kv0 = 0, kv1 = 0;
      if (!src.qgroups.empty()) {
        kv0 = src.qgroup_kv_begin.front();
        kv1 = int64_t(src.qgroup_kv_begin.back()) + src.qgroup_kv_count.back();
      }
      const int64_t base = int64_t(S->kv.size());
      for (size_t q = 0; q < src.qgroups.size(); ++q)  // SKIP clusters keep begin 0, count 0
        g.qgroup_kv_begin.push_back(src.skip ? 0 : int32_t(src.qgroup_kv_begin[q] - kv0 + base));
      S->kv.insert(S->kv.end(), P->kv.begin() + kv0, P->kv.begin() + kv1);
      if (P->fine && !src.skip) {
        S->fine_bit_off.push_back(int64_t(S->fine_bits.size()));
        const auto* b = P->fine_bits.data() + P->fine_bit_off[pg];
        S->fine_bits.insert(S->fine_bits.end(), b, b + P->grid.nb * wpr);
      } else {
        S->fine_bit_off.push_back(-1);
      }
      S->groups.push_back(std::move(g));
    }
    S->head_group[i] = remap[pg];
    S->groups[remap[pg]].heads.push_back(i);
  }
  build_items(S);
  *out = S;
  return SVD_OK;
}

int svd_plan_shard_ex(const svd_plan* P, int32_t world, int32_t rank, int32_t n_sms,
                      int32_t max_item_tiles, int32_t partition, svd_plan** shard) {
  if (!P || !shard) return fail(SVD_ERR_CONFIG, "NULL argument");
  if (P->sharded) return fail(SVD_ERR_CONFIG, "plan is already a shard");
  if (world < 1 || rank < 0 || rank >= world) return fail(SVD_ERR_CONFIG, "bad world/rank");
  if (n_sms < 1) return fail(SVD_ERR_CONFIG, "n_sms must be >= 1");
  if (partition != SVD_PARTITION_ITEMS && partition != SVD_PARTITION_HEADS)
    return fail(SVD_ERR_CONFIG, "unknown partition");
  auto* S = new svd_plan();
  S->layout = P->layout;
  S->grid = P->grid;
  S->nseg = P->nseg;
  S->n_heads = P->n_heads;
  S->fine = P->fine;
  S->cluster = P->cluster;
  S->head_group = P->head_group;
  S->groups = P->groups;
  S->kv = P->kv;
  S->fine_bits = P->fine_bits;
  S->fine_bit_off = P->fine_bit_off;
  S->active_pairs = P->active_pairs;
  S->sharded = true;
  // LPT over ranks on the tile cost (items are already heaviest-first); an
  // item stays whole across ranks — its split parts (below) share a rank.
  // Cost in 128-key tile steps + a fixed per-CTA overhead (TMEM / barrier
  // setup, Q load, pipeline fill, epilogue): short sparse items are not free.
  auto item_cost = [](const WorkItem& it) {
    return it.kv_count > 0 ? double(it.kv_count) + kItemOverhead : 0.5 * kItemOverhead;
  };
  std::vector<double> load(world, 0.0);
  std::vector<int32_t> owner(P->items.size());
  if (partition == SVD_PARTITION_ITEMS) {
    for (size_t i = 0; i < P->items.size(); ++i) {
      const int32_t best = int32_t(std::min_element(load.begin(), load.end()) - load.begin());
      load[best] += item_cost(P->items[i]);
      owner[i] = best;
    }
  } else {
    // McNaughton's wrap-around over a head sequence: rank r takes the cost
    // interval [r T, (r+1) T) of the head-ordered item sequence, so it holds
    // whole heads except for at most the two boundary heads of its interval
    // (split by query range) — its inputs are those heads only.  The sequence
    // interleaves heavy and light heads so that every interval also covers
    // about H / world heads (the rank's copy-in bytes): at each step the
    // lightest remaining head if the running cost share is ahead of the
    // running head share, else the heaviest.
    const int32_t H = P->n_heads;
    std::vector<std::vector<size_t>> by_head(static_cast<size_t>(H));
    std::vector<double> hcost(static_cast<size_t>(H), 0.0);
    double total = 0.0;
    for (size_t i = 0; i < P->items.size(); ++i) {
      by_head[size_t(P->items[i].head)].push_back(i);
      hcost[size_t(P->items[i].head)] += item_cost(P->items[i]);
      total += item_cost(P->items[i]);
    }
    std::vector<int32_t> desc(static_cast<size_t>(H));
    for (int32_t h = 0; h < H; ++h) desc[size_t(h)] = h;
    std::stable_sort(desc.begin(), desc.end(),
                     [&](int32_t a, int32_t b) { return hcost[size_t(a)] > hcost[size_t(b)]; });
    std::vector<int32_t> seq;
    size_t lo = 0, hi = desc.size();
    double seq_cost = 0.0;
    while (lo < hi) {
      const bool cost_ahead = seq_cost / total > double(seq.size()) / double(H);
      const int32_t h = cost_ahead ? desc[--hi] : desc[lo++];
      seq.push_back(h);
      seq_cost += hcost[size_t(h)];
    }
    const double T = total / double(world);
    double cum = 0.0;
    for (int32_t h : seq)
      for (size_t i : by_head[size_t(h)]) {
        const double c = item_cost(P->items[i]);
        const int32_t r = std::min<int32_t>(world - 1, int32_t((cum + 0.5 * c) / T));
        owner[i] = r;
        load[r] += c;
        cum += c;
      }
  }
  for (size_t i = 0; i < P->items.size(); ++i) {
    if (owner[i] != rank) continue;
    WorkItem w = P->items[i];
    w.out_base = int32_t(S->n_rows);
    for (int k = 0; k < kSlotsPerItem; ++k) {
      if (w.qseg[k] < 0) continue;
      for (int r = 0; r < kSeg; ++r) {
        const int64_t tok = int64_t(w.qseg[k]) * kSeg + r;
        S->row_head.push_back(tok < P->grid.n ? w.head : -1);
        S->row_token.push_back(tok < P->grid.n ? int32_t(tok) : -1);
      }
      S->n_rows += kSeg;
    }
    S->items.push_back(w);
  }
  // Split-KV cap, one for all ranks: each rank's items are packed onto n_sms
  // SMs by the hardware's heaviest-first dispatch; when a rank holds only a
  // few long items per SM (8 GPUs: ~2.6 FULL-row items per SM) that packing
  // is lumpy (~87% efficiency).  Try caps of 1/4 .. 1/16 of the mean per-SM
  // load, simulate every rank's dispatch (greedy onto the least-loaded SM,
  // +2 steps per split part for the merge) and keep the cap with the
  // smallest slowest-rank makespan.
  int64_t cap = max_item_tiles;
  if (cap == 0) {
    auto makespan = [&](int64_t c) {
      double worst = 0.0;
      for (int32_t r = 0; r < world; ++r) {
        std::vector<double> costs;
        for (size_t i = 0; i < P->items.size(); ++i) {
          if (owner[i] != r) continue;
          const WorkItem& it = P->items[i];
          const int64_t parts = (c > 0 && it.kv_count > c)
                                    ? std::min<int64_t>(kMaxSplitParts, (int64_t(it.kv_count) + c - 1) / c)
                                    : 1;
          for (int64_t p = 0; p < parts; ++p)
            costs.push_back(double(it.kv_count) / double(parts) + kItemOverhead + (parts > 1 ? 2.0 : 0.0));
        }
        std::sort(costs.begin(), costs.end(), std::greater<double>());
        std::priority_queue<double, std::vector<double>, std::greater<double>> sm;
        for (int i = 0; i < n_sms; ++i) sm.push(0.0);
        for (double c2 : costs) {
          const double t = sm.top() + c2;
          sm.pop();
          sm.push(t);
          worst = std::max(worst, t);
        }
      }
      return worst;
    };
    const double per_sm = *std::max_element(load.begin(), load.end()) / double(n_sms);
    double best = makespan(-1);
    cap = -1;
    for (int div : {4, 6, 8, 12, 16}) {
      const int64_t c = std::max<int64_t>(32, int64_t(per_sm / div));
      const double m = makespan(c);
      if (m < best * 0.995) {
        best = m;
        cap = c;
      }
    }
  }
  split_items(S, cap);
  S->computed_tiles = 0;
  for (const auto& it : S->items) S->computed_tiles += 2 * int64_t(it.kv_count);
  *shard = S;
  return SVD_OK;
}

int svd_plan_shard_sm(const svd_plan* P, int32_t world, int32_t rank, int32_t n_sms,
                      int32_t max_item_tiles, svd_plan** shard) {
  return svd_plan_shard_ex(P, world, rank, n_sms, max_item_tiles, SVD_PARTITION_ITEMS, shard);
}

int svd_plan_shard(const svd_plan* P, int32_t world, int32_t rank, svd_plan** shard) {
  return svd_plan_shard_sm(P, world, rank, 148, 0, shard);
}

// The items of a shard plan that belong to the listed heads (split-KV parts
// included: they share their head), as a shard plan with the parent's packed
// row layout — one chunk of a rank's pipelined end-to-end step.
int svd_plan_shard_heads(const svd_plan* S, const int32_t* heads, int32_t n_heads, svd_plan** out) {
  if (!S || !heads || !out) return fail(SVD_ERR_CONFIG, "NULL argument");
  *out = nullptr;
  if (!S->sharded) return fail(SVD_ERR_CONFIG, "not a shard plan");
  if (n_heads < 1) return fail(SVD_ERR_CONFIG, "need at least one head");
  std::vector<uint8_t> keep(size_t(S->n_heads), 0);
  for (int32_t i = 0; i < n_heads; ++i) {
    if (heads[i] < 0 || heads[i] >= S->n_heads) return fail(SVD_ERR_CONFIG, "head out of range");
    if (keep[size_t(heads[i])]++) return fail(SVD_ERR_CONFIG, "duplicate head");
  }
  auto* C = new svd_plan();
  C->layout = S->layout;
  C->grid = S->grid;
  C->nseg = S->nseg;
  C->n_heads = S->n_heads;
  C->fine = S->fine;
  C->cluster = S->cluster;
  C->head_group = S->head_group;
  C->groups = S->groups;
  C->kv = S->kv;
  C->fine_bits = S->fine_bits;
  C->fine_bit_off = S->fine_bit_off;
  C->active_pairs = S->active_pairs;
  C->sharded = true;
  C->n_split_groups = S->n_split_groups;  // group ids kept: scratch sized as the parent's
  C->max_split_parts = S->max_split_parts;
  C->n_rows = S->n_rows;
  C->row_head = S->row_head;
  C->row_token = S->row_token;
  for (const auto& it : S->items)
    if (keep[size_t(it.head)]) C->items.push_back(it);
  for (const auto& it : C->items) C->computed_tiles += 2 * int64_t(it.kv_count);
  *out = C;
  return SVD_OK;
}

int svd_plan_shard_rows(const svd_plan* S, int64_t* n_rows, int32_t* row_head, int32_t* row_token) {
  if (!S || !S->sharded) return fail(SVD_ERR_CONFIG, "not a shard plan");
  if (n_rows) *n_rows = S->n_rows;
  if (row_head) std::copy(S->row_head.begin(), S->row_head.end(), row_head);
  if (row_token) std::copy(S->row_token.begin(), S->row_token.end(), row_token);
  return SVD_OK;
}

}  // extern "C"
