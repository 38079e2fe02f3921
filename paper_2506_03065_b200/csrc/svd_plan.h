// Internal plan representation shared by the host plan builder (svd_plan.cpp)
// and the sm_100a forward kernel (svd_attn_fwd.cu).  Not part of the C ABI.
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/svdit_b200.h"

namespace svd {

// The kernel's mask grain: 64-token segments.  A 128-row MMA tile holds two
// query segments, a 128-key KV tile holds two key segments; the reference's
// block_size-64 blocks map 1:1 onto segments (layout.py:31 default).
constexpr int kSeg = 64;
constexpr int kSlotsPerItem = 4;  // two 128-row Q tiles (A, B) x two segments
constexpr int kDefaultCluster = 4;  // query segments per CTA (two 128-row tiles)

// KvEntry.flags
constexpr uint32_t kFlagAll = 1u << 8;    // every present (q slot, k slot) active, no tail
constexpr uint32_t kFlagTail = 1u << 9;   // a key slot holds tokens >= N
constexpr uint32_t kFlagFine = 1u << 10;  // block_size % 64 != 0: per-element lookup

// One CTA's work: up to four 64-row query segments of one head, all of which
// share the KV tile list kv[kv_begin, kv_begin + kv_count).  kv_count == 0 is
// a SKIP head's zero-fill item (attention.py:51-54).
struct WorkItem {
  int32_t head;
  int32_t group;
  int32_t kv_begin;
  int32_t kv_count;
  int32_t qseg[kSlotsPerItem];  // -1 = empty slot (empty slots form a suffix)
  int32_t out_base;             // packed output row of slot 0 (shards), else -1
  // split-KV: items whose KV list was cut into parts (to balance SMs in a
  // shard) carry split group id / part index / part count; -1 / 0 / 1 else
  int32_t split_group;
  int32_t split_part;
  int32_t split_parts;
};
static_assert(sizeof(WorkItem) == 48, "WorkItem layout");

// One 128-key tile: two key segments (kseg1 = -1: single segment) and the
// activity bits (q slot i, k slot j) -> bit (2*i + j).
struct KvEntry {
  int32_t kseg0;
  int32_t kseg1;
  uint32_t flags;
  int32_t pad;
};
static_assert(sizeof(KvEntry) == 16, "KvEntry layout");

struct NormSpec {
  int32_t mode = 0;
  int32_t halfwidth = 1;
  int32_t period = -1;  // -1 = None
  int32_t md_halfwidth = 0;
  int32_t stripe_count = 2;
  int32_t include_diagonal = 1;
  bool stripes_none = true;
  std::vector<int64_t> stripes;  // sorted unique
  bool operator<(const NormSpec& o) const;
  bool operator==(const NormSpec& o) const;
};

struct Group {
  NormSpec spec;
  bool skip = false;
  std::vector<int32_t> heads;
  std::vector<uint8_t> active;  // nb*nb; empty for SKIP
  // kernel schedule for this group (shared by all its heads)
  std::vector<std::array<int32_t, kSlotsPerItem>> qgroups;
  std::vector<int32_t> qgroup_kv_begin, qgroup_kv_count;
  double pairs = 0.0;  // active (query token, key token) pairs of one head
};

struct DeviceTables {
  void* items = nullptr;
  void* kv = nullptr;
  void* bits = nullptr;
  void* bit_off = nullptr;
  void* split_scratch = nullptr;  // fp32 partial O [group][part][256][128] + (m, l) [..][256][2]
  void* split_tickets = nullptr;  // int32 per split group (parts finished), self-resetting
  int64_t n_items = 0;
};

struct Grid {
  int64_t n = 0, nb = 0, bs = 0;
  std::vector<int64_t> bounds;
  std::vector<uint8_t> has_text, mixed;
  std::vector<int64_t> frame_index;
};

}  // namespace svd

struct svd_plan {
  svd_layout layout{};
  svd::Grid grid;
  int64_t nseg = 0;
  int32_t n_heads = 0;
  bool fine = false;
  std::vector<int32_t> head_group;
  std::vector<svd::Group> groups;
  std::vector<svd::WorkItem> items;  // sorted heaviest-first
  std::vector<svd::KvEntry> kv;
  std::vector<uint32_t> fine_bits;    // per group: nb rows x ceil(nb/32) words
  std::vector<int64_t> fine_bit_off;  // per group word offset (-1 for skip)
  double active_pairs = 0.0;
  int64_t computed_tiles = 0;
  // shard view
  bool sharded = false;
  int32_t cluster = 0;  // query segments per work item (kDefaultCluster)
  int32_t n_split_groups = 0, max_split_parts = 1;
  int64_t n_rows = 0;
  std::vector<int32_t> row_head, row_token;
  // device copies, per CUDA device ordinal
  mutable std::mutex mu;
  mutable std::map<int, svd::DeviceTables> dev;
};

namespace svd {
void set_error(const std::string& msg);
int fail(int status, const std::string& msg);
void release_device_tables(const svd_plan* plan);  // defined in the .cu
}  // namespace svd
