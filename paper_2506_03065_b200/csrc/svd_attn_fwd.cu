// sm_100a block-sparse attention forward for the Sparse-vDiT hot path.
//
// Reference semantics: attention.py:57-98 (sparse_attention: per query block,
// an online softmax over that block's active key blocks), attention.py:101-105
// (full_mask_attention = all blocks active), attention.py:51-54 (skip: zeros)
// and attention.py:186-212 (fused_layer_attention: every head of the layer in
// one call, heads dispatched by pattern group).  Here the whole layer is ONE
// launch: a CTA per work item (four 64-token query segments of one head that
// share a list of 128-key tiles), heaviest items first.
//
// CTA anatomy (384 threads, 1 CTA / SM):
//   warp 0       TMA producer: Q tiles once, then K and V tiles through two
//                separate smem rings (SWIZZLE_128B boxes of 64x64 bf16)
//   warp 1       TMEM allocator + tcgen05.mma issuer (d=128: the whole warp,
//                one elected lane per MMA; d=64: lane 0)
//   warps 4-7    softmax/epilogue for Q tile A (thread = row = TMEM lane)
//   warps 8-11   softmax/epilogue for Q tile B
// Per KV tile j the issuer runs, ping-ponging between the two Q tiles,
//   S_X = Q_X K_j^T          (SS MMA, M=128 N=128 K=d, fp32 in TMEM)
//   O_X += P_X V_j           (TS MMA: P bf16 from TMEM, V MN-major in smem;
//                             issued per part as P is handed over: keys 0-31
//                             then 32-127 at d=128, 32-key quarters at d=64)
// while the softmax warpgroups turn S_X into P_X (masking, running max with
// lazy rescale of O, exp2 — at d=128 3/8 of it on the FMA pipe — bf16 P,
// rounded row sums) — so one tile's exps overlap the other tile's MMAs.
// Split-KV items (shard plans) publish partial (m, l, O) and the last part
// merges; the epilogue can store into several ranks' O (peer memory).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "svd_plan.h"
#include "svd_ptx.cuh"

namespace svd {

constexpr int kThreads = 384;
constexpr int kMaxPeers = 8;
constexpr int kMaxSplitPartsDev = 8;  // == kMaxSplitParts of the plan builder
constexpr uint32_t kTmemCols = 512;

// Row sums over the bf16-rounded P (the values the PV MMA consumes) rather
// than the fp32 exps: numerator and denominator then see the same weights,
// which removes the bf16 rounding of the dominant weight from peaked rows.
// d=128: accumulate the row sums after each chunk's P store (the store
// goes out sooner; -0.4%); d=64 keeps them interleaved (+0.8% otherwise)
#ifndef SVD_SUM_AFTER_ST
#define SVD_SUM_AFTER_ST 1
#endif
// P handed to the PV MMA in 32-key quarters instead of 64-key halves
// (bit 0: d=64, bit 1: d=128).  d=64: the PV starts after the first 32 keys'
// exps (CogVideoX -1.7%); d=128: +6% (the extra st-waits lengthen the
// softmax, which is the tensor pipe's feeder there)
#ifndef SVD_P_QUARTERS
#define SVD_P_QUARTERS 1
#endif
template <int D>
constexpr bool kPQuarters = (SVD_P_QUARTERS >> (D == 128 ? 1 : 0)) & 1;
// Lagged quarter hand-off (bit 0: d=64, bit 1: d=128): chunk c's P store is
// waited for (tcgen05.wait::st) only after chunk c+1's exps, when it has long
// completed, so the hand-offs stop stalling the softmax; the PV MMA still
// starts one 32-key quarter behind the exps and the tail after the last
// chunk is one quarter's PV.  Implies quarters.
#ifndef SVD_P_LAG
#define SVD_P_LAG 0
#endif
template <int D>
constexpr bool kPLag = (SVD_P_LAG >> (D == 128 ? 1 : 0)) & 1;
// two-part P handoff (d=128): the first part ends after 32-key chunk
// SVD_P_FIRST (0..2).  0 — PV starts after the first 32 keys, the rest follows
// as one part: -0.5% vs even halves (1), +1% for 2
#ifndef SVD_P_FIRST
#define SVD_P_FIRST 0
#endif
#ifndef SVD_SUM_ROUNDED
#define SVD_SUM_ROUNDED 1
#endif

template <int D>
struct KCfg {
  static constexpr int kSlabs = D / 64;
  static constexpr int kBoxBytes = 64 * 64 * 2;        // one TMA box: 64 rows x 128 B
  static constexpr int kSlabBytes = 128 * 128;         // 128 rows x 128 B (one SW128 slab)
  static constexpr int kTileBytes = 128 * D * 2;       // a Q tile or a KV tile
  static constexpr int kKSt = D == 128 ? 2 : 4;
  static constexpr int kVSt = D == 128 ? 2 : 4;
  // d=128 needs all 512 columns for S_A, S_B, O_A, O_B, so P_X aliases S_X
  // (S_X(j+1) then follows PV_X(j) in the in-order tensor pipe); d=64 keeps P
  // in its own columns.
  static constexpr int kOffQ = 0;
  static constexpr int kOffK = kOffQ + 2 * kTileBytes;
  static constexpr int kOffV = kOffK + kKSt * kTileBytes;
  static constexpr int kOffBar = kOffV + kVSt * kTileBytes;
  // barriers: q | kfull[K] kempty[K] | vfull[V] vempty[V] | s[2] p0[2] p1[2] o[2]
  static constexpr int kBarQ = 0;
  static constexpr int kBarKF = 1;
  static constexpr int kBarKE = kBarKF + kKSt;
  static constexpr int kBarVF = kBarKE + kKSt;
  static constexpr int kBarVE = kBarVF + kVSt;
  static constexpr int kBarS = kBarVE + kVSt;
  static constexpr int kBarP0 = kBarS + 2;
  static constexpr int kBarP1 = kBarP0 + 2;
  static constexpr int kBarP2 = kBarP1 + 2;  // P in quarters (SVD_P_QUARTERS)
  static constexpr int kBarP3 = kBarP2 + 2;
  static constexpr int kBarO = kBarP3 + 2;
  static constexpr int kNumBars = kBarO + 2;
  static constexpr int kOffTmemSlot = kOffBar + kNumBars * 8;
  static constexpr int kSmemBytes = kOffTmemSlot + 16 + 1024;  // + alignment slack
  __device__ static constexpr uint32_t col_s(int x) { return x ? 128u : 0u; }
  __device__ static constexpr uint32_t col_o(int x) { return x ? 256u + D : 256u; }
  __device__ static constexpr uint32_t col_p(int x) {
    return D == 128 ? col_s(x) : (x ? 448u : 384u);
  }
};

struct FwdParams {
  const WorkItem* items;
  const KvEntry* kv;
  const uint32_t* bits;      // fine-mask tables
  const int64_t* bit_off;    // per group word offset
  __nv_bfloat16* o;
  int64_t o_sb, o_sh, o_sn;  // element strides of O (d stride is 1)
  int n_tokens;
  int block_size;
  int words_per_row;
  int n_blocks;
  int packed;                // shard plan: O is a packed [rows, d] buffer
  float scale_log2;          // log2(e) / sqrt(d)
  // Fused reassembly: when n_peers > 0 every output row is stored into all
  // n_peers O buffers (this rank's and its peers', mapped over NVLink), all
  // with the same [B, H, N, D] strides; `o` / `packed` are then unused.
  int n_peers;
  __nv_bfloat16* peer_o[kMaxPeers];
  // split-KV merge (items with split_group >= 0): partial O rows [group][part][256][128]
  // fp32, then (m, l) [group][part][256][2]; one ticket per group
  float* split_o;
  float* split_ml;
  int* split_tickets;
  int max_split_parts;
  // optional output head permutation: plan head h writes O head o_head_map[h]
  const int32_t* o_head_map;
  // attention.py:98 require_finite: OR-ed with 1 when an output row is non-finite
  int* nonfinite;
  // optional input head permutation: plan head h reads Q/K/V head in_head_map[h]
  const int32_t* in_head_map;
  // optional per-row softmax statistics (-m, 1/l) of plan heads < stats_heads,
  // in block_key_mass's pass-0 layout [B * stats_heads][n_tiles128][2][128]
  float* row_stats;
  int stats_heads;
  int n_tiles128;
};

// (-m, 1/l) of one row into the key-mass row-statistics layout
__device__ __forceinline__ void store_row_stats(const FwdParams& p, int b, int head, int tok, bool valid,
                                                float m, float l) {
  if (!p.row_stats || head >= p.stats_heads || tok < 0) return;
  const int64_t bh = int64_t(b) * p.stats_heads + head;
  float* sp = p.row_stats + (bh * p.n_tiles128 + (tok >> 7)) * 256;
  const bool ok = valid && l > 0.f;
  sp[tok & 127] = ok ? -m : -INFINITY;
  sp[128 + (tok & 127)] = ok ? 1.0f / l : 0.f;
}

// Store one 16-byte chunk of an output row: to o + off, or to every peer.
__device__ __forceinline__ void store_row16(const FwdParams& p, int64_t off, const uint4& val) {
  if (p.n_peers == 0) {
    *reinterpret_cast<uint4*>(p.o + off) = val;
  } else {
#pragma unroll 1
    for (int r = 0; r < p.n_peers; ++r) *reinterpret_cast<uint4*>(p.peer_o[r] + off) = val;
  }
}

__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

__device__ __forceinline__ KvEntry load_kv(const KvEntry* ptr) {
  const int4 v = __ldg(reinterpret_cast<const int4*>(ptr));
  KvEntry e;
  e.kseg0 = v.x;
  e.kseg1 = v.y;
  e.flags = uint32_t(v.z);
  e.pad = v.w;
  return e;
}

template <int D>
__device__ __forceinline__ void load_tile(const CUtensorMap* tmap, uint32_t dst, uint32_t bar,
                                          int seg0, int seg1, int head, int b, uint64_t pol) {
  using C = KCfg<D>;
#pragma unroll
  for (int slot = 0; slot < 2; ++slot) {
    const int seg = slot ? seg1 : seg0;
#pragma unroll
    for (int slab = 0; slab < C::kSlabs; ++slab)
      ptx::tma_load_4d(dst + slab * C::kSlabBytes + slot * C::kBoxBytes, tmap, bar, slab * 64,
                       seg * kSeg, head, b, pol);
  }
}

// Mask one 128-key tile of S for this thread's row.  Segment-grain tiles
// (block_size % 64 == 0) need only the tile's activity bits and the sequence
// end; FINE (block_size % 64 != 0) builds each key segment's 64-bit key mask
// from the few blocks it overlaps (one bit lookup per block), then selects.
__device__ __forceinline__ uint64_t fine_segment_mask(int seg, int lim, const FwdParams& p,
                                                      const uint32_t* bits_row) {
  if (lim <= 0) return 0ull;
  const int c0 = seg * kSeg;
  const int kb_first = c0 / p.block_size, kb_last = (c0 + lim - 1) / p.block_size;
  uint64_t m = 0ull;
  for (int kb = kb_first; kb <= kb_last; ++kb) {
    if (!((__ldg(bits_row + (kb >> 5)) >> (kb & 31)) & 1u)) continue;
    const int lo = max(kb * p.block_size - c0, 0), hi = min((kb + 1) * p.block_size - c0, lim);
    const uint64_t upto_hi = hi >= 64 ? ~0ull : ((1ull << hi) - 1ull);
    m |= upto_hi & ~((1ull << lo) - 1ull);
  }
  return m;
}

template <bool FINE>
__device__ __forceinline__ void apply_mask(float (&s)[128], const KvEntry& e, int qslot,
                                           const FwdParams& p, const uint32_t* bits_row) {
  const bool on0 = (e.flags >> (2 * qslot)) & 1u;
  const bool on1 = (e.flags >> (2 * qslot + 1)) & 1u;
  const int lim0 = on0 ? min(kSeg, p.n_tokens - e.kseg0 * kSeg) : 0;
  const int lim1 = (on1 && e.kseg1 >= 0) ? min(kSeg, p.n_tokens - e.kseg1 * kSeg) : 0;
  if constexpr (FINE) {
    const uint64_t m0 = fine_segment_mask(e.kseg0, lim0, p, bits_row);
    const uint64_t m1 = fine_segment_mask(e.kseg1, lim1, p, bits_row);
    const uint32_t w[4] = {uint32_t(m0), uint32_t(m0 >> 32), uint32_t(m1), uint32_t(m1 >> 32)};
#pragma unroll
    for (int i = 0; i < 128; ++i)
      if (!((w[i >> 5] >> (i & 31)) & 1u)) s[i] = -INFINITY;
  } else {
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      if (i >= lim0) s[i] = -INFINITY;
      if (i >= lim1) s[64 + i] = -INFINITY;
    }
  }
}

// Exp2 offload: of every 8 consecutive column pairs, kEmuPairs go through
// the FMA-pipe polynomial instead of MUFU.ex2 (MUFU is 16/clk/SM, as fast as
// the tensor pipe needs at d=128).  Default d=128: the first 3 of every 8
// pairs (their longer dependency chains start first), minimax quadratic —
// -3.5% layer time (profiles/r1/KERNEL_NOTES.md); d=64: off (measured slower).
#ifndef SVD_EMU128
#define SVD_EMU128 3
#endif
#ifndef SVD_EMU64
#define SVD_EMU64 0
#endif
template <int D>
constexpr int kEmuPairs = D == 128 ? SVD_EMU128 : SVD_EMU64;
// which pairs of each 8 are emulated: 0 = the last kEmuPairs, 1 = the first
// (their long dependency chains start early), 2 = spread evenly, 3 = the first
// 2*kEmuPairs of each 16
#ifndef SVD_EMU_FIRST
#define SVD_EMU_FIRST 1
#endif
#ifndef SVD_EMU_DEG2
#define SVD_EMU_DEG2 1
#endif
template <int D>
__device__ __forceinline__ constexpr bool emulated_pair(int i) {
  return kEmuPairs<D> == 0 ? false
         : SVD_EMU_FIRST == 1 ? ((i & 7) < kEmuPairs<D>)
         : SVD_EMU_FIRST == 2 ? ((i & 7) % (8 / kEmuPairs<D>) == 0)
         : SVD_EMU_FIRST == 3 ? ((i & 15) < 2 * kEmuPairs<D>)
                              : ((i & 7) >= 8 - kEmuPairs<D>);
}

#ifdef SVD_TRACE
// Debug-only pipeline trace: (clock, step<<8 | event) pairs for the first 8
// CTAs of batch 0; streams 0/1 = softmax tile A/B (warp 4/8, lane 0), 2 = MMA.
constexpr int kTraceCtas = 8, kTraceEvents = 2048;
__device__ uint32_t g_trace[kTraceCtas][4][kTraceEvents][2];
__device__ __forceinline__ void trace_ev(int stream, int& n, int step, int code) {
  if (blockIdx.x < kTraceCtas && blockIdx.y == 0 && n < kTraceEvents) {
    g_trace[blockIdx.x][stream][n][0] = uint32_t(clock());
    g_trace[blockIdx.x][stream][n][1] = uint32_t(step << 8 | code);
    ++n;
  }
}
#define TRACE(stream, n, step, code) trace_ev(stream, n, step, code)
#else
#define TRACE(stream, n, step, code) ((void)0)
#endif

template <int D, bool FINE>
__global__ void __launch_bounds__(kThreads, 1)
    svd_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                   const __grid_constant__ CUtensorMap tm_v, const FwdParams p) {
  using C = KCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* base_ptr = smem_raw + (base - raw);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  auto bar = [&](int i) { return base + C::kOffBar + 8u * uint32_t(i); };

  const WorkItem* itp = p.items + blockIdx.x;
  const int b = blockIdx.y;
  const int n_kv = itp->kv_count;
  const int head = itp->head;

  if (threadIdx.x == 0) {
    ptx::mbar_init(bar(C::kBarQ), 1);
    for (int i = 0; i < C::kKSt; ++i) {
      ptx::mbar_init(bar(C::kBarKF + i), 1);
      ptx::mbar_init(bar(C::kBarKE + i), 1);
    }
    for (int i = 0; i < C::kVSt; ++i) {
      ptx::mbar_init(bar(C::kBarVF + i), 1);
      ptx::mbar_init(bar(C::kBarVE + i), 1);
    }
    for (int x = 0; x < 2; ++x) {
      ptx::mbar_init(bar(C::kBarS + x), 1);
      ptx::mbar_init(bar(C::kBarP0 + x), 128);
      ptx::mbar_init(bar(C::kBarP1 + x), 128);
      ptx::mbar_init(bar(C::kBarP2 + x), 128);
      ptx::mbar_init(bar(C::kBarP3 + x), 128);
      ptx::mbar_init(bar(C::kBarO + x), 1);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc(base + C::kOffTmemSlot, kTmemCols);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(base_ptr + C::kOffTmemSlot);

  // Register split: the producer / MMA warpgroup needs few registers, the two
  // softmax warpgroups hold a 128-wide fp32 row of S each.
#ifndef SVD_REG_LOW
#define SVD_REG_LOW 56
#endif
#ifndef SVD_REG_HIGH
#define SVD_REG_HIGH 224
#endif
  if (warp < 4) {
    ptx::reg_dealloc<SVD_REG_LOW>();
    if (warp == 0) {
      // ---------------------------------------------------------- TMA producer
      if (lane == 0 && n_kv > 0) {
        ptx::prefetch_tmap(&tm_q);
        ptx::prefetch_tmap(&tm_k);
        ptx::prefetch_tmap(&tm_v);
        const uint64_t pol_q = ptx::policy_evict_first();
        const uint64_t pol_kv = ptx::policy_evict_last();
        const int first = itp->qseg[0];
        const int in_head = p.in_head_map ? __ldg(p.in_head_map + head) : head;
        ptx::mbar_arrive_expect_tx(bar(C::kBarQ), 2 * C::kTileBytes);
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          int s0 = itp->qseg[2 * x], s1 = itp->qseg[2 * x + 1];
          s0 = s0 >= 0 ? s0 : first;
          s1 = s1 >= 0 ? s1 : first;
          load_tile<D>(&tm_q, base + C::kOffQ + x * C::kTileBytes, bar(C::kBarQ), s0, s1, in_head, b,
                       pol_q);
        }
        const KvEntry* kvp = p.kv + itp->kv_begin;
#ifdef SVD_TRACE
        int ptn = 0;
#endif
        for (int j = 0; j < n_kv; ++j) {
          const KvEntry e = load_kv(kvp + j);
          const int k0 = e.kseg0, k1 = e.kseg1 >= 0 ? e.kseg1 : e.kseg0;
          const int ks = j % C::kKSt, vs = j % C::kVSt;
          ptx::mbar_wait(bar(C::kBarKE + ks), ((j / C::kKSt) & 1) ^ 1);
#ifdef SVD_TRACE
          TRACE(3, ptn, j, 70);
#endif
          ptx::mbar_arrive_expect_tx(bar(C::kBarKF + ks), C::kTileBytes);
          load_tile<D>(&tm_k, base + C::kOffK + ks * C::kTileBytes, bar(C::kBarKF + ks), k0, k1,
                       in_head, b, pol_kv);
          ptx::mbar_wait(bar(C::kBarVE + vs), ((j / C::kVSt) & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(bar(C::kBarVF + vs), C::kTileBytes);
          load_tile<D>(&tm_v, base + C::kOffV + vs * C::kTileBytes, bar(C::kBarVF + vs), k0, k1,
                       in_head, b, pol_kv);
        }
      }
      __syncwarp();
      return;
    }
    if (warp == 1) {
      // ---------------------------------------------------------- MMA issuer
      // d=128: the whole warp runs the issue loop (converged, warp-uniform
      // operands) and one elected lane issues each tcgen05 op — no per-MMA
      // divergence wrapper, descriptors in uniform registers (-2.4% layer
      // time).  d=64 (MUFU-bound, measured 2% slower that way): lane 0 alone.
      constexpr bool kElect = D == 128;
      auto mma_s = [&](uint32_t d, uint32_t alo, uint32_t blo, uint32_t hi_, uint32_t id, uint32_t acc) {
        if constexpr (kElect) ptx::mma_ss_e(d, alo, hi_, blo, hi_, id, acc);
        else ptx::mma_ss(d, (uint64_t(hi_) << 32) | alo, (uint64_t(hi_) << 32) | blo, id, acc);
      };
      auto mma_t = [&](uint32_t d, uint32_t a, uint32_t blo, uint32_t hi_, uint32_t id, uint32_t acc) {
        if constexpr (kElect) ptx::mma_ts_e(d, a, blo, hi_, id, acc);
        else ptx::mma_ts(d, a, (uint64_t(hi_) << 32) | blo, id, acc);
      };
      auto commit = [&](uint32_t b) {
        if constexpr (kElect) ptx::mma_commit_e(b);
        else ptx::mma_commit(b);
      };
      if (n_kv > 0 && (kElect || lane == 0)) {
        // smem / TMEM bases laundered once per KV step (asm barrier below):
        // stops ptxas hoisting every stage's descriptors out of the loop and
        // spilling them to local memory under the kernel-wide register cap
        uint32_t sb = base, tb = tmem;
        constexpr uint32_t id_s = ptx::idesc_bf16(128, 128, false);
        constexpr uint32_t id_pv = ptx::idesc_bf16(128, D, true);
        constexpr uint32_t hi = ptx::sw128_hi(1024);
        auto issue_s = [&](int x, int ks) {
          const uint32_t qlo = ptx::sw128_lo(sb + C::kOffQ + x * C::kTileBytes, 16);
          const uint32_t klo = ptx::sw128_lo(sb + C::kOffK + ks * C::kTileBytes, 16);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = ((kk >> 2) * C::kSlabBytes + (kk & 3) * 32) >> 4;
            mma_s(tb + C::col_s(x), qlo + off, klo + off, hi, id_s, kk > 0);
          }
        };
        // O_X += P_X V_j, keys [64*half, 64*half + 64): four K=16 steps
        auto issue_pv_half = [&](int x, int vs, int half, bool acc) {
          const uint32_t vlo = ptx::sw128_lo(sb + C::kOffV + vs * C::kTileBytes, C::kSlabBytes);
          constexpr int kSplit = 2 * (SVD_P_FIRST + 1);  // K=16 steps in the first part
#pragma unroll
          for (int kk = half ? kSplit : 0; kk < (half ? 8 : kSplit); ++kk) {
            mma_t(tb + C::col_o(x), tb + C::col_p(x) + kk * 8, vlo + ((kk * 2048) >> 4), hi, id_pv,
                  (acc || kk > 0) ? 1u : 0u);
          }
        };
        int tn = 0;
        (void)tn;
        auto issue_pv = [&](int x, int vs, int j) {
          if constexpr (kPQuarters<D> || kPLag<D>) {
            // P handed over in 32-key quarters: two K=16 MMAs per quarter
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
              ptx::mbar_wait(bar(C::kBarP0 + 2 * qq + x), j & 1);
              ptx::tc_fence_after();
              const uint32_t vlo = ptx::sw128_lo(sb + C::kOffV + vs * C::kTileBytes, C::kSlabBytes);
#pragma unroll
              for (int k2 = 0; k2 < 2; ++k2) {
                const int kk = qq * 2 + k2;
                mma_t(tb + C::col_o(x), tb + C::col_p(x) + kk * 8, vlo + ((kk * 2048) >> 4), hi, id_pv,
                      (j > 0 || kk > 0) ? 1u : 0u);
              }
            }
            return;
          }
          TRACE(2, tn, j, 30 + x);
          ptx::mbar_wait(bar(C::kBarP0 + x), j & 1);
          TRACE(2, tn, j, 40 + x);
          ptx::tc_fence_after();
          issue_pv_half(x, vs, 0, j > 0);
          ptx::mbar_wait(bar(C::kBarP1 + x), j & 1);
          TRACE(2, tn, j, 50 + x);
          ptx::tc_fence_after();
          issue_pv_half(x, vs, 1, j > 0);
          TRACE(2, tn, j, 10 + x);
        };
        ptx::mbar_wait(bar(C::kBarQ), 0);
        ptx::mbar_wait(bar(C::kBarKF + 0), 0);
        ptx::tc_fence_after();
        issue_s(0, 0);
        commit(bar(C::kBarS + 0));
        issue_s(1, 0);
        commit(bar(C::kBarS + 1));
        commit(bar(C::kBarKE + 0));
        for (int j = 0; j < n_kv; ++j) {
          asm volatile("" : "+r"(sb), "+r"(tb));
          const int vs = j % C::kVSt;
          const int ks1 = (j + 1) % C::kKSt;
          const bool more = j + 1 < n_kv;
          {
            ptx::mbar_wait(bar(C::kBarVF + vs), (j / C::kVSt) & 1);
            // tile A: PV (in two halves, as P arrives), then the next S
            issue_pv(0, vs, j);
            if (!more) commit(bar(C::kBarO + 0));
            if (more) {
              ptx::mbar_wait(bar(C::kBarKF + ks1), ((j + 1) / C::kKSt) & 1);
              TRACE(2, tn, j + 1, 60);
              ptx::tc_fence_after();
              issue_s(0, ks1);
              TRACE(2, tn, j + 1, 61);
              commit(bar(C::kBarS + 0));
              TRACE(2, tn, j + 1, 20);
            }
            // tile B
            issue_pv(1, vs, j);
            commit(bar(C::kBarVE + vs));
            if (!more) commit(bar(C::kBarO + 1));
            if (more) {
              issue_s(1, ks1);
              commit(bar(C::kBarS + 1));
              commit(bar(C::kBarKE + ks1));
              TRACE(2, tn, j + 1, 21);
            }
          }
        }
      }
      __syncwarp();
      named_bar_sync(1, 32 + 256);
      ptx::tc_fence_after();
      ptx::tmem_dealloc(tmem, kTmemCols);
      return;
    }
    return;  // warps 2-3: no role
  }  // warp < 4

  // -------------------------------------------------------------- softmax / epilogue
  ptx::reg_alloc<SVD_REG_HIGH>();
  const int x = (warp - 4) >> 2;           // Q tile A (0) or B (1)
  const int wq = warp & 3;                 // TMEM lane quarter
  const int row = wq * 32 + lane;          // row of the 128-row tile
  const uint32_t lane_off = uint32_t(wq * 32) << 16;
  const int qslot = 2 * x + (row >> 6);
  const int qseg = itp->qseg[2 * x + (row >> 6)];
  const int tok_r = qseg * kSeg + (row & 63);
  const bool row_valid = qseg >= 0 && tok_r < p.n_tokens;
  // element offset of this thread's output row (in O, the packed buffer, or
  // every peer's O)
  int64_t orow;
  if (p.packed && p.n_peers == 0)
    orow = (int64_t(itp->out_base) + qslot * kSeg + (row & 63)) * p.o_sn;
  else
    orow = int64_t(b) * p.o_sb + int64_t(p.o_head_map ? __ldg(p.o_head_map + head) : head) * p.o_sh +
           int64_t(tok_r) * p.o_sn;

  if (n_kv == 0) {
    // SKIP head (attention.py:51-54): exact zeros, no scores, no softmax
    if (row_valid) {
      const uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int c = 0; c < D / 8; ++c) store_row16(p, orow + c * 8, z);
    }
    named_bar_sync(1, 32 + 256);
    return;
  }

  const uint32_t* bits_row = nullptr;
  if constexpr (FINE) {
    const int qb = min(max(tok_r, 0) / p.block_size, p.n_blocks - 1);
    bits_row = p.bits + p.bit_off[itp->group] + int64_t(qb) * p.words_per_row;
  }
  const float sl2 = p.scale_log2;
  const float2 sl2x2 = make_float2(sl2, sl2);
  float m = -INFINITY;  // running max (log2 domain); lazily updated
  float l = 0.f;        // running denominator relative to m
  const KvEntry* kvp = p.kv + itp->kv_begin;
  KvEntry e_next = load_kv(kvp);

#ifdef SVD_TRACE
  int tn = 0;
  const bool tr = (warp == 4 || warp == 8) && lane == 0;
#endif
  // exps of one 32-key chunk of S against the reference max: packed bf16 P
  // (pk) and the running row sums (over the rounded P, SVD_SUM_ROUNDED)
  auto exp_chunk = [&](const float (&sv)[128], int c, const float2 nm, uint32_t (&pk)[16],
                       float2 (&acc)[4]) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float2 xv = ptx::ffma2(make_float2(sv[c * 32 + 2 * i], sv[c * 32 + 2 * i + 1]), sl2x2, nm);
      float2 pv;
      if (emulated_pair<D>(i)) {
        pv = SVD_EMU_DEG2 ? ptx::ex2_poly2_deg2(xv) : ptx::ex2_poly2(xv);
      } else {
        pv.x = ptx::ex2(xv.x);
        pv.y = ptx::ex2(xv.y);
      }
      pk[i] = ptx::pack_bf16(pv.x, pv.y);
      if (!SVD_SUM_ROUNDED) acc[i & 3] = ptx::fadd2(acc[i & 3], pv);
      else if (!(SVD_SUM_AFTER_ST && D == 128)) ptx::acc_bf16x2(acc[i & 3], pk[i]);
    }
  };
  const uint32_t tp = tmem + lane_off + C::col_p(x);
  for (int j = 0; j < n_kv; ++j) {
    const KvEntry e = e_next;
    if (j + 1 < n_kv) e_next = load_kv(kvp + j + 1);  // prefetch behind the S wait
#ifdef SVD_TRACE
    if (tr) TRACE(x, tn, j, 0);
#endif
    ptx::mbar_wait(bar(C::kBarS + x), j & 1);
#ifdef SVD_TRACE
    if (tr) TRACE(x, tn, j, 1);
#endif
    ptx::tc_fence_after();
    float s[128];
    const uint32_t ts = tmem + lane_off + C::col_s(x);
    ptx::tmem_ld32(ts + 0, *reinterpret_cast<float(*)[32]>(&s[0]));
    ptx::tmem_ld32(ts + 32, *reinterpret_cast<float(*)[32]>(&s[32]));
    ptx::tmem_ld32(ts + 64, *reinterpret_cast<float(*)[32]>(&s[64]));
    ptx::tmem_ld32(ts + 96, *reinterpret_cast<float(*)[32]>(&s[96]));
    ptx::tmem_wait_ld();
#ifdef SVD_TRACE
    if (tr) TRACE(x, tn, j, 3);  // S in registers
#endif
    if (!(e.flags & kFlagAll)) apply_mask<FINE>(s, e, qslot, p, bits_row);

    // row max: 8 independent chains, then a short tree
    float mp[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) mp[t] = fmaxf(s[t], s[8 + t]);
#pragma unroll
    for (int i = 16; i < 128; i += 16)
#pragma unroll
      for (int t = 0; t < 8; ++t) mp[t] = fmaxf(mp[t], fmaxf(s[i + t], s[i + 8 + t]));
    const float mx = fmaxf(fmaxf(fmaxf(mp[0], mp[1]), fmaxf(mp[2], mp[3])),
                           fmaxf(fmaxf(mp[4], mp[5]), fmaxf(mp[6], mp[7])));
    const float m_new = fmaxf(m, mx * sl2);
    // lazy rescale: keep a stale max unless it grew by more than 2^8
    const bool resc = m_new > m + 8.0f;
    if (__any_sync(0xffffffffu, resc)) {
      const float alpha = resc ? ptx::ex2(m - m_new) : 1.0f;
      if (j > 0) {
        const uint32_t to = tmem + lane_off + C::col_o(x);
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          float ov[32];
          ptx::tmem_ld32(to + c * 32, ov);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) ov[i] *= alpha;
          ptx::tmem_st32(to + c * 32, ov);
        }
      }
      if (resc) {
        l *= alpha;
        m = m_new;
      }
    }
    const float mref = (m == -INFINITY) ? 0.f : m;
    const float2 nm = make_float2(-mref, -mref);
#ifdef SVD_TRACE
    if (tr) TRACE(x, tn, j, 4);  // max + rescale done
#endif
    float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                     make_float2(0.f, 0.f)};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t pk[16];
      exp_chunk(s, c, nm, pk, acc);
      if constexpr (kPLag<D>) {
        if (c > 0) {  // chunk c-1's store completed under this chunk's exps
          ptx::tmem_wait_st();
          ptx::tc_fence_before();
          ptx::mbar_arrive(bar(C::kBarP0 + 2 * (c - 1) + x));
        }
        ptx::tmem_st16(tp + c * 16, pk);
        if (SVD_SUM_ROUNDED && SVD_SUM_AFTER_ST && D == 128) {
#pragma unroll
          for (int i = 0; i < 16; ++i) ptx::acc_bf16x2(acc[i & 3], pk[i]);
        }
        if (c == 3) {
          ptx::tmem_wait_st();
          ptx::tc_fence_before();
          ptx::mbar_arrive(bar(C::kBarP0 + 2 * 3 + x));
        }
        continue;
      }
      ptx::tmem_st16(tp + c * 16, pk);
      if (SVD_SUM_ROUNDED && SVD_SUM_AFTER_ST && D == 128) {
#pragma unroll
        for (int i = 0; i < 16; ++i) ptx::acc_bf16x2(acc[i & 3], pk[i]);
      }
      if (kPQuarters<D>) {
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        ptx::mbar_arrive(bar(C::kBarP0 + 2 * c + x));
      } else if (c == SVD_P_FIRST || c == 3) {
        // hand P over in two parts: PV on the first part overlaps the exps
        // of the rest
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        ptx::mbar_arrive(bar(c == SVD_P_FIRST ? C::kBarP0 + x : C::kBarP1 + x));
#ifdef SVD_TRACE
        if (tr) TRACE(x, tn, j, c == SVD_P_FIRST ? 6 : 2);  // P part 0 / 1 handed over
#endif
      }
    }
    const float2 a01 = ptx::fadd2(acc[0], acc[1]), a23 = ptx::fadd2(acc[2], acc[3]);
    const float2 a = ptx::fadd2(a01, a23);
    l += a.x + a.y;
  }

  // epilogue: O / l -> bf16 rows
  ptx::mbar_wait(bar(C::kBarO + x), 0);
  ptx::tc_fence_after();
  const uint32_t to = tmem + lane_off + C::col_o(x);
  if (itp->split_group < 0) {
    const float inv = l > 0.f ? 1.0f / l : 0.f;
    float chk = l * 0.f;  // NaN once any accumulator (or l) is Inf / NaN
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      float ov[32];
      ptx::tmem_ld32(to + c * 32, ov);
      ptx::tmem_wait_ld();
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) pk[i] = ptx::pack_bf16(ov[2 * i] * inv, ov[2 * i + 1] * inv);
#pragma unroll
      for (int i = 0; i < 32; ++i) chk = fmaf(ov[i], 0.f, chk);
      if (row_valid) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          store_row16(p, orow + c * 32 + i * 8,
                      make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]));
      }
    }
    if (p.nonfinite && row_valid && chk != 0.f) atomicOr(p.nonfinite, 1);
    if (qseg >= 0) store_row_stats(p, b, head, tok_r, row_valid, m, l);
  } else {
    // split-KV part: publish the partial state (O relative to m, l), then the
    // part that finishes last merges all parts (flash-decoding style):
    // M = max m_p, O = sum 2^(m_p - M) O_p, L = sum 2^(m_p - M) l_p.
    const int sg = itp->split_group, parts = itp->split_parts;
    const int64_t slot = (int64_t(sg) * p.max_split_parts + itp->split_part) * 256 + x * 128 + row;
    float* po = p.split_o + slot * 128;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      float ov[32];
      ptx::tmem_ld32(to + c * 32, ov);
      ptx::tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 8; ++i)
        __stcg(reinterpret_cast<float4*>(po + c * 32) + i,
               make_float4(ov[4 * i], ov[4 * i + 1], ov[4 * i + 2], ov[4 * i + 3]));
    }
    __stcg(reinterpret_cast<float2*>(p.split_ml) + slot, make_float2(m, l));
    __threadfence();
    volatile int* flag = reinterpret_cast<volatile int*>(base_ptr + C::kOffTmemSlot + 4);
    named_bar_sync(2, 256);
    if (threadIdx.x == 128) *flag = (atomicAdd(p.split_tickets + sg, 1) == parts - 1) ? 1 : 0;
    named_bar_sync(2, 256);
    if (*flag) {
      __threadfence();
      const int64_t row0 = int64_t(sg) * p.max_split_parts * 256 + x * 128 + row;
      float mp[kMaxSplitPartsDev], wp[kMaxSplitPartsDev];
      float M = -INFINITY;
#pragma unroll
      for (int q = 0; q < kMaxSplitPartsDev; ++q) {
        mp[q] = -INFINITY;
        if (q < parts) {
          const float2 ml = __ldcg(reinterpret_cast<const float2*>(p.split_ml) + row0 + q * 256);
          mp[q] = ml.x;
          wp[q] = ml.y;  // l_p for now
          M = fmaxf(M, ml.x);
        }
      }
      float L = 0.f;
#pragma unroll
      for (int q = 0; q < kMaxSplitPartsDev; ++q) {
        const float w = (q < parts && mp[q] != -INFINITY) ? ptx::ex2(mp[q] - M) : 0.f;
        if (q < parts) L += w * wp[q];
        wp[q] = w;
      }
      const float inv = L > 0.f ? 1.0f / L : 0.f;
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        float acc[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[i] = 0.f;
#pragma unroll
        for (int q = 0; q < kMaxSplitPartsDev; ++q) {
          if (q >= parts) break;
          const float4* src = reinterpret_cast<const float4*>(p.split_o + (row0 + q * 256) * 128 + c * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 v = __ldcg(src + i);
            acc[4 * i] += wp[q] * v.x;
            acc[4 * i + 1] += wp[q] * v.y;
            acc[4 * i + 2] += wp[q] * v.z;
            acc[4 * i + 3] += wp[q] * v.w;
          }
        }
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) pk[i] = ptx::pack_bf16(acc[2 * i] * inv, acc[2 * i + 1] * inv);
        float chk = L * 0.f;
#pragma unroll
        for (int i = 0; i < 32; ++i) chk = fmaf(acc[i], 0.f, chk);
        if (p.nonfinite && row_valid && chk != 0.f) atomicOr(p.nonfinite, 1);
        if (row_valid) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
            store_row16(p, orow + c * 32 + i * 8,
                        make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]));
        }
      }
      if (qseg >= 0) store_row_stats(p, b, head, tok_r, row_valid, M, L);
      if (threadIdx.x == 128) p.split_tickets[sg] = 0;  // ready for the next launch
    }
  }
  if (p.n_peers > 0) __threadfence_system();  // peer rows visible before the kernel retires
  ptx::tc_fence_before();
  named_bar_sync(1, 32 + 256);
}

// ---------------------------------------------------------------------------
// d=128 half-row pair kernel (`svd_hp_kernel<FINE>`).
//
// The two-tile kernel above keeps S_A, S_B, O_A, O_B in the 512 TMEM columns,
// so P_X must alias S_X and every tile step is the serial chain
// softmax_X(j) -> PV_X(j) -> S_X(j+1) -> softmax_X(j+1): the softmax warps
// wait for S ~36% of the time.  Here one work item (two 128-row Q tiles with
// one KV list) runs on a cluster of two CTAs, ONE tile per CTA, and TMEM
// holds two S buffers and two O accumulators per CTA:
//   S[0], S[1]  double-buffered scores: S(j+1) (even S(j+2)) is computed while
//               the softmax works on S(j)
//   O_0, O_1    the output of key halves 0 / 1: softmax warpgroup h owns the
//               64-key half h of every 128-key step with its own running max,
//               row sum and O_h (no per-step exchange); the epilogue merges
//               O = (2^(m0-M) O_0 + 2^(m1-M) O_1) / (2^(m0-M) l0 + 2^(m1-M) l1)
// The leader CTA issues cta_group::2 MMAs (M = 256: both CTAs' tiles) whose B
// operand is split across the pair — each CTA stages one 64-key segment of
// K (S = Q K^T, N = 128 keys) and one 64-column half of d of V
// (O_h += P_h V_h, N = d) — so the pair reads every K / V tile from L2 once.
//
// CTA (384 threads): warp 0 TMA producer, warp 1 TMEM allocator + MMA issuer
// (leader only), warps 4-7 / 8-11 softmax for key half 0 / 1, epilogue for
// columns [0, 64) / [64, 128) of d.
namespace hp {
constexpr int kQBytes = 128 * 128 * 2;   // this CTA's Q tile: 2 slabs x 128 rows x 128 B
constexpr int kQSlab = 128 * 128;
constexpr int kKStage = 64 * 128 * 2;    // one 64-key segment, all of d (2 slabs x 64 rows)
constexpr int kKSlab = 64 * 128;
constexpr int kVStage = 128 * 64 * 2;    // 128 keys, this CTA's 64 columns of d
constexpr int kKSt = 5, kVSt = 5;
constexpr int kOffQ = 0;
constexpr int kOffK = kOffQ + kQBytes;
constexpr int kOffV = kOffK + kKSt * kKStage;
constexpr int kOffBar = kOffV + kVSt * kVStage;
// barriers: q | kfull kempty | vfull vempty | s_full[2] | p[2 bufs][2 halves] | pv_done[2] | o_full
constexpr int kBarQ = 0;
constexpr int kBarKF = 1, kBarKE = kBarKF + kKSt;
constexpr int kBarVF = kBarKE + kKSt, kBarVE = kBarVF + kVSt;
constexpr int kBarSF = kBarVE + kVSt;
constexpr int kBarP = kBarSF + 2;   // + 2 * buf + h (leader's; both CTAs' warps arrive)
constexpr int kBarPD = kBarP + 4;   // + h: PV_h(j) complete (O_h final through step j)
constexpr int kBarO = kBarPD + 2;
constexpr int kNumBars = kBarO + 1;
constexpr int kOffSlot = kOffBar + kNumBars * 8;
constexpr int kOffXch = (kOffSlot + 16 + 15) & ~15;  // (m, l) per [half][row]
constexpr int kSmemBytes = kOffXch + 2 * 2 * 128 * 4 + 1024;
__device__ constexpr uint32_t col_s(int buf) { return buf ? 128u : 0u; }
__device__ constexpr uint32_t col_o(int h) { return h ? 384u : 256u; }
}  // namespace hp

#ifndef SVD_HP_EMU
#define SVD_HP_EMU 3
#endif


template <bool FINE>
__global__ void __launch_bounds__(kThreads, 1)
    svd_hp_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                  const __grid_constant__ CUtensorMap tm_v, const FwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* base_ptr = smem_raw + (base - raw);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  auto bar = [&](int i) { return base + hp::kOffBar + 8u * uint32_t(i); };
  const int rank = int(ptx::cluster_ctarank());  // = the Q tile of the item this CTA holds
  const bool leader = rank == 0;
  const WorkItem* itp = p.items + (blockIdx.x >> 1);
  const int b = blockIdx.y;
  const int n_kv = itp->kv_count;
  const int head = itp->head;

  if (threadIdx.x == 0) {
    ptx::mbar_init(bar(hp::kBarQ), 1);
    for (int i = 0; i < hp::kKSt; ++i) {
      ptx::mbar_init(bar(hp::kBarKF + i), 1);
      ptx::mbar_init(bar(hp::kBarKE + i), 1);
    }
    for (int i = 0; i < hp::kVSt; ++i) {
      ptx::mbar_init(bar(hp::kBarVF + i), 1);
      ptx::mbar_init(bar(hp::kBarVE + i), 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(bar(hp::kBarSF + i), 1);
      ptx::mbar_init(bar(hp::kBarPD + i), 1);
    }
    for (int i = 0; i < 4; ++i) ptx::mbar_init(bar(hp::kBarP + i), 2 * 4);  // 4 warps x 2 CTAs
    ptx::mbar_init(bar(hp::kBarO), 1);
    ptx::fence_barrier_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc_cg2(base + hp::kOffSlot, kTmemCols);
    ptx::tmem_relinquish_cg2();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();  // the peer's barriers and TMEM exist
  ptx::tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(base_ptr + hp::kOffSlot);
  auto pair_exit = [&]() {
    ptx::tc_fence_before();
    ptx::cluster_sync();  // the leader's MMAs into this CTA's TMEM and all remote arrivals are done
    if (warp == 1) {
      ptx::tc_fence_after();
      ptx::tmem_dealloc_cg2(tmem, kTmemCols);
    }
  };

  if (warp < 4) {
    ptx::reg_dealloc<SVD_REG_LOW>();
    if (warp == 0 && lane == 0 && n_kv > 0) {
      // ---------------------------------------------------------- TMA producer (both CTAs)
      ptx::prefetch_tmap(&tm_q);
      ptx::prefetch_tmap(&tm_k);
      ptx::prefetch_tmap(&tm_v);
      const uint64_t pol_q = ptx::policy_evict_first();
      const uint64_t pol_kv = ptx::policy_evict_last();
      const int in_head = p.in_head_map ? __ldg(p.in_head_map + head) : head;
      const int first = itp->qseg[0];
      if (leader) ptx::mbar_arrive_expect_tx(bar(hp::kBarQ), 2 * hp::kQBytes);
      const uint32_t qbar = ptx::mapa_shared(bar(hp::kBarQ), 0);
#pragma unroll
      for (int slot = 0; slot < 2; ++slot) {
        const int sg = itp->qseg[2 * rank + slot];
        const int seg = sg >= 0 ? sg : first;
#pragma unroll
        for (int slab = 0; slab < 2; ++slab)
          ptx::tma_load_4d_cg2(base + hp::kOffQ + slab * hp::kQSlab + slot * (64 * 128), &tm_q, qbar, slab * 64,
                               seg * kSeg, in_head, b, pol_q);
      }
      const KvEntry* kvp = p.kv + itp->kv_begin;
      for (int j = 0; j < n_kv; ++j) {
        const KvEntry e = load_kv(kvp + j);
        const int k0 = e.kseg0, k1 = e.kseg1 >= 0 ? e.kseg1 : e.kseg0;
        const int ks = j % hp::kKSt, vs = j % hp::kVSt;
        // K: this CTA's 64-key segment (the B rows its half of the S MMA reads)
        ptx::mbar_wait(bar(hp::kBarKE + ks), ((j / hp::kKSt) & 1) ^ 1);
        if (leader) ptx::mbar_arrive_expect_tx(bar(hp::kBarKF + ks), 2 * hp::kKStage);
        const uint32_t kbar = ptx::mapa_shared(bar(hp::kBarKF + ks), 0);
        const int kseg = rank ? k1 : k0;
#pragma unroll
        for (int slab = 0; slab < 2; ++slab)
          ptx::tma_load_4d_cg2(base + hp::kOffK + ks * hp::kKStage + slab * hp::kKSlab, &tm_k, kbar, slab * 64,
                               kseg * kSeg, in_head, b, pol_kv);
        // V: both segments, this CTA's 64 columns of d
        ptx::mbar_wait(bar(hp::kBarVE + vs), ((j / hp::kVSt) & 1) ^ 1);
        if (leader) ptx::mbar_arrive_expect_tx(bar(hp::kBarVF + vs), 2 * hp::kVStage);
        const uint32_t vbar = ptx::mapa_shared(bar(hp::kBarVF + vs), 0);
#pragma unroll
        for (int slot = 0; slot < 2; ++slot)
          ptx::tma_load_4d_cg2(base + hp::kOffV + vs * hp::kVStage + slot * (64 * 128), &tm_v, vbar, rank * 64,
                               (slot ? k1 : k0) * kSeg, in_head, b, pol_kv);
      }
    }
    if (warp == 1 && leader && n_kv > 0) {
      // ---------------------------------------------------------- MMA issuer (leader)
      uint32_t sb = base, tb = tmem;
      constexpr uint32_t id_s = ptx::idesc_bf16(256, 128, false);
      constexpr uint32_t id_pv = ptx::idesc_bf16(256, 128, true);
      constexpr uint32_t hi = ptx::sw128_hi(1024);
      constexpr uint16_t kBoth = 0x3;
      auto issue_s = [&](int buf, int ks) {
        const uint32_t qlo = ptx::sw128_lo(sb + hp::kOffQ, 16);
        const uint32_t klo = ptx::sw128_lo(sb + hp::kOffK + ks * hp::kKStage, 16);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t qoff = ((kk >> 2) * hp::kQSlab + (kk & 3) * 32) >> 4;
          const uint32_t koff = ((kk >> 2) * hp::kKSlab + (kk & 3) * 32) >> 4;
          ptx::mma_ss_cg2_e(tb + hp::col_s(buf), qlo + qoff, hi, klo + koff, hi, id_s, kk > 0);
        }
      };
      ptx::mbar_wait(bar(hp::kBarQ), 0);
      ptx::mbar_wait(bar(hp::kBarKF + 0), 0);
      ptx::tc_fence_after();
      issue_s(0, 0);
      ptx::mma_commit_cg2_mc_e(bar(hp::kBarSF + 0), kBoth);
      ptx::mma_commit_cg2_mc_e(bar(hp::kBarKE + 0), kBoth);
      if (n_kv > 1) {
        ptx::mbar_wait(bar(hp::kBarKF + 1 % hp::kKSt), 0);
        ptx::tc_fence_after();
        issue_s(1, 1 % hp::kKSt);
        ptx::mma_commit_cg2_mc_e(bar(hp::kBarSF + 1), kBoth);
        ptx::mma_commit_cg2_mc_e(bar(hp::kBarKE + 1 % hp::kKSt), kBoth);
      }
      for (int j = 0; j < n_kv; ++j) {
        asm volatile("" : "+r"(sb), "+r"(tb));
        const int buf = j & 1;
        const int vs = j % hp::kVSt;
        ptx::mbar_wait(bar(hp::kBarVF + vs), (j / hp::kVSt) & 1);
        const uint32_t vlo = ptx::sw128_lo(sb + hp::kOffV + vs * hp::kVStage, hp::kVStage);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          // O_h += P_h(j) V_h(j): keys [64h, 64h + 64) of the step
          ptx::mbar_wait(bar(hp::kBarP + 2 * buf + h), (j >> 1) & 1);
          ptx::tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            ptx::mma_ts_cg2_e(tb + hp::col_o(h), tb + hp::col_s(buf) + 64 * h + kk * 8,
                              vlo + ((h * 8192 + kk * 2048) >> 4), hi, id_pv, (j > 0 || kk > 0) ? 1u : 0u);
          ptx::mma_commit_cg2_mc_e(bar(hp::kBarPD + h), kBoth);
        }
        ptx::mma_commit_cg2_mc_e(bar(hp::kBarVE + vs), kBoth);
        if (j + 2 < n_kv) {
          // S(j+2) into the buffer P(j) occupied: the in-order tensor pipe
          // runs it after both PV halves have read P(j)
          const int ks = (j + 2) % hp::kKSt;
          ptx::mbar_wait(bar(hp::kBarKF + ks), ((j + 2) / hp::kKSt) & 1);
          ptx::tc_fence_after();
          issue_s(buf, ks);
          ptx::mma_commit_cg2_mc_e(bar(hp::kBarSF + buf), kBoth);
          ptx::mma_commit_cg2_mc_e(bar(hp::kBarKE + ks), kBoth);
        }
      }
      ptx::mma_commit_cg2_mc_e(bar(hp::kBarO), kBoth);
    }
    __syncwarp();
    pair_exit();
    return;
  }

  // -------------------------------------------------------------- softmax (key half h) / epilogue
  ptx::reg_alloc<SVD_REG_HIGH>();
  const int h = (warp - 4) >> 2;
  const int wq = warp & 3;
  const int row = wq * 32 + lane;
  const uint32_t lane_off = uint32_t(wq * 32) << 16;
  const int x = rank;
  const int qslot = 2 * x + (row >> 6);
  const int qseg = itp->qseg[qslot];
  const int tok_r = qseg * kSeg + (row & 63);
  const bool row_valid = qseg >= 0 && tok_r < p.n_tokens;
  int64_t orow;
  if (p.packed && p.n_peers == 0)
    orow = (int64_t(itp->out_base) + qslot * kSeg + (row & 63)) * p.o_sn;
  else
    orow = int64_t(b) * p.o_sb + int64_t(p.o_head_map ? __ldg(p.o_head_map + head) : head) * p.o_sh +
           int64_t(tok_r) * p.o_sn;
  orow += 64 * h;  // this warpgroup's 64 columns of d
  if (n_kv == 0) {
    // SKIP head (attention.py:51-54): exact zeros
    if (row_valid) {
      const uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int c = 0; c < 8; ++c) store_row16(p, orow + c * 8, z);
    }
    pair_exit();
    return;
  }
  const uint32_t* bits_row = nullptr;
  if constexpr (FINE) {
    const int qb = min(max(tok_r, 0) / p.block_size, p.n_blocks - 1);
    bits_row = p.bits + p.bit_off[itp->group] + int64_t(qb) * p.words_per_row;
  }
  const float sl2 = p.scale_log2;
  const float2 sl2x2 = make_float2(sl2, sl2);
  float m = -INFINITY;  // this half's running max (log2 domain), lazily updated
  float l = 0.f;        // this half's running denominator relative to m
  const KvEntry* kvp = p.kv + itp->kv_begin;
  KvEntry e_next = load_kv(kvp);
  const uint32_t to = tmem + lane_off + hp::col_o(h);
  const uint32_t p_arrive = ptx::mapa_shared(bar(hp::kBarP), 0);  // the leader's P barriers
  for (int j = 0; j < n_kv; ++j) {
    const KvEntry e = e_next;
    if (j + 1 < n_kv) e_next = load_kv(kvp + j + 1);
    const int buf = j & 1;
    const uint32_t ts = tmem + lane_off + hp::col_s(buf) + 64u * uint32_t(h);
    ptx::mbar_wait(bar(hp::kBarSF + buf), (j >> 1) & 1);
    ptx::tc_fence_after();
    float s[64];
    ptx::tmem_ld32(ts + 0, *reinterpret_cast<float(*)[32]>(&s[0]));
    ptx::tmem_ld32(ts + 32, *reinterpret_cast<float(*)[32]>(&s[32]));
    ptx::tmem_wait_ld();
    if (!(e.flags & kFlagAll)) {
      const int kseg = h ? e.kseg1 : e.kseg0;
      const bool on = ((e.flags >> (2 * qslot + h)) & 1u) && kseg >= 0;
      const int lim = on ? min(kSeg, p.n_tokens - kseg * kSeg) : 0;
      if constexpr (FINE) {
        const uint64_t mk = fine_segment_mask(kseg, lim, p, bits_row);
        const uint32_t w0 = uint32_t(mk), w1 = uint32_t(mk >> 32);
#pragma unroll
        for (int i = 0; i < 64; ++i)
          if (!((((i < 32) ? w0 : w1) >> (i & 31)) & 1u)) s[i] = -INFINITY;
      } else {
#pragma unroll
        for (int i = 0; i < 64; ++i)
          if (i >= lim) s[i] = -INFINITY;
      }
    }
    float mp[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) mp[t] = fmaxf(s[t], s[8 + t]);
#pragma unroll
    for (int i = 16; i < 64; i += 16)
#pragma unroll
      for (int t = 0; t < 8; ++t) mp[t] = fmaxf(mp[t], fmaxf(s[i + t], s[i + 8 + t]));
    const float mx = fmaxf(fmaxf(fmaxf(mp[0], mp[1]), fmaxf(mp[2], mp[3])),
                           fmaxf(fmaxf(mp[4], mp[5]), fmaxf(mp[6], mp[7])));
    const float m_new = fmaxf(m, mx * sl2);
    const bool resc = m_new > m + 8.0f;  // lazy rescale: keep a stale max unless it grew by > 2^8
    if (__any_sync(0xffffffffu, resc)) {
      const float alpha = resc ? ptx::ex2(m - m_new) : 1.0f;
      if (j > 0) {
        // O_h is final through step j-1 once PV_h(j-1) completes
        ptx::mbar_wait(bar(hp::kBarPD + h), (j - 1) & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          float ov[16];
          ptx::tmem_ld16(to + c * 16, ov);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) ov[i] *= alpha;
          ptx::tmem_st16(to + c * 16, *reinterpret_cast<const uint32_t(*)[16]>(ov));
        }
      }
      if (resc) {
        l *= alpha;
        m = m_new;
      }
    }
    const float mref = (m == -INFINITY) ? 0.f : m;
    const float2 nm = make_float2(-mref, -mref);
    float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                     make_float2(0.f, 0.f)};
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float2 xv = ptx::ffma2(make_float2(s[c * 32 + 2 * i], s[c * 32 + 2 * i + 1]), sl2x2, nm);
        float2 pv;
        if (SVD_HP_EMU > 0 && (i & 7) < SVD_HP_EMU) {
          pv = ptx::ex2_poly2_deg2(xv);
        } else {
          pv.x = ptx::ex2(xv.x);
          pv.y = ptx::ex2(xv.y);
        }
        pk[i] = ptx::pack_bf16(pv.x, pv.y);
        ptx::acc_bf16x2(acc[i & 3], pk[i]);
      }
      // P_h of keys [32c, 32c + 32) of this half -> columns [16c, 16c + 16)
      // of the half's (already loaded) S columns
      ptx::tmem_st16(ts + c * 16, pk);
    }
    ptx::tmem_wait_st();
    ptx::tc_fence_before();
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive_remote(p_arrive + 8u * uint32_t(2 * buf + h));
    const float2 a = ptx::fadd2(ptx::fadd2(acc[0], acc[1]), ptx::fadd2(acc[2], acc[3]));
    l += a.x + a.y;
  }

  // epilogue: merge the halves' (m, l, O_h); this warpgroup writes d columns [64h, 64h + 64)
  ptx::mbar_wait(bar(hp::kBarO), 0);
  ptx::tc_fence_after();
  float* xch = reinterpret_cast<float*>(base_ptr + hp::kOffXch);  // [h][m|l][128]
  xch[(h * 2 + 0) * 128 + row] = m;
  xch[(h * 2 + 1) * 128 + row] = l;
  named_bar_sync(2, 256);
  const float m_o = xch[((1 - h) * 2 + 0) * 128 + row], l_o = xch[((1 - h) * 2 + 1) * 128 + row];
  const float M = fmaxf(m, m_o);
  const float w_me = m == -INFINITY ? 0.f : ptx::ex2(m - M);
  const float w_ot = m_o == -INFINITY ? 0.f : ptx::ex2(m_o - M);
  const float L = w_me * l + w_ot * l_o;
  const float inv = L > 0.f ? 1.0f / L : 0.f;
  const float w0 = (h == 0 ? w_me : w_ot) * inv, w1 = (h == 0 ? w_ot : w_me) * inv;
  float chk = L * 0.f;  // NaN once any accumulator (or L) is Inf / NaN
  const uint32_t o0 = tmem + lane_off + hp::col_o(0) + 64u * uint32_t(h);
  const uint32_t o1 = tmem + lane_off + hp::col_o(1) + 64u * uint32_t(h);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    float a0[16], a1[16];
    ptx::tmem_ld16(o0 + c * 16, a0);
    ptx::tmem_ld16(o1 + c * 16, a1);
    ptx::tmem_wait_ld();
    uint32_t pk[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      pk[i] = ptx::pack_bf16(a0[2 * i] * w0 + a1[2 * i] * w1, a0[2 * i + 1] * w0 + a1[2 * i + 1] * w1);
#pragma unroll
    for (int i = 0; i < 16; ++i) chk = fmaf(a0[i] + a1[i], 0.f, chk);
    if (row_valid) {
      store_row16(p, orow + c * 16, make_uint4(pk[0], pk[1], pk[2], pk[3]));
      store_row16(p, orow + c * 16 + 8, make_uint4(pk[4], pk[5], pk[6], pk[7]));
    }
  }
  if (p.nonfinite && row_valid && chk != 0.f) atomicOr(p.nonfinite, 1);
  if (h == 0 && qseg >= 0) store_row_stats(p, b, head, tok_r, row_valid, M, L);
  if (p.n_peers > 0) __threadfence_system();
  pair_exit();
}

// Stream-ordered barrier over peer memory (multi-GPU step boundary without a
// host sync): thread r publishes `epoch` into slot `rank` of rank r's flag
// array (release, system scope), then thread r waits until slot r of this
// rank's own array reaches `epoch` (acquire).  Stream order puts it after the
// shard kernel, whose peer stores are fenced system-wide.  A wait longer than
// timeout_ns sets *timed_out and gives up (a dead peer must not hang the GPU).
struct PeerFlags {
  int32_t* f[kMaxPeers];
};
__global__ void svd_peer_barrier_kernel(PeerFlags flags, int n, int rank, int32_t epoch,
                                        int32_t* timed_out, uint64_t timeout_ns) {
  const int r = threadIdx.x;
  if (r >= n) return;
  __threadfence_system();
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(flags.f[r] + rank), "r"(epoch) : "memory");
  const int32_t* mine = flags.f[rank] + r;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    int32_t v;
    asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
    if (int32_t(uint32_t(v) - uint32_t(epoch)) >= 0) break;  // wrap-around safe
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) {
      if (timed_out) atomicExch(timed_out, 1);
      break;
    }
    __nanosleep(200);
  }
}

// Multi-GPU reassembly: packed shard rows -> O[0, head, token, :]
__global__ void svd_unpack_kernel(const int32_t* __restrict__ row_head,
                                  const int32_t* __restrict__ row_token, int64_t n_rows,
                                  const __nv_bfloat16* __restrict__ packed, int64_t prs,
                                  __nv_bfloat16* __restrict__ o, int64_t o_sh, int64_t o_sn,
                                  int vec_per_row) {
  const int64_t gid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t r = gid / vec_per_row;
  const int c = int(gid % vec_per_row);
  if (r >= n_rows) return;
  const int h = row_head[r];
  if (h < 0) return;
  const int t = row_token[r];
  const uint4 v = reinterpret_cast<const uint4*>(packed + r * prs)[c];
  reinterpret_cast<uint4*>(o + int64_t(h) * o_sh + int64_t(t) * o_sn)[c] = v;
}

// Per-head fp64 sum of squared differences (the search's MSE, numerics.py:114-121).
__global__ void svd_sqdiff_kernel(const __nv_bfloat16* __restrict__ a,
                                  const __nv_bfloat16* __restrict__ b, int64_t asb, int64_t ash,
                                  int64_t asn, int64_t bsb, int64_t bsh, int64_t bsn, int B, int64_t N,
                                  int d, double* __restrict__ out) {
  const int h = blockIdx.y;
  const int64_t rows = int64_t(B) * N;
  double acc = 0.0;
  for (int64_t r = int64_t(blockIdx.x) * blockDim.y + threadIdx.y; r < rows;
       r += int64_t(gridDim.x) * blockDim.y) {
    const int bi = int(r / N);
    const int64_t n = r % N;
    const __nv_bfloat16* pa = a + bi * asb + h * ash + n * asn;
    const __nv_bfloat16* pb = b ? b + bi * bsb + h * bsh + n * bsn : nullptr;
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
      const double x = double(__bfloat162float(pa[c])) - (pb ? double(__bfloat162float(pb[c])) : 0.0);
      acc += x * x;
    }
  }
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  __shared__ double part[32];
  const int wid = (threadIdx.y * blockDim.x + threadIdx.x) >> 5;
  if ((threadIdx.x & 31) == 0) part[wid] = acc;
  __syncthreads();
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    double t = 0.0;
    const int nw = (blockDim.x * blockDim.y) >> 5;
    for (int w = 0; w < nw; ++w) t += part[w];
    atomicAdd(out + h, t);
  }
}

// ---------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

// shared with svd_key_mass.cu
int make_tmap(CUtensorMap* map, const void* ptr, const int64_t* st, int64_t B, int64_t H,
                     int64_t N, int D, const char* name) {
  auto enc = get_encode_fn();
  if (!enc) return fail(SVD_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
  if (st[3] != 1) return fail(SVD_ERR_UNSUPPORTED, std::string(name) + ": head_dim stride must be 1");
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) != 0)
    return fail(SVD_ERR_UNSUPPORTED, std::string(name) + ": base pointer not 16-byte aligned");
  cuuint64_t dims[4] = {cuuint64_t(D), cuuint64_t(N), cuuint64_t(H), cuuint64_t(B)};
  cuuint64_t strides[3] = {cuuint64_t(st[2] * 2), cuuint64_t(st[1] * 2), cuuint64_t(st[0] * 2)};
  for (int i = 0; i < 3; ++i)
    if (strides[i] % 16 != 0 && dims[i + 1] > 1)
      return fail(SVD_ERR_UNSUPPORTED, std::string(name) + ": strides must be 16-byte multiples");
  for (int i = 0; i < 3; ++i)
    if (dims[i + 1] == 1) strides[i] = std::max<cuuint64_t>(strides[i], 16) / 16 * 16;
  cuuint32_t box[4] = {64, 64, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(SVD_ERR_CUDA, std::string(name) + ": cuTensorMapEncodeTiled failed (" +
                                  std::to_string(int(r)) + ")");
  return SVD_OK;
}

static int cuda_fail(cudaError_t e, const char* what) {
  return fail(SVD_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

static int ensure_device_tables(const svd_plan* P, DeviceTables** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  std::lock_guard<std::mutex> lock(P->mu);
  auto it = P->dev.find(dev);
  if (it != P->dev.end()) {
    *out = &it->second;
    return SVD_OK;
  }
  DeviceTables t;
  auto upload = [&](void** dst, const void* src, size_t bytes) -> cudaError_t {
    if (bytes == 0) bytes = 16;
    cudaError_t err = cudaMalloc(dst, bytes);
    if (err != cudaSuccess) return err;
    if (src) return cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
    return cudaMemset(*dst, 0, bytes);
  };
  if ((e = upload(&t.items, P->items.data(), P->items.size() * sizeof(WorkItem))) != cudaSuccess ||
      (e = upload(&t.kv, P->kv.empty() ? nullptr : P->kv.data(), P->kv.size() * sizeof(KvEntry))) !=
          cudaSuccess ||
      (e = upload(&t.bits, P->fine_bits.empty() ? nullptr : P->fine_bits.data(),
                  P->fine_bits.size() * 4)) != cudaSuccess ||
      (e = upload(&t.bit_off, P->fine_bit_off.data(), P->fine_bit_off.size() * 8)) != cudaSuccess)
    return cuda_fail(e, "plan upload");
  if (P->n_split_groups > 0) {
    const size_t parts = size_t(P->n_split_groups) * size_t(P->max_split_parts) * 256;
    if ((e = upload(&t.split_scratch, nullptr, parts * (128 + 2) * sizeof(float))) != cudaSuccess ||
        (e = upload(&t.split_tickets, nullptr, size_t(P->n_split_groups) * sizeof(int32_t))) != cudaSuccess)
      return cuda_fail(e, "split-KV scratch");
  }
  t.n_items = int64_t(P->items.size());
  auto res = P->dev.emplace(dev, t);
  *out = &res.first->second;
  return SVD_OK;
}

void release_device_tables(const svd_plan* P) {
  std::lock_guard<std::mutex> lock(P->mu);
  int cur = 0;
  cudaGetDevice(&cur);
  for (auto& kv : P->dev) {
    cudaSetDevice(kv.first);
    cudaFree(kv.second.items);
    cudaFree(kv.second.kv);
    cudaFree(kv.second.bits);
    cudaFree(kv.second.bit_off);
    cudaFree(kv.second.split_scratch);
    cudaFree(kv.second.split_tickets);
  }
  P->dev.clear();
  cudaSetDevice(cur);
}

// d=128 half-row pair kernel only with SVD_HP=1: correct (the GPU suite runs
// it) and free of the per-tile S wait, but measured 2-3% slower than the
// two-tile kernel (profiles/r2/KERNEL_NOTES_r2.md)
static bool use_hp() {
  const char* v = std::getenv("SVD_HP");
  return v && std::strcmp(v, "1") == 0;
}

template <bool FINE>
static cudaError_t launch_hp(const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
                             const FwdParams& prm, int64_t n_items, int batch, cudaStream_t stream) {
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(unsigned(2 * n_items), unsigned(batch));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = hp::kSmemBytes;
  cfg.stream = stream;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, svd_hp_kernel<FINE>, mq, mk, mv, prm);
}

template <int D>
static int launch_fwd(const svd_plan* P, DeviceTables* T, const svd_fwd_args& a, cudaStream_t stream,
                      void* const* peers = nullptr, int n_peers = 0) {
  using C = KCfg<D>;
  CUtensorMap mq, mk, mv;
  const int64_t N = P->grid.n, H = P->n_heads;
  const int64_t Hin = a.in_heads > 0 ? a.in_heads : H;
  const int batch = a.batch, head_dim = a.head_dim;
  void* o = a.o;
  const int64_t* os = a.o_strides;
  int st;
  if ((st = make_tmap(&mq, a.q, a.q_strides, batch, Hin, N, D, "q"))) return st;
  if ((st = make_tmap(&mk, a.k, a.k_strides, batch, Hin, N, D, "k"))) return st;
  if ((st = make_tmap(&mv, a.v, a.v_strides, batch, Hin, N, D, "v"))) return st;
  static bool attr_set[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(svd_fwd_kernel<D, false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(svd_fwd_kernel<D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               C::kSmemBytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
    attr_set[dev] = true;
  }
  FwdParams prm{};
  prm.items = static_cast<const WorkItem*>(T->items);
  prm.kv = static_cast<const KvEntry*>(T->kv);
  prm.bits = P->fine ? static_cast<const uint32_t*>(T->bits) : nullptr;
  prm.bit_off = static_cast<const int64_t*>(T->bit_off);
  prm.o = static_cast<__nv_bfloat16*>(o);
  prm.o_sb = os[0];
  prm.o_sh = os[1];
  prm.o_sn = os[2];
  prm.n_tokens = int(N);
  prm.block_size = int(P->grid.bs);
  prm.words_per_row = int((P->grid.nb + 31) / 32);
  prm.n_blocks = int(P->grid.nb);
  prm.packed = P->sharded ? 1 : 0;
  prm.scale_log2 = float(1.4426950408889634 / std::sqrt(double(head_dim)));
  prm.n_peers = n_peers;
  prm.o_head_map = a.o_head_map;
  prm.nonfinite = reinterpret_cast<int*>(a.nonfinite);
  prm.in_head_map = a.in_head_map;
  prm.row_stats = a.row_stats;
  prm.stats_heads = a.row_stats ? a.stats_heads : 0;
  prm.n_tiles128 = int((N + 127) / 128);
  if (P->n_split_groups > 0) {
    const size_t rows = size_t(P->n_split_groups) * size_t(P->max_split_parts) * 256;
    prm.split_o = static_cast<float*>(T->split_scratch);
    prm.split_ml = prm.split_o + rows * 128;
    prm.split_tickets = static_cast<int*>(T->split_tickets);
    prm.max_split_parts = P->max_split_parts;
  }
  for (int r = 0; r < n_peers; ++r) prm.peer_o[r] = static_cast<__nv_bfloat16*>(peers[r]);
  if (T->n_items == 0) return SVD_OK;
  if (D == 128 && P->n_split_groups == 0 && use_hp()) {
    static bool hp_attr[64] = {false};
    if (dev < 64 && !hp_attr[dev]) {
      cudaError_t e = cudaFuncSetAttribute(svd_hp_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           hp::kSmemBytes);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(svd_hp_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, hp::kSmemBytes);
      if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute (half-row pair kernel)");
      hp_attr[dev] = true;
    }
    cudaError_t e = P->fine ? launch_hp<true>(mq, mk, mv, prm, T->n_items, batch, stream)
                            : launch_hp<false>(mq, mk, mv, prm, T->n_items, batch, stream);
    if (e != cudaSuccess) return cuda_fail(e, "svd_hp_kernel launch");
    return SVD_OK;
  }
  dim3 grid(unsigned(T->n_items), unsigned(batch));
  if (P->fine) {
    svd_fwd_kernel<D, true><<<grid, kThreads, C::kSmemBytes, stream>>>(mq, mk, mv, prm);
  } else {
    svd_fwd_kernel<D, false><<<grid, kThreads, C::kSmemBytes, stream>>>(mq, mk, mv, prm);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "svd_fwd_kernel launch");
  return SVD_OK;
}

}  // namespace svd

using namespace svd;

extern "C" {

const char* svd_version(void) { return "svdit_b200 0.1.0 sm_100a tcgen05/TMA"; }

static int check_args(const svd_plan* P, const svd_fwd_args* a) {
  if (!P) return fail(SVD_ERR_CONFIG, "plan is NULL");
  if (!a) return fail(SVD_ERR_CONFIG, "args is NULL");
  if (a->dtype != 0) return fail(SVD_ERR_UNSUPPORTED, "only bf16 (dtype 0) is supported");
  if (a->head_dim < 1 || a->head_dim > a->tensor_dim)
    return fail(SVD_ERR_SHAPE, "head_dim must be in [1, tensor_dim]");
  if (a->batch < 1) return fail(SVD_ERR_SHAPE, "batch must be >= 1");
  if (a->in_heads < 0) return fail(SVD_ERR_SHAPE, "in_heads must be >= 0");
  if (a->in_heads > 0 && a->in_heads != P->n_heads && !a->in_head_map)
    return fail(SVD_ERR_CONFIG, "in_heads differs from the plan's heads: give in_head_map");
  if (a->row_stats && (a->stats_heads < 1 || a->stats_heads > P->n_heads))
    return fail(SVD_ERR_CONFIG, "stats_heads must be in [1, plan heads]");
  if (!a->q || !a->k || !a->v) return fail(SVD_ERR_CONFIG, "NULL tensor pointer");
  if (a->tensor_dim != 64 && a->tensor_dim != 128)
    return fail(SVD_ERR_UNSUPPORTED,
                "tensor_dim " + std::to_string(a->tensor_dim) + " unsupported (64 or 128; pad)");
  return SVD_OK;
}

int svd_attn_fwd_args(const svd_plan* P, const svd_fwd_args* a, void* stream) {
  int st = check_args(P, a);
  if (st) return st;
  if (P->sharded && a->batch != 1) return fail(SVD_ERR_UNSUPPORTED, "shard plans run with batch 1");
  if (P->sharded && a->o_head_map) return fail(SVD_ERR_UNSUPPORTED, "shard plans write packed rows");
  if (!a->o) return fail(SVD_ERR_CONFIG, "NULL tensor pointer");
  if (a->o_strides[3] != 1 || (a->o_strides[2] * 2) % 16 != 0 ||
      (reinterpret_cast<uintptr_t>(a->o) & 15) != 0)
    return fail(SVD_ERR_UNSUPPORTED, "o: rows must be contiguous and 16-byte aligned");
  DeviceTables* T = nullptr;
  if ((st = ensure_device_tables(P, &T))) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return a->tensor_dim == 64 ? launch_fwd<64>(P, T, *a, s) : launch_fwd<128>(P, T, *a, s);
}

static svd_fwd_args make_args(const void* q, const void* k, const void* v, void* o, const int64_t* qs,
                              const int64_t* ks, const int64_t* vs, const int64_t* os, int32_t batch,
                              int32_t head_dim, int32_t tensor_dim, int32_t dtype) {
  svd_fwd_args a{};
  a.q = q;
  a.k = k;
  a.v = v;
  a.o = o;
  for (int i = 0; i < 4; ++i) {
    a.q_strides[i] = qs[i];
    a.k_strides[i] = ks[i];
    a.v_strides[i] = vs[i];
    a.o_strides[i] = os[i];
  }
  a.batch = batch;
  a.head_dim = head_dim;
  a.tensor_dim = tensor_dim;
  a.dtype = dtype;
  return a;
}

int svd_attn_fwd_v2(const svd_plan* P, const void* q, const void* k, const void* v, void* o,
                    const int64_t* q_strides, const int64_t* k_strides, const int64_t* v_strides,
                    const int64_t* o_strides, int32_t batch, int32_t head_dim, int32_t tensor_dim,
                    int32_t dtype, const int32_t* o_head_map, int32_t* nonfinite, void* stream) {
  if (!q_strides || !k_strides || !v_strides || !o_strides) return fail(SVD_ERR_CONFIG, "NULL strides");
  svd_fwd_args a = make_args(q, k, v, o, q_strides, k_strides, v_strides, o_strides, batch, head_dim,
                             tensor_dim, dtype);
  a.o_head_map = o_head_map;
  a.nonfinite = nonfinite;
  return svd_attn_fwd_args(P, &a, stream);
}

int svd_attn_fwd_ex(const svd_plan* P, const void* q, const void* k, const void* v, void* o,
                    const int64_t* q_strides, const int64_t* k_strides, const int64_t* v_strides,
                    const int64_t* o_strides, int32_t batch, int32_t head_dim, int32_t tensor_dim,
                    int32_t dtype, const int32_t* o_head_map, void* stream) {
  return svd_attn_fwd_v2(P, q, k, v, o, q_strides, k_strides, v_strides, o_strides, batch, head_dim,
                         tensor_dim, dtype, o_head_map, nullptr, stream);
}

int svd_attn_fwd(const svd_plan* P, const void* q, const void* k, const void* v, void* o,
                 const int64_t* q_strides, const int64_t* k_strides, const int64_t* v_strides,
                 const int64_t* o_strides, int32_t batch, int32_t head_dim, int32_t tensor_dim,
                 int32_t dtype, void* stream) {
  return svd_attn_fwd_ex(P, q, k, v, o, q_strides, k_strides, v_strides, o_strides, batch, head_dim,
                         tensor_dim, dtype, nullptr, stream);
}

#ifdef SVD_TRACE
int svd_debug_trace(void* host, int64_t bytes, int32_t reset) {
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess && host) e = cudaMemcpyFromSymbol(host, g_trace, size_t(bytes));
  if (e == cudaSuccess && reset) {
    void* ptr = nullptr;
    e = cudaGetSymbolAddress(&ptr, g_trace);
    if (e == cudaSuccess) e = cudaMemset(ptr, 0, sizeof(g_trace));
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
  }
  return e == cudaSuccess ? SVD_OK : cuda_fail(e, "trace");
}
#endif

int svd_ipc_export(const void* ptr, uint8_t* handle64, int64_t* offset) {
  if (!ptr || !handle64 || !offset) return fail(SVD_ERR_CONFIG, "NULL argument");
  static PFN_cuMemGetAddressRange_v3020 range_fn = nullptr;
  if (!range_fn) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return fail(SVD_ERR_CUDA, "cuMemGetAddressRange unavailable");
    range_fn = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range_fn(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
    return fail(SVD_ERR_CUDA, "cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(handle64, &h, 64);
  *offset = int64_t(reinterpret_cast<CUdeviceptr>(ptr) - base);
  return SVD_OK;
}

int svd_ipc_import(const uint8_t* handle64, int64_t offset, void** ptr) {
  if (!handle64 || !ptr) return fail(SVD_ERR_CONFIG, "NULL argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, 64);
  void* base = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
  *ptr = static_cast<uint8_t*>(base) + offset;
  return SVD_OK;
}

int svd_ipc_close(void* ptr, int64_t offset) {
  if (!ptr) return SVD_OK;
  cudaError_t e = cudaIpcCloseMemHandle(static_cast<uint8_t*>(ptr) - offset);
  return e == cudaSuccess ? SVD_OK : cuda_fail(e, "cudaIpcCloseMemHandle");
}

int svd_attn_fwd_peers(const svd_plan* P, const void* q, const void* k, const void* v,
                       void* const* o_peers, int32_t n_peers, const int64_t* q_strides,
                       const int64_t* k_strides, const int64_t* v_strides,
                       const int64_t* o_strides, int32_t batch, int32_t head_dim,
                       int32_t tensor_dim, int32_t dtype, void* stream) {
  if (n_peers < 1 || n_peers > kMaxPeers || !o_peers)
    return fail(SVD_ERR_CONFIG, "n_peers must be in [1, " + std::to_string(kMaxPeers) + "]");
  if (!q_strides || !k_strides || !v_strides || !o_strides) return fail(SVD_ERR_CONFIG, "NULL strides");
  svd_fwd_args a = make_args(q, k, v, o_peers[0], q_strides, k_strides, v_strides, o_strides, batch,
                             head_dim, tensor_dim, dtype);
  int st = check_args(P, &a);
  if (st) return st;
  if (o_strides[3] != 1 || (o_strides[2] * 2) % 16 != 0)
    return fail(SVD_ERR_UNSUPPORTED, "o: rows must be contiguous and 16-byte aligned");
  for (int r = 0; r < n_peers; ++r)
    if (!o_peers[r] || (reinterpret_cast<uintptr_t>(o_peers[r]) & 15) != 0)
      return fail(SVD_ERR_UNSUPPORTED, "peer O pointers must be non-NULL and 16-byte aligned");
  DeviceTables* T = nullptr;
  if ((st = ensure_device_tables(P, &T))) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return tensor_dim == 64 ? launch_fwd<64>(P, T, a, s, o_peers, n_peers)
                          : launch_fwd<128>(P, T, a, s, o_peers, n_peers);
}

int svd_peer_barrier(int32_t* const* flags, int32_t n_peers, int32_t rank, int32_t epoch,
                     int32_t* timed_out, double timeout_s, void* stream) {
  if (!flags || n_peers < 1 || n_peers > kMaxPeers || rank < 0 || rank >= n_peers)
    return fail(SVD_ERR_CONFIG, "peer barrier: bad flags / n_peers / rank");
  PeerFlags pf{};
  for (int r = 0; r < n_peers; ++r) {
    if (!flags[r] || (reinterpret_cast<uintptr_t>(flags[r]) & 3) != 0)
      return fail(SVD_ERR_CONFIG, "peer barrier: flag arrays must be non-NULL and 4-byte aligned");
    pf.f[r] = flags[r];
  }
  const uint64_t tns = timeout_s > 0 ? uint64_t(timeout_s * 1e9) : uint64_t(30e9);
  svd_peer_barrier_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(pf, n_peers, rank, epoch,
                                                                         timed_out, tns);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "svd_peer_barrier_kernel launch");
  return SVD_OK;
}

int svd_head_sqdiff(const void* a, const void* b, const int64_t* as, const int64_t* bs,
                    int32_t batch, int32_t heads, int64_t n_tokens, int32_t head_dim, double* out,
                    void* stream) {
  if (!a || !out) return fail(SVD_ERR_CONFIG, "NULL tensor pointer");
  if (batch < 1 || heads < 1 || n_tokens < 1 || head_dim < 1) return fail(SVD_ERR_SHAPE, "bad shape");
  if (as[3] != 1 || (b && bs[3] != 1)) return fail(SVD_ERR_UNSUPPORTED, "head_dim stride must be 1");
  const dim3 block(32, 8);
  const int64_t rows = int64_t(batch) * n_tokens;
  const dim3 grid(unsigned(std::min<int64_t>((rows + 7) / 8, 1024)), unsigned(heads));
  svd_sqdiff_kernel<<<grid, block, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(a), static_cast<const __nv_bfloat16*>(b), as[0], as[1], as[2],
      b ? bs[0] : 0, b ? bs[1] : 0, b ? bs[2] : 0, batch, n_tokens, head_dim, out);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "svd_sqdiff_kernel launch");
  return SVD_OK;
}

int svd_unpack_rows(const int32_t* row_head_dev, const int32_t* row_token_dev, int64_t n_rows,
                    const void* packed, int64_t packed_row_stride, void* o, const int64_t* o_strides,
                    int32_t head_dim, void* stream) {
  if (head_dim % 8 != 0) return fail(SVD_ERR_UNSUPPORTED, "head_dim must be a multiple of 8");
  if (n_rows <= 0) return SVD_OK;
  const int vec = head_dim / 8;
  const int64_t total = n_rows * vec;
  const int threads = 256;
  const unsigned blocks = unsigned((total + threads - 1) / threads);
  svd_unpack_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(
      row_head_dev, row_token_dev, n_rows, static_cast<const __nv_bfloat16*>(packed),
      packed_row_stride, static_cast<__nv_bfloat16*>(o), o_strides[1], o_strides[2], vec);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "svd_unpack_kernel launch");
  return SVD_OK;
}

}  // extern "C"
