// sm_100a GEMMs of the vDiT block around the attention operator (SURVEY §8
// row f4): the projections of layer_qkv (model.py:372-391) and layer_finish
// (model.py:394-402), with the element-wise step that follows each one fused
// into its epilogue:
//
//   h [M, D] . Wqkv [D, 3D]  -> bf16, RoPE on the q and k column blocks (model.py:383-388)
//   O [M, D] . Wo   [D, D]   -> fp32, + x            (the attention residual, model.py:398)
//   h2 [M, D] . W1  [D, 4D]  -> bf16, exact GELU     (model.py:400, 357-359)
//   u [M, 4D] . W2  [4D, D]  -> fp32, + a            (the MLP residual, model.py:401)
//
// C[M, N] = A[M, K] B[K, N]: A bf16 row-major (K-major operand), B bf16
// row-major [K, N] (an MN-major operand, the weight as stored), fp32
// accumulation in TMEM.  One persistent CTA per SM walks 128 x 256 output
// tiles (row-major tile order: the CTAs in flight share A row panels, B stays
// L2-resident):
//   warp 0      TMA producer: per 64-deep K step one 128 x 64 A box and four
//               64 x 64 B boxes (SWIZZLE_128B) into a 4-stage ring
//   warp 1      TMEM allocator (2 x 256 columns) + single-thread tcgen05.mma
//               issuer, M=128 N=256 K=16, accumulator double-buffered so the
//               epilogue of tile i overlaps the MMAs of tile i+1
//   warps 4-11  epilogue: two warpgroups, thread = output row = TMEM lane,
//               each warpgroup half of the columns, tcgen05.ld of 32 columns
//               at a time, the fused op, 16-byte global stores
// Bound: the tensor pipe (2*M*N*K FLOPs); operand traffic per K step is 48 KB
// of smem for 4.2 MFLOP (96 B/clk at the tensor rate).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>

#include "svd_plan.h"
#include "svd_ptx.cuh"

namespace svd {
namespace gemm {

constexpr int BM = 128, BN = 256, BK = 64, kStages = 4;
// warps 0 (TMA), 1 (MMA), 2-3 idle, 4-11 epilogue: two warpgroups, each taking
// half of the tile's columns for its 128 rows (TMEM lane quarter = warp % 4)
constexpr int kEpiWarps = 8, kThreads = 32 * (4 + kEpiWarps);
constexpr int kEpiCols = BN / (kEpiWarps / 4);
constexpr int kABytes = BM * BK * 2;             // 16 KB
constexpr int kBBoxBytes = BK * 64 * 2;          // 8 KB: 64 K rows x 64 N columns
constexpr int kBBytes = BK * BN * 2;             // 32 KB
constexpr int kStageBytes = kABytes + kBBytes;   // 48 KB
constexpr int kOffBar = kStages * kStageBytes;
// barriers: full[S] empty[S] acc_full[2] acc_empty[2]
constexpr int kBarFull = 0, kBarEmpty = kStages, kBarAccFull = 2 * kStages, kBarAccEmpty = 2 * kStages + 2;
constexpr int kNumBars = 2 * kStages + 4;
constexpr int kOffSlot = kOffBar + kNumBars * 8;
constexpr int kSmemBytes = kOffSlot + 16 + 1024;
constexpr uint32_t kTmemCols = 512;

enum Epi : int { kBf16 = 0, kRope = 1, kGelu = 2, kF32Resid = 3, kF32 = 4 };

struct Params {
  int M, N, K;
  int tiles_m, tiles_n;
  void* out;
  int64_t ldo;           // elements
  const float* resid;    // kF32Resid: fp32 [M, ldr]
  int64_t ldr;
  const float2* rope;    // kRope: (cos, sin) [n_tokens][head_dim / 2]
  int rope_cols;         // columns [0, rope_cols) get RoPE (q and k blocks)
  int head_dim;
  int n_tokens;
};

// GELU(x) = x/2 (1 + erf(x / sqrt 2)) (model.py:357-359).  SVD_GELU_AS: erf by
// Abramowitz-Stegun 7.1.26 (|error| <= 1.5e-7: 1 MUFU rcp, 1 MUFU ex2, 6 FMA)
// instead of the libdevice erff polynomial.
#ifndef SVD_GELU_AS
#define SVD_GELU_AS 1
#endif
__device__ __forceinline__ float gelu_exact(float x) {
  if (SVD_GELU_AS) {
    const float z = fabsf(x) * 0.70710678118654752f;
    const float t = __frcp_rn(fmaf(0.3275911f, z, 1.0f));
    float poly = fmaf(1.061405429f, t, -1.453152027f);
    poly = fmaf(poly, t, 1.421413741f);
    poly = fmaf(poly, t, -0.284496736f);
    poly = fmaf(poly, t, 0.254829592f);
    poly *= t;
    const float e = exp2f(-z * z * 1.4426950408889634f);
    const float erf_abs = fmaf(-poly, e, 1.0f);
    const float erf_x = copysignf(erf_abs, x);
    return 0.5f * x * (1.f + erf_x);
  }
  return 0.5f * x * (1.f + erff(x * 0.70710678118654752f));
}

// kEpiCols columns of one output row (this thread's TMEM lane) starting at
// n0: tcgen05.ld of 32 columns at a time, the fused element-wise op, 16-byte
// global stores.
template <int EPI>
__device__ __forceinline__ void epilogue_row(const Params& p, uint32_t acc, int row, int n0, bool row_ok,
                                             int tok) {
  // kF32Resid: the residual row segment of chunk c+1 is loaded while chunk c
  // is converted and stored (two 128-byte buffers per thread in registers),
  // so the epilogue is not bound by one chunk's load latency at a time
  float4 rbuf[2][8];
  auto load_resid = [&](int c, float4 (&r)[8]) {
    const int col0 = n0 + c * 32;
    if (!row_ok || col0 >= p.N) return;
    const float4* src = reinterpret_cast<const float4*>(p.resid + int64_t(row) * p.ldr + col0);
    const int ncols = min(32, p.N - col0);
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (4 * i < ncols) r[i] = __ldg(src + i);
  };
  if constexpr (EPI == kF32Resid) load_resid(0, rbuf[0]);
#pragma unroll
  for (int c = 0; c < kEpiCols / 32; ++c) {
    if constexpr (EPI == kF32Resid) {
      if (c + 1 < kEpiCols / 32) load_resid(c + 1, rbuf[(c + 1) & 1]);
    }
    float v[32];
    ptx::tmem_ld32(acc + c * 32, v);
    ptx::tmem_wait_ld();
    const int col0 = n0 + c * 32;
    if (!row_ok || col0 >= p.N) continue;
    if constexpr (EPI == kRope) {
      if (col0 < p.rope_cols) {
        const int half = p.head_dim / 2;
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const int hc = (col0 + e) % p.head_dim;
          const float2 cs = __ldg(p.rope + int64_t(tok) * half + (hc >> 1));
          const float x0 = v[e], x1 = v[e + 1];
          v[e] = x0 * cs.x - x1 * cs.y;
          v[e + 1] = x0 * cs.y + x1 * cs.x;
        }
      }
    }
    if constexpr (EPI == kGelu) {
#pragma unroll
      for (int e = 0; e < 32; ++e) v[e] = gelu_exact(v[e]);
    }
    const int ncols = min(32, p.N - col0);  // N % 8 == 0 (host check)
    if constexpr (EPI == kF32Resid || EPI == kF32) {
      float* o = static_cast<float*>(p.out) + int64_t(row) * p.ldo + col0;
      if constexpr (EPI == kF32Resid) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (4 * i >= ncols) break;
          const float4 w = rbuf[c & 1][i];
          v[4 * i] += w.x;
          v[4 * i + 1] += w.y;
          v[4 * i + 2] += w.z;
          v[4 * i + 3] += w.w;
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (4 * i >= ncols) break;
        reinterpret_cast<float4*>(o)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
      }
    } else {
      __nv_bfloat16* o = static_cast<__nv_bfloat16*>(p.out) + int64_t(row) * p.ldo + col0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (8 * i >= ncols) break;
        reinterpret_cast<uint4*>(o)[i] =
            make_uint4(ptx::pack_bf16(v[8 * i], v[8 * i + 1]), ptx::pack_bf16(v[8 * i + 2], v[8 * i + 3]),
                       ptx::pack_bf16(v[8 * i + 4], v[8 * i + 5]), ptx::pack_bf16(v[8 * i + 6], v[8 * i + 7]));
      }
    }
  }
}

// CM > 1: a cluster of CM CTAs along M works on CM consecutive 128-row tiles
// of one 256-column panel; each CTA loads 4/CM of the B boxes and multicasts
// them to the whole cluster, so B crosses L2 -> SM once per cluster instead
// of once per CTA.  A stage is refilled only after every CTA of the cluster
// has consumed it (the MMA commit arrives on the empty barrier of all CTAs).
template <int EPI, int CM>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                const Params p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* base_ptr = smem_raw + (base - raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto bar = [&](int i) { return base + kOffBar + 8u * uint32_t(i); };
  const int k_steps = (p.K + BK - 1) / BK;
  // tile groups: CM consecutive M tiles of one N panel, one per cluster rank
  const int groups_m = (p.tiles_m + CM - 1) / CM;
  const int n_groups = groups_m * p.tiles_n;
  const int rank = CM > 1 ? int(ptx::cluster_ctarank()) : 0;
  const int g0 = CM > 1 ? int(ptx::cluster_id_x()) : int(blockIdx.x);
  const int g_step = CM > 1 ? int(ptx::n_clusters_x()) : int(gridDim.x);
  constexpr uint16_t kMask = uint16_t((1u << CM) - 1u);

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      ptx::mbar_init(bar(kBarFull + i), 1);
      ptx::mbar_init(bar(kBarEmpty + i), CM);  // one MMA commit per cluster CTA
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(bar(kBarAccFull + i), 1);
      ptx::mbar_init(bar(kBarAccEmpty + i), 32 * kEpiWarps);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc(base + kOffSlot, kTmemCols);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if constexpr (CM > 1) ptx::cluster_sync();  // peers' barriers exist before any multicast
  ptx::tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(base_ptr + kOffSlot);

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      ptx::prefetch_tmap(&tm_a);
      ptx::prefetch_tmap(&tm_b);
      // an A row panel is read by every N panel (tiles_n CTAs, nearly at the
      // same time): evict_first would send most of those reads to DRAM
      // (measured 14.7 GB of DRAM reads for a 0.8 GB QKV projection)
#ifndef SVD_GEMM_A_POLICY
#define SVD_GEMM_A_POLICY 1
#endif
      const uint64_t pol_a = SVD_GEMM_A_POLICY == 0 ? ptx::policy_evict_first()
                             : SVD_GEMM_A_POLICY == 1 ? ptx::policy_evict_normal()
                                                      : ptx::policy_evict_last();
      const uint64_t pol_b = ptx::policy_evict_last();
      int step = 0;
      for (int g = g0; g < n_groups; g += g_step) {
        const int m0 = ((g / p.tiles_n) * CM + rank) * BM, n0 = (g % p.tiles_n) * BN;
        for (int ks = 0; ks < k_steps; ++ks, ++step) {
          const int s = step % kStages;
          ptx::mbar_wait(bar(kBarEmpty + s), ((step / kStages) & 1) ^ 1);
          const uint32_t dst = base + s * kStageBytes;
          ptx::mbar_arrive_expect_tx(bar(kBarFull + s), kStageBytes);
          ptx::tma_load_2d(dst, &tm_a, bar(kBarFull + s), ks * BK, m0, pol_a);
          if constexpr (CM == 1) {
#pragma unroll
            for (int i = 0; i < BN / 64; ++i)
              ptx::tma_load_2d(dst + kABytes + i * kBBoxBytes, &tm_b, bar(kBarFull + s), n0 + 64 * i, ks * BK,
                               pol_b);
          } else {
#pragma unroll
            for (int j = 0; j < (BN / 64) / CM; ++j) {
              const int i = rank * ((BN / 64) / CM) + j;
              ptx::tma_load_2d_mc(dst + kABytes + i * kBBoxBytes, &tm_b, bar(kBarFull + s), n0 + 64 * i, ks * BK,
                                  kMask, pol_b);
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16(BM, BN, true);
      constexpr uint32_t hi = ptx::sw128_hi(1024);
      int step = 0, it = 0;
      for (int g = g0; g < n_groups; g += g_step, ++it) {
        const int buf = it & 1;
        ptx::mbar_wait(bar(kBarAccEmpty + buf), ((it >> 1) & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t acc = tmem + uint32_t(buf * BN);
        for (int ks = 0; ks < k_steps; ++ks, ++step) {
          const int s = step % kStages;
          ptx::mbar_wait(bar(kBarFull + s), (step / kStages) & 1);
          ptx::tc_fence_after();
          const uint32_t a_lo = ptx::sw128_lo(base + s * kStageBytes, 16);
          const uint32_t b_lo = ptx::sw128_lo(base + s * kStageBytes + kABytes, kBBoxBytes);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            ptx::mma_ss(acc, (uint64_t(hi) << 32) | (a_lo + ((kk * 32) >> 4)),
                        (uint64_t(hi) << 32) | (b_lo + ((kk * 2048) >> 4)), idesc, (ks | kk) ? 1u : 0u);
          if constexpr (CM == 1) ptx::mma_commit(bar(kBarEmpty + s));
          else ptx::mma_commit_mc(bar(kBarEmpty + s), kMask);  // the stage is free once every CTA is done
        }
        ptx::mma_commit(bar(kBarAccFull + buf));
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int row_in_tile = (warp & 3) * 32 + lane;
    const uint32_t lane_off = uint32_t((warp & 3) * 32) << 16;
    const int col_off = ((warp - 4) >> 2) * kEpiCols;
    int it = 0;
    for (int g = g0; g < n_groups; g += g_step, ++it) {
      const int buf = it & 1;
      const int m0 = ((g / p.tiles_n) * CM + rank) * BM, n0 = (g % p.tiles_n) * BN;
      const int row = m0 + row_in_tile;
      ptx::mbar_wait(bar(kBarAccFull + buf), (it >> 1) & 1);
      ptx::tc_fence_after();
      const uint32_t acc = tmem + lane_off + uint32_t(buf * BN + col_off);
      const bool row_ok = row < p.M;
      const int tok = row_ok ? row % p.n_tokens : 0;
      epilogue_row<EPI>(p, acc, row, n0 + col_off, row_ok, tok);
      ptx::tc_fence_before();
      ptx::mbar_arrive(bar(kBarAccEmpty + buf));
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if constexpr (CM > 1) ptx::cluster_sync();  // no CTA leaves while peers may still multicast into it
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, kTmemCols);
  }
}

// ---------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a cluster of two CTAs on one TPC computes a
// 256 x 256 tile with M=256 N=256 MMAs issued by the leader CTA.  Each CTA
// stages its own 128 rows of A and HALF of B (128 columns) per K step — the
// tensor cores of the pair read both halves — so per SM the smem fill and
// the L2 -> SM traffic of B halve and a stage is 32 KB (6 stages).  Each
// CTA's TMEM holds its 128 rows x 256 columns (double-buffered).
//   leader:  full[s] (expects both CTAs' bytes), acc_empty[b] (512 arrivals:
//            both CTAs' epilogue threads)
//   both:    empty[s], acc_full[b] (the leader's commits multicast to the pair)
constexpr int k2Stages = 6;
constexpr int k2ABytes = 128 * BK * 2;           // 16 KB: this CTA's 128 rows
constexpr int k2BBytes = BK * 128 * 2;           // 16 KB: this CTA's 128 columns
constexpr int k2StageBytes = k2ABytes + k2BBytes;
constexpr int k2OffBar = k2Stages * k2StageBytes;
constexpr int k2BarFull = 0, k2BarEmpty = k2Stages, k2BarAccFull = 2 * k2Stages, k2BarAccEmpty = 2 * k2Stages + 2;
constexpr int k2NumBars = 2 * k2Stages + 4;
constexpr int k2OffSlot = k2OffBar + k2NumBars * 8;
constexpr int k2SmemBytes = k2OffSlot + 16 + 1024;

template <int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                 const Params p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* base_ptr = smem_raw + (base - raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto bar = [&](int i) { return base + k2OffBar + 8u * uint32_t(i); };
  const int k_steps = (p.K + BK - 1) / BK;
  const int rank = int(ptx::cluster_ctarank());
  const bool leader = rank == 0;
  const int pairs_m = (p.tiles_m + 1) / 2;  // 256-row groups
  const int n_groups = pairs_m * p.tiles_n;
  const int g0 = int(ptx::cluster_id_x()), g_step = int(ptx::n_clusters_x());

  if (threadIdx.x == 0) {
    for (int i = 0; i < k2Stages; ++i) {
      ptx::mbar_init(bar(k2BarFull + i), 1);
      ptx::mbar_init(bar(k2BarEmpty + i), 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(bar(k2BarAccFull + i), 1);
      ptx::mbar_init(bar(k2BarAccEmpty + i), 2 * 32 * kEpiWarps);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc_cg2(base + k2OffSlot, kTmemCols);
    ptx::tmem_relinquish_cg2();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();  // both CTAs' barriers and TMEM exist
  ptx::tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(base_ptr + k2OffSlot);

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      ptx::prefetch_tmap(&tm_a);
      ptx::prefetch_tmap(&tm_b);
      const uint64_t pol_a = ptx::policy_evict_normal();
      const uint64_t pol_b = ptx::policy_evict_last();
      int step = 0;
      for (int g = g0; g < n_groups; g += g_step) {
        const int m0 = (g / p.tiles_n) * 256 + rank * 128, n0 = (g % p.tiles_n) * BN + rank * 128;
        for (int ks = 0; ks < k_steps; ++ks, ++step) {
          const int s = step % k2Stages;
          ptx::mbar_wait(bar(k2BarEmpty + s), ((step / k2Stages) & 1) ^ 1);
          const uint32_t full_leader = ptx::mapa_shared(bar(k2BarFull + s), 0);
          if (leader) ptx::mbar_arrive_expect_tx(bar(k2BarFull + s), 2 * k2StageBytes);
          const uint32_t dst = base + s * k2StageBytes;
          ptx::tma_load_2d_cg2(dst, &tm_a, full_leader, ks * BK, m0, pol_a);
#pragma unroll
          for (int i = 0; i < 2; ++i)
            ptx::tma_load_2d_cg2(dst + k2ABytes + i * kBBoxBytes, &tm_b, full_leader, n0 + 64 * i, ks * BK, pol_b);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader)
    if (leader && lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16(256, BN, true);
      constexpr uint32_t hi = ptx::sw128_hi(1024);
      int step = 0, it = 0;
      for (int g = g0; g < n_groups; g += g_step, ++it) {
        const int buf = it & 1;
        ptx::mbar_wait(bar(k2BarAccEmpty + buf), ((it >> 1) & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t acc = tmem + uint32_t(buf * BN);
        for (int ks = 0; ks < k_steps; ++ks, ++step) {
          const int s = step % k2Stages;
          ptx::mbar_wait(bar(k2BarFull + s), (step / k2Stages) & 1);
          ptx::tc_fence_after();
          const uint32_t a_lo = ptx::sw128_lo(base + s * k2StageBytes, 16);
          const uint32_t b_lo = ptx::sw128_lo(base + s * k2StageBytes + k2ABytes, kBBoxBytes);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            ptx::mma_ss_cg2(acc, (uint64_t(hi) << 32) | (a_lo + ((kk * 32) >> 4)),
                            (uint64_t(hi) << 32) | (b_lo + ((kk * 2048) >> 4)), idesc, (ks | kk) ? 1u : 0u);
          ptx::mma_commit_cg2_mc(bar(k2BarEmpty + s), 0x3);
        }
        ptx::mma_commit_cg2_mc(bar(k2BarAccFull + buf), 0x3);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int row_in_tile = (warp & 3) * 32 + lane;
    const uint32_t lane_off = uint32_t((warp & 3) * 32) << 16;
    const int col_off = ((warp - 4) >> 2) * kEpiCols;
    int it = 0;
    for (int g = g0; g < n_groups; g += g_step, ++it) {
      const int buf = it & 1;
      const int m0 = (g / p.tiles_n) * 256 + rank * 128, n0 = (g % p.tiles_n) * BN;
      const int row = m0 + row_in_tile;
      ptx::mbar_wait(bar(k2BarAccFull + buf), (it >> 1) & 1);
      ptx::tc_fence_after();
      const bool row_ok = row < p.M;
      epilogue_row<EPI>(p, tmem + lane_off + uint32_t(buf * BN + col_off), row, n0 + col_off, row_ok,
                        row_ok ? row % p.n_tokens : 0);
      ptx::tc_fence_before();
      ptx::mbar_arrive_cluster(ptx::mapa_shared(bar(k2BarAccEmpty + buf), 0));
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();  // the pair's MMAs, commits and remote arrivals are all done
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_cg2(tmem, kTmemCols);
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

// 2-D bf16 row-major [rows, cols] (leading dimension ld elements), box
// {64 columns, box_rows rows}, SWIZZLE_128B; out-of-range boxes zero-fill.
static int tmap_2d(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                   const char* name) {
  auto enc = encode_fn();
  if (!enc) return fail(SVD_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) != 0 || (ld * 2) % 16 != 0)
    return fail(SVD_ERR_UNSUPPORTED, std::string(name) + ": 16-byte aligned rows required");
  cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(ld * 2)};
  cuuint32_t box[2] = {64, cuuint32_t(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(SVD_ERR_CUDA, std::string(name) + ": cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  return SVD_OK;
}

int sm_count_dev() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

#ifndef SVD_GEMM_CLUSTER
#define SVD_GEMM_CLUSTER 2
#endif

template <int EPI, int CM>
static int launch_cm(const CUtensorMap& ma, const CUtensorMap& mb, const Params& p, cudaStream_t s) {
  static bool attr[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr[dev]) {
    cudaError_t e =
        cudaFuncSetAttribute(gemm_kernel<EPI, CM>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e == cudaSuccess && CM > 1)
      e = cudaFuncSetAttribute(gemm_kernel<EPI, CM>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return fail(SVD_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    attr[dev] = true;
  }
  const int groups = ((p.tiles_m + CM - 1) / CM) * p.tiles_n;
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CM;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  // persistent: as many clusters as can be resident at once (SMs that cannot
  // pair up inside a GPC would otherwise leave a second wave)
  static int resident[64] = {0};
  if (dev < 64 && resident[dev] == 0) {
    int n = 0;
    cfg.gridDim = dim3(unsigned(CM));
    if (cudaOccupancyMaxActiveClusters(&n, gemm_kernel<EPI, CM>, &cfg) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = sm_count_dev() / CM;
    }
    resident[dev] = n;
  }
  const int clusters = std::min(groups, dev < 64 ? resident[dev] : sm_count_dev() / CM);
  cfg.gridDim = dim3(unsigned(clusters * CM));
  cudaError_t e = cudaLaunchKernelEx(&cfg, gemm_kernel<EPI, CM>, ma, mb, p);
  if (e != cudaSuccess) return fail(SVD_ERR_CUDA, std::string("gemm_kernel launch: ") + cudaGetErrorString(e));
  return SVD_OK;
}

template <int EPI>
static int launch_pair(const CUtensorMap& ma, const CUtensorMap& mb, const Params& p, cudaStream_t s) {
  static bool attr[64] = {false};
  static int resident[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr[dev]) {
    cudaError_t e = cudaFuncSetAttribute(gemm2_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, k2SmemBytes);
    if (e != cudaSuccess) return fail(SVD_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    attr[dev] = true;
  }
  const int groups = ((p.tiles_m + 1) / 2) * p.tiles_n;
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = k2SmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (dev < 64 && resident[dev] == 0) {
    int n = 0;
    cfg.gridDim = dim3(2u);
    if (cudaOccupancyMaxActiveClusters(&n, gemm2_kernel<EPI>, &cfg) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = sm_count_dev() / 2;
    }
    resident[dev] = n;
  }
  const int clusters = std::min(groups, dev < 64 ? resident[dev] : sm_count_dev() / 2);
  cfg.gridDim = dim3(unsigned(clusters * 2));
  cudaError_t e = cudaLaunchKernelEx(&cfg, gemm2_kernel<EPI>, ma, mb, p);
  if (e != cudaSuccess) return fail(SVD_ERR_CUDA, std::string("gemm2_kernel launch: ") + cudaGetErrorString(e));
  return SVD_OK;
}

#ifndef SVD_GEMM_PAIR
#define SVD_GEMM_PAIR 1
#endif

template <int EPI>
static int launch(const CUtensorMap& ma, const CUtensorMap& mb, const Params& p, cudaStream_t s) {
  if (SVD_GEMM_PAIR && p.tiles_m >= 2) return launch_pair<EPI>(ma, mb, p, s);
  // a one-tile-row problem gains nothing from B multicast
  if (SVD_GEMM_CLUSTER == 4 && p.tiles_m >= 4) return launch_cm<EPI, 4>(ma, mb, p, s);
  if (SVD_GEMM_CLUSTER >= 2 && p.tiles_m >= 2) return launch_cm<EPI, 2>(ma, mb, p, s);
  return launch_cm<EPI, 1>(ma, mb, p, s);
}

}  // namespace gemm
}  // namespace svd

using namespace svd;

extern "C" {

int svd_gemm(const void* a, int64_t lda, const void* b, int64_t ldb, void* out, int64_t ldo, int64_t M,
             int64_t N, int64_t K, int32_t epilogue, const float* resid, int64_t ldr, const void* rope_table,
             int32_t rope_cols, int32_t head_dim, int64_t n_tokens, void* stream) {
  using namespace gemm;
  if (!a || !b || !out) return fail(SVD_ERR_CONFIG, "NULL pointer");
  if (M < 1 || N < 1 || K < 1 || M > (int64_t(1) << 31) || N > (int64_t(1) << 24) || K > (int64_t(1) << 24))
    return fail(SVD_ERR_SHAPE, "gemm: bad M / N / K");
  if (N % 8 != 0 || K % 8 != 0) return fail(SVD_ERR_UNSUPPORTED, "gemm: N and K must be multiples of 8");
  if (lda < K || ldb < N || ldo < N) return fail(SVD_ERR_SHAPE, "gemm: leading dimensions too small");
  const bool f32 = epilogue == kF32 || epilogue == kF32Resid;
  if ((reinterpret_cast<uintptr_t>(out) & 15) != 0 || (ldo * (f32 ? 4 : 2)) % 16 != 0)
    return fail(SVD_ERR_UNSUPPORTED, "gemm: out rows must be 16-byte aligned");
  if (epilogue == kF32Resid &&
      (!resid || (reinterpret_cast<uintptr_t>(resid) & 15) != 0 || ldr % 4 != 0 || ldr < N))
    return fail(SVD_ERR_UNSUPPORTED, "gemm: residual must be a 16-byte aligned fp32 [M, >= N]");
  if (epilogue == kRope && (!rope_table || head_dim < 2 || head_dim % 2 != 0 || n_tokens < 1 ||
                            M % n_tokens != 0 || rope_cols < 0 || rope_cols > N))
    return fail(SVD_ERR_CONFIG, "gemm: RoPE needs a table, an even head_dim and M = B * n_tokens");
  Params p{};
  p.M = int(M);
  p.N = int(N);
  p.K = int(K);
  p.tiles_m = int((M + BM - 1) / BM);
  p.tiles_n = int((N + BN - 1) / BN);
  p.out = out;
  p.ldo = ldo;
  p.resid = resid;
  p.ldr = ldr;
  p.rope = static_cast<const float2*>(rope_table);
  p.rope_cols = rope_cols;
  p.head_dim = head_dim > 0 ? head_dim : 1;
  p.n_tokens = n_tokens > 0 ? int(n_tokens) : 1;
  CUtensorMap ma, mb;
  int st;
  if ((st = tmap_2d(&ma, a, M, K, lda, BM, "a"))) return st;
  if ((st = tmap_2d(&mb, b, K, N, ldb, BK, "b"))) return st;
  auto s = static_cast<cudaStream_t>(stream);
  switch (epilogue) {
    case kBf16: return launch<kBf16>(ma, mb, p, s);
    case kRope: return launch<kRope>(ma, mb, p, s);
    case kGelu: return launch<kGelu>(ma, mb, p, s);
    case kF32Resid: return launch<kF32Resid>(ma, mb, p, s);
    case kF32: return launch<kF32>(ma, mb, p, s);
    default: return fail(SVD_ERR_CONFIG, "gemm: unknown epilogue");
  }
}

}  // extern "C"
