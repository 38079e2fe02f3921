// sm_100a per-key-block attention mass: the stripe-calibration input of the
// offline search.
//
// Reference semantics: attention.py:108-146 block_key_mass(q, k, grid) —
// mass[b, h, kb] = (1/N) * sum over query rows r of sum over keys j in block
// kb of softmax_r(q_r . k_j / sqrt(d)); each (b, h) row sums to 1.  The
// reference streams an online softmax per query block in fp64; search.py:
// 342-346 takes a stable top-k of the result.
//
// Two passes of QK^T on the tensor cores, no [N, N] map and no atomics:
//   pass 0 (row statistics)  CTA = (two 128-row Q tiles, head, batch).  S = Q_t K_j^T
//       for every 128-key tile j; per row the max m and sum l of 2^(s*c - m)
//       -> stats[bh][tile] = (-m, 1/l) for 128 rows (pad rows: (-inf, 0)).
//   pass 1 (key sums)        CTA = (two 128-key K tiles, head, batch).  S = K_t Q_i^T
//       for every 128-row Q tile i (thread = key = TMEM lane); each key sums
//       2^(s*c - m_r) / l_r over all rows r -> key_acc[bh][key] (fp64).
// then a deterministic per-block fp64 sum (layout.py:139 bounds) / N.
// Both passes are exp-bound (16 MUFU ex2 / clk / SM vs. half an attention
// tile's MMA), i.e. one pass costs about one FULL attention pass; the previous
// formulation (FULL attention with one-hot value columns) cost nb / d passes.
//
// CTA anatomy (384 threads, 1 CTA / SM): warp 0 TMA producer (stationary tile
// once, streaming tiles + pass-1 row statistics through a ring), warp 1 TMEM
// allocator + MMA issuer (S of each stationary tile double-buffered in TMEM,
// 4 x 128 columns), warps 4-7 / 8-11 the S tiles of stationary tile 0 / 1
// (thread = TMEM lane = stationary row): each streaming tile read from L2
// feeds two S tiles.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <string>

#include "svd_plan.h"
#include "svd_ptx.cuh"

namespace svd {

int make_tmap(CUtensorMap* map, const void* ptr, const int64_t* st, int64_t B, int64_t H, int64_t N,
              int D, const char* name);

namespace km {

constexpr int kThreads = 384;
constexpr uint32_t kTmemCols = 512;
// KM_EMU=k: k of every 8 exp pairs on the FMA pipe (cubic, rel. err 7.5e-5;
// masses stay within 1e-9 of fp64).  2: -14% at d=64, -3% at d=128 (where
// the MUFU pipe runs at 86% of peak without it).
#ifndef KM_EMU
#define KM_EMU 2
#endif
__device__ __forceinline__ float2 exp2_pair(float2 x, int i) {
  if (KM_EMU > 0 && (i & 7) < KM_EMU) return ptx::ex2_poly2(x);
  return make_float2(ptx::ex2(x.x), ptx::ex2(x.y));
}

template <int D>
struct Cfg {
  static constexpr int kSlabs = D / 64;
  static constexpr int kBoxBytes = 64 * 64 * 2;   // one TMA box: 64 rows x 128 B
  static constexpr int kSlabBytes = 128 * 128;    // 128 rows x 128 B (one SW128 slab)
  static constexpr int kTileBytes = 128 * D * 2;  // one 128-row tile
  static constexpr int kStages = D == 128 ? 4 : 8;
  static constexpr int kStatBytes = 1024;         // (-m, 1/l) of 128 rows
  static constexpr int kOffA = 0;                 // two stationary tiles
  static constexpr int kOffB = 2 * kTileBytes;
  static constexpr int kOffStat = kOffB + kStages * kTileBytes;
  static constexpr int kOffBar = kOffStat + kStages * kStatBytes;
  // barriers: a | full[S] | empty[S] | s_full[2 tiles][2 bufs] | s_empty[2][2]
  static constexpr int kBarA = 0;
  static constexpr int kBarF = 1;
  static constexpr int kBarE = kBarF + kStages;
  static constexpr int kBarSF = kBarE + kStages;
  static constexpr int kBarSE = kBarSF + 4;
  static constexpr int kNumBars = kBarSE + 4;
  static constexpr int kOffSlot = kOffBar + kNumBars * 8;
  static constexpr int kSmemBytes = kOffSlot + 16 + 1024;  // + alignment slack
};

struct Params {
  int n_tokens;
  int n_tiles;        // ceil(N / 128)
  int heads;
  float scale_log2;   // log2(e) / sqrt(d)
  float* stats;       // [B*H][n_tiles][2][128]: -m (log2 domain), 1/l
  double* key_acc;    // [B*H][n_tiles * 128]
};

__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// MODE 0: row statistics (A = Q tiles, streaming K tiles);
// MODE 1: key sums (A = K tiles, streaming Q tiles + their row statistics).
// A CTA holds two stationary tiles (2*blockIdx.x, +1), one per warpgroup, so
// every streaming tile it pulls through L2 feeds two S tiles.
template <int D, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    key_mass_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                    const Params p) {
  using C = Cfg<D>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* base_ptr = smem_raw + (base - raw);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  auto bar = [&](int i) { return base + C::kOffBar + 8u * uint32_t(i); };
  const int head = blockIdx.y, b = blockIdx.z;
  const int T = p.n_tiles;
  const int64_t bh = int64_t(b) * p.heads + head;

  if (threadIdx.x == 0) {
    ptx::mbar_init(bar(C::kBarA), 1);
    for (int i = 0; i < C::kStages; ++i) {
      ptx::mbar_init(bar(C::kBarF + i), 1);
      // pass 1: the stage also holds row statistics the 8 exp warps read
      ptx::mbar_init(bar(C::kBarE + i), MODE ? 9 : 1);
    }
    for (int i = 0; i < 4; ++i) {
      ptx::mbar_init(bar(C::kBarSF + i), 1);
      ptx::mbar_init(bar(C::kBarSE + i), 4);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc(base + C::kOffSlot, kTmemCols);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(base_ptr + C::kOffSlot);
  const int nseg = (p.n_tokens + 63) / 64;

  if (warp < 4) {
    ptx::reg_dealloc<56>();
    if (warp == 0 && lane == 0) {
      // ------------------------------------------------------------ TMA producer
      ptx::prefetch_tmap(&tm_a);
      ptx::prefetch_tmap(&tm_b);
      const uint64_t pol_a = ptx::policy_evict_first();
      const uint64_t pol_b = ptx::policy_evict_last();
      // a 128-row tile = two 64-row segments; a segment past the sequence end
      // repeats the first (its rows are masked / carry zero weight)
      auto load = [&](const CUtensorMap* tm, uint32_t dst, uint32_t br, int t, uint64_t pol) {
#pragma unroll
        for (int slot = 0; slot < 2; ++slot) {
          const int seg = 2 * t + slot < nseg ? 2 * t + slot : 2 * t;
#pragma unroll
          for (int slab = 0; slab < C::kSlabs; ++slab)
            ptx::tma_load_4d(dst + slab * C::kSlabBytes + slot * C::kBoxBytes, tm, br, slab * 64,
                             seg * 64, head, b, pol);
        }
      };
      ptx::mbar_arrive_expect_tx(bar(C::kBarA), 2 * C::kTileBytes);
#pragma unroll
      for (int x = 0; x < 2; ++x)  // an odd tile count's last CTA repeats tile T-1
        load(&tm_a, base + C::kOffA + x * C::kTileBytes, bar(C::kBarA), min(2 * int(blockIdx.x) + x, T - 1),
             pol_a);
      for (int t = 0; t < T; ++t) {
        const int st = t % C::kStages;
        ptx::mbar_wait(bar(C::kBarE + st), ((t / C::kStages) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(bar(C::kBarF + st), C::kTileBytes + (MODE ? C::kStatBytes : 0));
        load(&tm_b, base + C::kOffB + st * C::kTileBytes, bar(C::kBarF + st), t, pol_b);
        if (MODE)
          ptx::bulk_load(base + C::kOffStat + st * C::kStatBytes, p.stats + (bh * T + t) * 256,
                         C::kStatBytes, bar(C::kBarF + st));
      }
    } else if (warp == 1) {
      // ------------------------------------------------------------ MMA issuer
      if (lane == 0) {
        constexpr uint32_t id_s = ptx::idesc_bf16(128, 128, false);
        constexpr uint32_t hi = ptx::sw128_hi(1024);
        uint32_t sb = base, tb = tmem;
        ptx::mbar_wait(bar(C::kBarA), 0);
        for (int t = 0; t < T; ++t) {
          asm volatile("" : "+r"(sb), "+r"(tb));
          const int st = t % C::kStages, buf = t & 1;
          ptx::mbar_wait(bar(C::kBarF + st), (t / C::kStages) & 1);
          const uint32_t blo = ptx::sw128_lo(sb + C::kOffB + st * C::kTileBytes, 16);
#pragma unroll
          for (int x = 0; x < 2; ++x) {
            ptx::mbar_wait(bar(C::kBarSE + 2 * x + buf), ((t >> 1) & 1) ^ 1);
            ptx::tc_fence_after();
            const uint32_t alo = ptx::sw128_lo(sb + C::kOffA + x * C::kTileBytes, 16);
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint32_t off = ((kk >> 2) * C::kSlabBytes + (kk & 3) * 32) >> 4;
              ptx::mma_ss(tb + uint32_t(x * 256 + buf * 128), (uint64_t(hi) << 32) | (alo + off),
                          (uint64_t(hi) << 32) | (blo + off), id_s, kk > 0 ? 1u : 0u);
            }
            ptx::mma_commit(bar(C::kBarSF + 2 * x + buf));
          }
          ptx::mma_commit(bar(C::kBarE + st));
        }
      }
      __syncwarp();
      named_bar_sync(1, 32 + 256);
      ptx::tc_fence_after();
      ptx::tmem_dealloc(tmem, kTmemCols);
    }
    return;
  }

  // ---------------------------------------------------------------- exp warps
  ptx::reg_alloc<224>();
  const int x = (warp - 4) >> 2;   // stationary tile of this warpgroup
  const int wq = warp & 3;         // TMEM lane quarter
  const int row = wq * 32 + lane;  // TMEM lane = A row (query row / key)
  const int tile = 2 * int(blockIdx.x) + x;
  const uint32_t ts0 = tmem + (uint32_t(wq * 32) << 16) + uint32_t(x * 256);
  const float sl2 = p.scale_log2;
  const float2 sl2x2 = make_float2(sl2, sl2);

  // S of streaming tile t into registers; the TMEM buffer is released at once
  auto load_s = [&](int t, float (&s)[128]) {
    const int buf = t & 1;
    ptx::mbar_wait(bar(C::kBarSF + 2 * x + buf), (t >> 1) & 1);
    ptx::tc_fence_after();
#pragma unroll
    for (int c = 0; c < 4; ++c)
      ptx::tmem_ld32(ts0 + buf * 128u + 32u * c, *reinterpret_cast<float(*)[32]>(&s[32 * c]));
    ptx::tmem_wait_ld();
    ptx::tc_fence_before();
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(bar(C::kBarSE + 2 * x + buf));
  };

  if constexpr (MODE == 0) {
    float m = -INFINITY, l = 0.f;  // log2-domain running max, sum of 2^(s*c - m)
    for (int t = 0; t < T; ++t) {
      float s[128];
      load_s(t, s);
      const int k0 = t * 128;
      if (k0 + 128 > p.n_tokens) {
#pragma unroll
        for (int i = 0; i < 128; ++i)
          if (k0 + i >= p.n_tokens) s[i] = -INFINITY;
      }
      float mp[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mp[i] = fmaxf(s[i], s[8 + i]);
#pragma unroll
      for (int i = 16; i < 128; i += 16)
#pragma unroll
        for (int j = 0; j < 8; ++j) mp[j] = fmaxf(mp[j], fmaxf(s[i + j], s[i + 8 + j]));
      const float mx = fmaxf(fmaxf(fmaxf(mp[0], mp[1]), fmaxf(mp[2], mp[3])),
                             fmaxf(fmaxf(mp[4], mp[5]), fmaxf(mp[6], mp[7])));
      const float m_new = fmaxf(m, mx * sl2);
      if (m_new > m) {
        l *= ptx::ex2(m - m_new);
        m = m_new;
      }
      const float2 nm = make_float2(-m, -m);  // m is finite: every tile holds a valid key
      float2 a[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                     make_float2(0.f, 0.f)};
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        const float2 xv = ptx::ffma2(make_float2(s[2 * i], s[2 * i + 1]), sl2x2, nm);
        a[i & 3] = ptx::fadd2(a[i & 3], exp2_pair(xv, i));
      }
      const float2 a2 = ptx::fadd2(ptx::fadd2(a[0], a[1]), ptx::fadd2(a[2], a[3]));
      l += a2.x + a2.y;
    }
    if (tile < T) {
      const bool valid = tile * 128 + row < p.n_tokens && l > 0.f;
      float* sp = p.stats + (bh * T + tile) * 256;
      sp[row] = valid ? -m : -INFINITY;
      sp[128 + row] = valid ? 1.0f / l : 0.f;
    }
  } else {
    double tot = 0.0;  // this key's mass over the rows seen so far
    for (int t = 0; t < T; ++t) {
      float s[128];
      load_s(t, s);
      const int st = t % C::kStages;
      // the stage's statistics landed with its tiles (already complete: the
      // MMA that produced S waited on the same barrier phase)
      ptx::mbar_wait(bar(C::kBarF + st), (t / C::kStages) & 1);
      const float4* sn = reinterpret_cast<const float4*>(base_ptr + C::kOffStat + st * C::kStatBytes);
      const float4* si = sn + 32;  // 1/l of the same rows
      float2 a[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                     make_float2(0.f, 0.f)};
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float4 nm = sn[i], il = si[i];
        const float2 x0 = ptx::ffma2(make_float2(s[4 * i], s[4 * i + 1]), sl2x2, make_float2(nm.x, nm.y));
        const float2 x1 =
            ptx::ffma2(make_float2(s[4 * i + 2], s[4 * i + 3]), sl2x2, make_float2(nm.z, nm.w));
        a[(2 * i) & 3] = ptx::ffma2(exp2_pair(x0, 2 * i), make_float2(il.x, il.y), a[(2 * i) & 3]);
        a[(2 * i + 1) & 3] = ptx::ffma2(exp2_pair(x1, 2 * i + 1), make_float2(il.z, il.w), a[(2 * i + 1) & 3]);
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(bar(C::kBarE + st));
      const float2 a2 = ptx::fadd2(ptx::fadd2(a[0], a[1]), ptx::fadd2(a[2], a[3]));
      tot += double(a2.x) + double(a2.y);
    }
    if (tile < T) p.key_acc[bh * int64_t(T) * 128 + tile * 128 + row] = tot;
  }
  ptx::tc_fence_before();
  named_bar_sync(1, 32 + 256);
}

// mass[bh][kb] = (sum of key_acc over block kb's keys) / N, sequential fp64
__global__ void block_sum_kernel(const double* __restrict__ key_acc, int64_t acc_stride, int n_tokens,
                                 int block_size, int n_blocks, int64_t n_bh, double* __restrict__ mass) {
  const int64_t gid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gid >= n_bh * n_blocks) return;
  const int64_t bh = gid / n_blocks;
  const int kb = int(gid % n_blocks);
  const int lo = min(int64_t(kb) * block_size, int64_t(n_tokens));
  const int hi = min(int64_t(kb + 1) * block_size, int64_t(n_tokens));
  const double* src = key_acc + bh * acc_stride;
  double s = 0.0;
  for (int j = lo; j < hi; ++j) s += src[j];
  mass[gid] = s / double(n_tokens);
}

static int cuda_fail(cudaError_t e, const char* what) {
  return fail(SVD_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// row_pass: run pass 0 (row statistics); false = stats already hold them
// (svd_fwd_args.row_stats of a forward launch), only the key-sum pass runs
template <int D>
static int launch(const void* q, const void* k, const int64_t* qs, const int64_t* ks, int batch,
                  int heads, int64_t n, int head_dim, int block_size, float* stats, double* key_acc,
                  double* mass, cudaStream_t stream, bool row_pass = true) {
  using C = Cfg<D>;
  CUtensorMap mq, mk;
  int st;
  if ((st = make_tmap(&mq, q, qs, batch, heads, n, D, "q"))) return st;
  if ((st = make_tmap(&mk, k, ks, batch, heads, n, D, "k"))) return st;
  static bool attr_set[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(key_mass_kernel<D, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::kSmemBytes);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(key_mass_kernel<D, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               C::kSmemBytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
    attr_set[dev] = true;
  }
  Params p{};
  p.n_tokens = int(n);
  p.n_tiles = int((n + 127) / 128);
  p.heads = heads;
  p.scale_log2 = float(1.4426950408889634 / std::sqrt(double(head_dim)));
  p.stats = stats;
  p.key_acc = key_acc;
  const dim3 grid(unsigned((p.n_tiles + 1) / 2), unsigned(heads), unsigned(batch));
  if (row_pass) key_mass_kernel<D, 0><<<grid, kThreads, C::kSmemBytes, stream>>>(mq, mk, p);
  key_mass_kernel<D, 1><<<grid, kThreads, C::kSmemBytes, stream>>>(mk, mq, p);
  const int64_t n_bh = int64_t(batch) * heads;
  const int nb = int((n + block_size - 1) / block_size);
  const int64_t total = n_bh * nb;
  block_sum_kernel<<<unsigned((total + 255) / 256), 256, 0, stream>>>(
      key_acc, int64_t(p.n_tiles) * 128, int(n), block_size, nb, n_bh, mass);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "key_mass_kernel launch");
  return SVD_OK;
}

}  // namespace km
}  // namespace svd

using namespace svd;

extern "C" {

int64_t svd_key_mass_workspace(int32_t batch, int32_t heads, int64_t n_tokens) {
  if (batch < 1 || heads < 1 || n_tokens < 1) return 0;
  const int64_t tiles = (n_tokens + 127) / 128;
  return int64_t(batch) * heads * tiles * (256 * 4 + 128 * 8);
}

int svd_block_key_mass(const void* q, const void* k, const int64_t* q_strides, const int64_t* k_strides,
                       int32_t batch, int32_t heads, int64_t n_tokens, int32_t head_dim,
                       int32_t tensor_dim, int32_t block_size, int32_t dtype, void* workspace,
                       int64_t workspace_bytes, double* mass, void* stream) {
  if (!q || !k || !mass || !workspace) return fail(SVD_ERR_CONFIG, "NULL pointer");
  if (dtype != 0) return fail(SVD_ERR_UNSUPPORTED, "only bf16 (dtype 0) is supported");
  if (batch < 1 || heads < 1 || n_tokens < 1) return fail(SVD_ERR_SHAPE, "bad shape");
  if (n_tokens > (int64_t(1) << 30)) return fail(SVD_ERR_UNSUPPORTED, "n_tokens too large");
  if (block_size < 1) return fail(SVD_ERR_CONFIG, "block_size must be >= 1");
  if (head_dim < 1 || head_dim > tensor_dim)
    return fail(SVD_ERR_SHAPE, "head_dim must be in [1, tensor_dim]");
  const int64_t need = svd_key_mass_workspace(batch, heads, n_tokens);
  if (workspace_bytes < need)
    return fail(SVD_ERR_CONFIG, "workspace too small: need " + std::to_string(need) + " bytes");
  if ((reinterpret_cast<uintptr_t>(workspace) & 15) != 0)
    return fail(SVD_ERR_UNSUPPORTED, "workspace must be 16-byte aligned");
  const int64_t tiles = (n_tokens + 127) / 128;
  float* stats = static_cast<float*>(workspace);
  double* key_acc = reinterpret_cast<double*>(stats + int64_t(batch) * heads * tiles * 256);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  switch (tensor_dim) {
    case 64:
      return km::launch<64>(q, k, q_strides, k_strides, batch, heads, n_tokens, head_dim, block_size,
                            stats, key_acc, mass, s);
    case 128:
      return km::launch<128>(q, k, q_strides, k_strides, batch, heads, n_tokens, head_dim, block_size,
                             stats, key_acc, mass, s);
    default:
      return fail(SVD_ERR_UNSUPPORTED,
                  "tensor_dim " + std::to_string(tensor_dim) + " unsupported (64 or 128; pad)");
  }
}

int svd_block_key_mass_from_stats(const void* q, const void* k, const int64_t* q_strides,
                                  const int64_t* k_strides, int32_t batch, int32_t heads,
                                  int64_t n_tokens, int32_t head_dim, int32_t tensor_dim,
                                  int32_t block_size, int32_t dtype, const float* row_stats,
                                  void* workspace, int64_t workspace_bytes, double* mass,
                                  void* stream) {
  if (!q || !k || !mass || !workspace || !row_stats) return fail(SVD_ERR_CONFIG, "NULL pointer");
  if (dtype != 0) return fail(SVD_ERR_UNSUPPORTED, "only bf16 (dtype 0) is supported");
  if (batch < 1 || heads < 1 || n_tokens < 1) return fail(SVD_ERR_SHAPE, "bad shape");
  if (n_tokens > (int64_t(1) << 30)) return fail(SVD_ERR_UNSUPPORTED, "n_tokens too large");
  if (block_size < 1) return fail(SVD_ERR_CONFIG, "block_size must be >= 1");
  if (head_dim < 1 || head_dim > tensor_dim)
    return fail(SVD_ERR_SHAPE, "head_dim must be in [1, tensor_dim]");
  const int64_t need = svd_key_mass_workspace(batch, heads, n_tokens);
  if (workspace_bytes < need)
    return fail(SVD_ERR_CONFIG, "workspace too small: need " + std::to_string(need) + " bytes");
  if ((reinterpret_cast<uintptr_t>(workspace) & 15) != 0 || (reinterpret_cast<uintptr_t>(row_stats) & 15) != 0)
    return fail(SVD_ERR_UNSUPPORTED, "workspace and row_stats must be 16-byte aligned");
  const int64_t tiles = (n_tokens + 127) / 128;
  float* stats = const_cast<float*>(row_stats);  // read only by the key-sum pass
  double* key_acc = reinterpret_cast<double*>(static_cast<float*>(workspace) + int64_t(batch) * heads * tiles * 256);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  switch (tensor_dim) {
    case 64:
      return km::launch<64>(q, k, q_strides, k_strides, batch, heads, n_tokens, head_dim, block_size,
                            stats, key_acc, mass, s, false);
    case 128:
      return km::launch<128>(q, k, q_strides, k_strides, batch, heads, n_tokens, head_dim, block_size,
                             stats, key_acc, mass, s, false);
    default:
      return fail(SVD_ERR_UNSUPPORTED,
                  "tensor_dim " + std::to_string(tensor_dim) + " unsupported (64 or 128; pad)");
  }
}

}  // extern "C"
