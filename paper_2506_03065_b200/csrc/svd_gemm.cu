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
//   warps 4-7   epilogue: thread = output row = TMEM lane, tcgen05.ld of 32
//               columns at a time, the fused op, 16-byte global stores
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

constexpr int BM = 128, BN = 256, BK = 64, kStages = 4, kThreads = 256;
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

__device__ __forceinline__ float gelu_exact(float x) {
  return 0.5f * x * (1.f + erff(x * 0.70710678118654752f));
}

template <int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                const Params p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* base_ptr = smem_raw + (base - raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto bar = [&](int i) { return base + kOffBar + 8u * uint32_t(i); };
  const int n_tiles = p.tiles_m * p.tiles_n;
  const int k_steps = (p.K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      ptx::mbar_init(bar(kBarFull + i), 1);
      ptx::mbar_init(bar(kBarEmpty + i), 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(bar(kBarAccFull + i), 1);
      ptx::mbar_init(bar(kBarAccEmpty + i), 128);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc(base + kOffSlot, kTmemCols);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(base_ptr + kOffSlot);

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      ptx::prefetch_tmap(&tm_a);
      ptx::prefetch_tmap(&tm_b);
      const uint64_t pol_a = ptx::policy_evict_first();
      const uint64_t pol_b = ptx::policy_evict_last();
      int step = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int m0 = (t / p.tiles_n) * BM, n0 = (t % p.tiles_n) * BN;
        for (int ks = 0; ks < k_steps; ++ks, ++step) {
          const int s = step % kStages;
          ptx::mbar_wait(bar(kBarEmpty + s), ((step / kStages) & 1) ^ 1);
          const uint32_t dst = base + s * kStageBytes;
          ptx::mbar_arrive_expect_tx(bar(kBarFull + s), kStageBytes);
          ptx::tma_load_2d(dst, &tm_a, bar(kBarFull + s), ks * BK, m0, pol_a);
#pragma unroll
          for (int i = 0; i < BN / 64; ++i)
            ptx::tma_load_2d(dst + kABytes + i * kBBoxBytes, &tm_b, bar(kBarFull + s), n0 + 64 * i, ks * BK,
                             pol_b);
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
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
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
          ptx::mma_commit(bar(kBarEmpty + s));
        }
        ptx::mma_commit(bar(kBarAccFull + buf));
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int row_in_tile = (warp - 4) * 32 + lane;
    const uint32_t lane_off = uint32_t((warp - 4) * 32) << 16;
    int it = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
      const int buf = it & 1;
      const int m0 = (t / p.tiles_n) * BM, n0 = (t % p.tiles_n) * BN;
      const int row = m0 + row_in_tile;
      ptx::mbar_wait(bar(kBarAccFull + buf), (it >> 1) & 1);
      ptx::tc_fence_after();
      const uint32_t acc = tmem + lane_off + uint32_t(buf * BN);
      const bool row_ok = row < p.M;
      const int tok = row_ok ? row % p.n_tokens : 0;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
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
            const float4* r = reinterpret_cast<const float4*>(p.resid + int64_t(row) * p.ldr + col0);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              if (4 * i >= ncols) break;
              const float4 w = __ldg(r + i);
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
      ptx::tc_fence_before();
      ptx::mbar_arrive(bar(kBarAccEmpty + buf));
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, kTmemCols);
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

template <int EPI>
static int launch(const CUtensorMap& ma, const CUtensorMap& mb, const Params& p, cudaStream_t s) {
  static bool attr[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr[dev]) {
    cudaError_t e = cudaFuncSetAttribute(gemm_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e != cudaSuccess) return fail(SVD_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    attr[dev] = true;
  }
  const int tiles = p.tiles_m * p.tiles_n;
  const int grid = std::min(tiles, sm_count_dev());
  gemm_kernel<EPI><<<grid, kThreads, kSmemBytes, s>>>(ma, mb, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(SVD_ERR_CUDA, std::string("gemm_kernel launch: ") + cudaGetErrorString(e));
  return SVD_OK;
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
