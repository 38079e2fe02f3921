// The steps either side of the attention operator in a vDiT block (SURVEY
// §8 row f4): the row-wise / element-wise work of the reference's
// layer_qkv (model.py:372-391) and layer_finish (model.py:394-402).  The
// projections themselves are plain GEMMs (cuBLAS through torch); what is
// here is everything between them, written so that no extra pass over the
// activations is needed:
//
//   layer_qkv:    x (fp32) --LN--> h (bf16) --GEMM--> [N, 3D] --RoPE(q,k) in place-->
//                 q/k/v read by the attention kernel through strides (no split-heads copy)
//   layer_finish: O stored [B, N, H, d] (= merged heads, no copy) --GEMM(fp32 out)-->
//                 a = x + proj, h2 = LN(a) (one fused pass) --GEMM--> GELU in place
//                 --GEMM(fp32 out)--> + a
//
// All kernels are HBM-bound streaming passes: 16-byte vector accesses, a
// warp per row for the row reductions, grids sized in multiples of the SM
// count.  Stats and transcendental math in fp32 (LayerNorm's reference is
// fp64; its outputs feed bf16 GEMMs).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "svd_plan.h"
#include "svdit_b200.h"

namespace svd {
namespace {

constexpr int kRowWarps = 8;  // rows per CTA in the row kernels (one warp per row)

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// LayerNorm without affine (model.py:352-355): y = (x - mean) / sqrt(var + eps),
// var the biased variance.  Optional fused residual: x := x + r, written back
// to `a` (fp32) before the statistics.  Two passes over the row in fp32 (the
// row is L1-resident after the first), bf16 output.
template <bool RESID>
__global__ void __launch_bounds__(kRowWarps * 32) layernorm_kernel(
    const float* __restrict__ x, const float* __restrict__ r, float* __restrict__ a,
    __nv_bfloat16* __restrict__ y, int64_t rows, int dim, float eps) {
  const int lane = threadIdx.x & 31;
  const int64_t row0 = int64_t(blockIdx.x) * kRowWarps + (threadIdx.x >> 5);
  const int64_t stride = int64_t(gridDim.x) * kRowWarps;
  const int nv = dim / 4;  // float4 chunks (dim % 4 == 0 checked on the host)
  for (int64_t row = row0; row < rows; row += stride) {
    const float4* xr = reinterpret_cast<const float4*>(x + row * dim);
    const float4* rr = RESID ? reinterpret_cast<const float4*>(r + row * dim) : nullptr;
    float4* ar = RESID ? reinterpret_cast<float4*>(a + row * dim) : nullptr;
    float s = 0.f;
    for (int i = lane; i < nv; i += 32) {
      float4 v = xr[i];
      if constexpr (RESID) {
        const float4 w = rr[i];
        v.x += w.x;
        v.y += w.y;
        v.z += w.z;
        v.w += w.w;
        ar[i] = v;
      }
      s += (v.x + v.y) + (v.z + v.w);
    }
    const float mean = warp_sum(s) / float(dim);
    const float4* src = RESID ? reinterpret_cast<const float4*>(ar) : xr;
    if constexpr (RESID) __syncwarp();
    float q = 0.f;
    for (int i = lane; i < nv; i += 32) {
      const float4 v = src[i];
      const float d0 = v.x - mean, d1 = v.y - mean, d2 = v.z - mean, d3 = v.w - mean;
      q += (d0 * d0 + d1 * d1) + (d2 * d2 + d3 * d3);
    }
    const float rstd = rsqrtf(warp_sum(q) / float(dim) + eps);
    uint2* yr = reinterpret_cast<uint2*>(y + row * dim);
    for (int i = lane; i < nv; i += 32) {
      const float4 v = src[i];
      const __nv_bfloat162 lo = __floats2bfloat162_rn((v.x - mean) * rstd, (v.y - mean) * rstd);
      const __nv_bfloat162 hi = __floats2bfloat162_rn((v.z - mean) * rstd, (v.w - mean) * rstd);
      uint2 o;
      o.x = *reinterpret_cast<const uint32_t*>(&lo);
      o.y = *reinterpret_cast<const uint32_t*>(&hi);
      yr[i] = o;
    }
  }
}

// RoPE table (model.py:169-195): cos / sin of position * base^(-2c/d) for
// c < d/2, angles and trig in fp64 (positions reach 1e5 rad), stored fp32.
__global__ void rope_table_kernel(float2* __restrict__ table, int64_t n, int half, double base,
                                  int d) {
  const int64_t total = n * half;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t pos = i / half;
    const int c = int(i % half);
    const double theta = pow(base, -2.0 * double(c) / double(d));
    double sn, cs;
    sincos(double(pos) * theta, &sn, &cs);
    table[i] = make_float2(float(cs), float(sn));
  }
}

// RoPE in place on the q and k column blocks of the fused projection output
// [rows = B*N, ld] (q at column 0, k at column `k_off`), head h occupying
// columns [h*d, (h+1)*d) of each block.  Pair (2c, 2c+1) rotates by the
// table's angle for the row's token.  One thread per 4 pairs (16 bytes).
__global__ void rope_apply_kernel(__nv_bfloat16* __restrict__ qkv, int64_t rows, int64_t ld,
                                  int64_t k_off, int64_t n_tokens, int heads, int d,
                                  const float2* __restrict__ table) {
  const int half = d / 2;
  const int vec_per_head = half / 4;              // 4 pairs = 8 bf16 = 16 B
  const int64_t vec_per_row = int64_t(heads) * vec_per_head;
  const int64_t total = rows * vec_per_row * 2;   // q and k
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int which = int(i % 2);                 // 0 = q, 1 = k
    const int64_t j = i / 2;
    const int64_t row = j / vec_per_row;
    const int64_t rem = j % vec_per_row;
    const int h = int(rem / vec_per_head);
    const int c0 = int(rem % vec_per_head) * 4;   // first pair index
    const int64_t tok = row % n_tokens;
    uint4* p = reinterpret_cast<uint4*>(qkv + row * ld + (which ? k_off : 0) + int64_t(h) * d + 2 * c0);
    uint4 v = *p;
    const float4* tb = reinterpret_cast<const float4*>(table + tok * half + c0);
    const float4 t01 = tb[0], t23 = tb[1];        // (cos, sin) for pairs c0..c0+3
    const float cs[4] = {t01.x, t01.z, t23.x, t23.z};
    const float sn[4] = {t01.y, t01.w, t23.y, t23.w};
    uint32_t* w = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
      const __nv_bfloat162 o =
          __floats2bfloat162_rn(f.x * cs[e] - f.y * sn[e], f.x * sn[e] + f.y * cs[e]);
      w[e] = *reinterpret_cast<const uint32_t*>(&o);
    }
    *p = v;
  }
}

// Exact GELU (model.py:357-359: 0.5 x (1 + erf(x / sqrt 2))) in place on bf16.
__global__ void gelu_kernel(__nv_bfloat16* __restrict__ u, int64_t n8) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n8;
       i += int64_t(gridDim.x) * blockDim.x) {
    uint4 v = reinterpret_cast<uint4*>(u)[i];
    uint32_t* w = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
      const float g0 = 0.5f * f.x * (1.f + erff(f.x * 0.70710678118654752f));
      const float g1 = 0.5f * f.y * (1.f + erff(f.y * 0.70710678118654752f));
      const __nv_bfloat162 o = __floats2bfloat162_rn(g0, g1);
      w[e] = *reinterpret_cast<const uint32_t*>(&o);
    }
    reinterpret_cast<uint4*>(u)[i] = v;
  }
}

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

unsigned stream_grid(int64_t work, int threads, int per_sm = 8) {
  const int64_t want = (work + threads - 1) / threads;
  const int64_t cap = int64_t(sm_count()) * per_sm;
  return unsigned(want < cap ? (want > 0 ? want : 1) : cap);
}

int launched(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(SVD_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return SVD_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace
}  // namespace svd

using namespace svd;

extern "C" {

int svd_layernorm(const float* x, const float* resid, float* x_out, void* y, int64_t rows,
                  int32_t dim, float eps, void* stream) {
  if (!x || !y || (resid && !x_out)) return fail(SVD_ERR_CONFIG, "NULL pointer");
  if (rows < 0 || dim < 4 || dim % 4 != 0)
    return fail(SVD_ERR_UNSUPPORTED, "layernorm: dim must be a positive multiple of 4");
  if (!aligned16(x) || !aligned16(y) || (resid && (!aligned16(resid) || !aligned16(x_out))))
    return fail(SVD_ERR_UNSUPPORTED, "layernorm: pointers must be 16-byte aligned");
  if (rows == 0) return SVD_OK;
  const unsigned grid = stream_grid(rows, kRowWarps, 16);
  auto s = static_cast<cudaStream_t>(stream);
  if (resid)
    layernorm_kernel<true><<<grid, kRowWarps * 32, 0, s>>>(
        x, resid, x_out, static_cast<__nv_bfloat16*>(y), rows, dim, eps);
  else
    layernorm_kernel<false><<<grid, kRowWarps * 32, 0, s>>>(
        x, nullptr, nullptr, static_cast<__nv_bfloat16*>(y), rows, dim, eps);
  return launched("layernorm_kernel");
}

int svd_rope_table(void* table, int64_t n_tokens, int32_t head_dim, double base, void* stream) {
  if (!table) return fail(SVD_ERR_CONFIG, "NULL pointer");
  if (n_tokens < 1 || head_dim < 2 || head_dim % 2 != 0)
    return fail(SVD_ERR_SHAPE, "rope table: even head_dim and n_tokens >= 1 required");
  const int half = head_dim / 2;
  rope_table_kernel<<<stream_grid(n_tokens * half, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<float2*>(table), n_tokens, half, base, head_dim);
  return launched("rope_table_kernel");
}

int svd_rope_apply(void* qkv, int64_t rows, int64_t ld, int64_t k_off, int64_t n_tokens,
                   int32_t heads, int32_t head_dim, const void* table, void* stream) {
  if (!qkv || !table) return fail(SVD_ERR_CONFIG, "NULL pointer");
  if (head_dim % 8 != 0)
    return fail(SVD_ERR_UNSUPPORTED, "rope: head_dim must be a multiple of 8");
  if (ld % 8 != 0 || k_off % 8 != 0 || !aligned16(qkv) || !aligned16(table))
    return fail(SVD_ERR_UNSUPPORTED, "rope: 16-byte aligned rows required");
  if (n_tokens < 1 || rows % n_tokens != 0) return fail(SVD_ERR_SHAPE, "rope: rows must be B * N");
  const int64_t total = rows * heads * (head_dim / 8) * 2;
  if (total == 0) return SVD_OK;
  rope_apply_kernel<<<stream_grid(total, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<__nv_bfloat16*>(qkv), rows, ld, k_off, n_tokens, heads, head_dim,
      static_cast<const float2*>(table));
  return launched("rope_apply_kernel");
}

int svd_gelu(void* u, int64_t count, void* stream) {
  if (!u) return fail(SVD_ERR_CONFIG, "NULL pointer");
  if (count % 8 != 0 || !aligned16(u))
    return fail(SVD_ERR_UNSUPPORTED, "gelu: count % 8 == 0 and 16-byte alignment required");
  if (count == 0) return SVD_OK;
  gelu_kernel<<<stream_grid(count / 8, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<__nv_bfloat16*>(u), count / 8);
  return launched("gelu_kernel");
}

}  // extern "C"
