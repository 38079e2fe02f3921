// Microbenchmark: packed half-precision MUFU exp2 for the softmax exp phase.
// Each thread turns a 128-wide fp32 row into packed bf16 P plus rounded row
// sums, like one tile-step of the attention kernel; 1 or 2 warps per SMSP.
//   V0  fp32 ex2 per element (MUFU.EX2 x2 per pair)            — the kernel today
//   V1  x -> f16x2, ex2.approx.f16x2 (one MUFU per pair), f16 -> f32 -> bf16x2
//   V2  x -> bf16x2, ex2.approx.ftz.bf16x2 (one MUFU per pair), result is P
//   V3  fp32 ex2 + F2FP pack, no row sums          (which ops share the MUFU's pipe?)
//   V4  fp32 ex2 + fp32 FADD2 row sums, no pack
//   V5  fp32 ex2 only (results xor-folded)
//   V6  fp32 ex2 + F2FP pack + rounded row sums by unpacking the packed pair
//       (bf16 -> f32 is a 16-bit shift: SHF / LOP + one FADD2) instead of FHADD.BF16
//   V7  as V6, the sums taken after all 16 pairs of the chunk are packed
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../paper_2506_03065_b200/csrc/svd_ptx.cuh"

using namespace svd;

__device__ __forceinline__ uint32_t ex2_f16x2(uint32_t x) {
  uint32_t y;
  asm("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t ex2_bf16x2(uint32_t x) {
  uint32_t y;
  asm("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_f16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ float2 unpack_f16(uint32_t h) {
  float2 r;
  asm("{\n\t.reg .f16 lo, hi;\n\tmov.b32 {lo, hi}, %2;\n\tcvt.f32.f16 %0, lo;\n\tcvt.f32.f16 %1, hi;\n\t}"
      : "=f"(r.x), "=f"(r.y)
      : "r"(h));
  return r;
}

template <int V>
__global__ void __launch_bounds__(256, 1) k_exp(int iters, const float* in, uint32_t* sink, long long* cyc) {
  float s[128];
#pragma unroll
  for (int i = 0; i < 128; ++i) s[i] = in[(threadIdx.x * 7 + i) & 1023] * 0.01f - 3.0f;
  const float2 sl = make_float2(0.1275f, 0.1275f);
  float l = 0.f;
  uint32_t acc_pk = 0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const float2 nm = make_float2(-float(it & 7) * 0.01f, -float(it & 7) * 0.01f);
    float2 acc[4] = {make_float2(0, 0), make_float2(0, 0), make_float2(0, 0), make_float2(0, 0)};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float2 xv = ptx::ffma2(make_float2(s[c * 32 + 2 * i], s[c * 32 + 2 * i + 1]), sl, nm);
        if (V == 6) {
          pk[i] = ptx::pack_bf16(ptx::ex2(xv.x), ptx::ex2(xv.y));
          acc[i & 3] = ptx::fadd2(acc[i & 3], make_float2(__uint_as_float(pk[i] << 16),
                                                          __uint_as_float(pk[i] & 0xFFFF0000u)));
          continue;
        }
        if (V == 7) {
          pk[i] = ptx::pack_bf16(ptx::ex2(xv.x), ptx::ex2(xv.y));
          continue;
        }
        if (V >= 3) {
          const float2 pv = make_float2(ptx::ex2(xv.x), ptx::ex2(xv.y));
          if (V == 3) pk[i] = ptx::pack_bf16(pv.x, pv.y);
          else if (V == 4) { acc[i & 3] = ptx::fadd2(acc[i & 3], pv); pk[i] = 0; }
          else pk[i] = __float_as_uint(pv.x) ^ __float_as_uint(pv.y);
          continue;
        }
        if (V == 0) {
          pk[i] = ptx::pack_bf16(ptx::ex2(xv.x), ptx::ex2(xv.y));
        } else if (V == 1) {
          const float2 p = unpack_f16(ex2_f16x2(pack_f16(xv.x, xv.y)));
          pk[i] = ptx::pack_bf16(p.x, p.y);
        } else {
          pk[i] = ex2_bf16x2(ptx::pack_bf16(xv.x, xv.y));
        }
        ptx::acc_bf16x2(acc[i & 3], pk[i]);
      }
      if (V == 7) {
#pragma unroll
        for (int i = 0; i < 16; ++i)
          acc[i & 3] = ptx::fadd2(acc[i & 3], make_float2(__uint_as_float(pk[i] << 16),
                                                          __uint_as_float(pk[i] & 0xFFFF0000u)));
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) acc_pk ^= pk[i];
    }
    const float2 a = ptx::fadd2(ptx::fadd2(acc[0], acc[1]), ptx::fadd2(acc[2], acc[3]));
    l += a.x + a.y;
    asm volatile("" : "+f"(l), "+r"(acc_pk));
  }
  const long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc_pk ^ __float_as_uint(l);
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int V>
void run(int sms, int threads, const float* in, uint32_t* sink, long long* cyc) {
  const int iters = 2000;
  k_exp<V><<<sms, threads>>>(20, in, sink, cyc);
  k_exp<V><<<sms, threads>>>(iters, in, sink, cyc);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("warps/SMSP %d  V%d: %.0f cycles per 128-wide row-step\n", threads / 128, V, double(h) / iters);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* in;
  uint32_t* sink;
  long long* cyc;
  cudaMalloc(&in, 4096 * 4);
  cudaMemset(in, 0, 4096 * 4);
  cudaMalloc(&sink, sms * 256 * 4);
  cudaMalloc(&cyc, 8);
  for (int threads : {128, 256}) {
    run<0>(sms, threads, in, sink, cyc);
    run<1>(sms, threads, in, sink, cyc);
    run<2>(sms, threads, in, sink, cyc);
    run<3>(sms, threads, in, sink, cyc);
    run<4>(sms, threads, in, sink, cyc);
    run<5>(sms, threads, in, sink, cyc);
    run<6>(sms, threads, in, sink, cyc);
    run<7>(sms, threads, in, sink, cyc);
  }
  return 0;
}
