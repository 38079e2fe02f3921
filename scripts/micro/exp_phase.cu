// Microbenchmark of the softmax exp phase in isolation: each thread turns a
// 128-wide fp32 row into packed bf16 P (FFMA2 scale-subtract, exp2, F2FP) and
// a row sum, like one tile-step of the attention kernel; 2 or 1 warps per
// SMSP (256 / 128 threads per CTA, one CTA per SM, all SMs).  Variants: the
// fraction of exp2 pairs on the FMA-pipe polynomial, and the polynomial form.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2506_03065_b200/csrc/svd_ptx.cuh"

using namespace svd;

// degree-2 polynomial variant (cheaper, rel. err ~1.7e-3)
__device__ __forceinline__ float2 ex2_poly2_deg2(float2 x) {
  const float2 magic = make_float2(12582912.0f, 12582912.0f);
  const float2 nmagic = make_float2(-12582912.0f, -12582912.0f);
  const float2 mone = make_float2(-1.0f, -1.0f);
  x.x = fmaxf(x.x, -125.0f);
  x.y = fmaxf(x.y, -125.0f);
  const float2 t = ptx::fadd2(x, magic);
  const float2 j = ptx::fadd2(t, nmagic);
  const float2 f = ptx::ffma2(j, mone, x);
  float2 p = ptx::ffma2(make_float2(0.2400f, 0.2400f), f, make_float2(0.6930f, 0.6930f));
  p = ptx::ffma2(p, f, make_float2(1.0f, 1.0f));
  float2 r;
  r.x = __uint_as_float((__float_as_uint(t.x) << 23) + __float_as_uint(p.x));
  r.y = __uint_as_float((__float_as_uint(t.y) << 23) + __float_as_uint(p.y));
  return r;
}

template <int EMU, int DEG>
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
        float2 pv;
        if ((i & 7) >= 8 - EMU) {
          pv = DEG == 3 ? ptx::ex2_poly2(xv) : ex2_poly2_deg2(xv);
        } else {
          pv.x = ptx::ex2(xv.x);
          pv.y = ptx::ex2(xv.y);
        }
        pk[i] = ptx::pack_bf16(pv.x, pv.y);
        ptx::acc_bf16x2(acc[i & 3], pk[i]);
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

template <int EMU, int DEG>
void run(int sms, int threads, const float* in, uint32_t* sink, long long* cyc) {
  const int iters = 2000;
  k_exp<EMU, DEG><<<sms, threads>>>(20, in, sink, cyc);
  k_exp<EMU, DEG><<<sms, threads>>>(iters, in, sink, cyc);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("warps/SMSP %d  emu %d/8 pairs deg %d: %.0f cycles per 128-wide row-step\n", threads / 128, EMU, DEG,
         double(h) / iters);
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
    run<0, 3>(sms, threads, in, sink, cyc);
    run<1, 3>(sms, threads, in, sink, cyc);
    run<2, 3>(sms, threads, in, sink, cyc);
    run<3, 3>(sms, threads, in, sink, cyc);
    run<1, 2>(sms, threads, in, sink, cyc);
    run<2, 2>(sms, threads, in, sink, cyc);
    run<3, 2>(sms, threads, in, sink, cyc);
  }
  return 0;
}
