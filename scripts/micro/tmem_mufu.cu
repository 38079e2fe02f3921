// Microbenchmark: per-SM throughput of TMEM loads (tcgen05.ld 32x32b.x32),
// MUFU.EX2 and their mix, with 2 softmax-like warps per SMSP (warps 4-11 of a
// 384-thread CTA, one CTA per SM, 512 TMEM columns).  Prints cycles per
// iteration per warp for each mode; build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2506_03065_b200/csrc tmem_mufu.cu -o tmem_mufu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "svd_ptx.cuh"

using namespace svd;

// MODE 0: LDTM only, 1: MUFU only, 2: LDTM + MUFU, 3 + e: LDTM + exps (e of every 8 pairs on
// the FMA pipe) + pack + FHADD sums + STTM
template <int MODE>
__global__ void __launch_bounds__(384, 1) bench(int iters, unsigned long long* cyc, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 1) {
    ptx::tmem_alloc(ptx::smem_u32(&slot), 512);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  float acc = 0.f;
  unsigned long long t0 = 0, t1 = 0;
  if (warp >= 4) {
    const int wq = warp & 3, x = (warp - 4) >> 2;
    const uint32_t ts = tmem + (uint32_t(wq * 32) << 16) + uint32_t(x * 128);
    float s[128];
#pragma unroll
    for (int i = 0; i < 128; ++i) s[i] = 0.001f * i;
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (MODE != 1) {
        ptx::tmem_ld32(ts + 0, *reinterpret_cast<float(*)[32]>(&s[0]));
        ptx::tmem_ld32(ts + 32, *reinterpret_cast<float(*)[32]>(&s[32]));
        ptx::tmem_ld32(ts + 64, *reinterpret_cast<float(*)[32]>(&s[64]));
        ptx::tmem_ld32(ts + 96, *reinterpret_cast<float(*)[32]>(&s[96]));
        ptx::tmem_wait_ld();
      }
      if (MODE == 0) {
#pragma unroll
        for (int i = 0; i < 128; i += 8) acc += s[i];
      } else if (MODE == 1 || MODE == 2) {
#pragma unroll
        for (int i = 0; i < 128; ++i) acc += ptx::ex2(s[i] - acc * 1e-30f);
      } else {
        float2 a2[4] = {};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float2 pv;
            if ((i & 7) < MODE - 3) {
              pv = ptx::ex2_poly2_deg2(make_float2(s[c * 32 + 2 * i], s[c * 32 + 2 * i + 1]));
            } else {
              pv.x = ptx::ex2(s[c * 32 + 2 * i]);
              pv.y = ptx::ex2(s[c * 32 + 2 * i + 1]);
            }
            pk[i] = ptx::pack_bf16(pv.x, pv.y);
            ptx::acc_bf16x2(a2[i & 3], pk[i]);
          }
          ptx::tmem_st16(ts + c * 16, pk);
        }
        ptx::tmem_wait_st();
        acc += a2[0].x + a2[1].y + a2[2].x + a2[3].y;
      }
    }
    t1 = clock64();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
  if (warp >= 4 && (threadIdx.x & 31) == 0) cyc[blockIdx.x * 8 + (warp - 4)] = t1 - t0;
  if (acc == 12345.f) sink[0] = acc;
}

template <int MODE>
void run(const char* name, int iters) {
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, 148 * 8 * sizeof(unsigned long long));
  cudaMalloc(&sink, 4);
  bench<MODE><<<148, 384>>>(iters, d, sink);
  bench<MODE><<<148, 384>>>(iters, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148 * 8];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148 * 8; ++i) avg += double(h[i]);
  avg /= 148 * 8;
  const double per = avg / iters;
  // per SMSP: 2 warps; per SM: 8 warps x 32 lanes x 128 values
  printf("%-34s %s  cycles/iter/warp %.0f   TMEM-ld B/clk/SM %.0f   EX2/clk/SM %.1f\n", name,
         e == cudaSuccess ? "ok " : cudaGetErrorString(e), per,
         MODE == 1 ? 0.0 : 8.0 * 32 * 128 * 4 / per, MODE == 0 ? 0.0 : 8.0 * 32 * 128 / per);  // exps (MUFU + FMA) per clk
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  run<0>("LDTM 4 x x32 (+ wait)", 2000);
  run<1>("128 MUFU.EX2", 2000);
  run<2>("LDTM + 128 MUFU.EX2", 2000);
  run<3>("LDTM + EX2 + pack + FHADD + STTM", 2000);
  run<4>("same, 1/8 pairs on FMA", 2000);
  run<5>("same, 2/8 pairs on FMA", 2000);
  run<6>("same, 3/8 pairs on FMA", 2000);
  run<7>("same, 4/8 pairs on FMA", 2000);
  run<9>("same, 6/8 pairs on FMA", 2000);
  return 0;
}
