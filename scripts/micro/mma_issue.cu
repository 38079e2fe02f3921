// Microbenchmark: cycles per tcgen05.mma (kind::f16, cta_group::1) issued
// back to back by one thread, M=128, N in {32,64,128,256}, K=16, SS (A, B in
// smem) and TS (A in TMEM).  One CTA per SM on all SMs; the smem operands are
// garbage (timing only).  Build: nvcc -gencode arch=compute_100a,code=sm_100a
//   -I include -o scripts/micro/mma_issue scripts/micro/mma_issue.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2506_03065_b200/csrc/svd_ptx.cuh"

using namespace svd;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) k_mma(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t mbar;
  const uint32_t base = (ptx::smem_u32(sm) + 1023u) & ~1023u;
  if (threadIdx.x < 32) {
    ptx::tmem_alloc(ptx::smem_u32(&slot), 512);
    ptx::tmem_relinquish();
  }
  if (threadIdx.x == 0) {
    ptx::mbar_init(ptx::smem_u32(&mbar), 1);
    ptx::fence_barrier_init();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t id = ptx::idesc_bf16(128, N, false);
    const uint32_t hi = ptx::sw128_hi(1024);
    const uint32_t alo = ptx::sw128_lo(base, 16), blo = ptx::sw128_lo(base + 65536, 16);
    const uint64_t a = (uint64_t(hi) << 32) | alo, bd = (uint64_t(hi) << 32) | blo;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if (TS) ptx::mma_ts(tmem + 256, tmem + (kk & 3) * 8, bd, id, 1);
        else ptx::mma_ss(tmem + 256, a + (kk & 3) * 2, bd + (kk & 3) * 2, id, 1);
      }
    }
    const long long t1 = clock64();
    ptx::mma_commit(ptx::smem_u32(&mbar));
    ptx::mbar_wait(ptx::smem_u32(&mbar), 0);
    const long long t2 = clock64();
    if (blockIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (threadIdx.x < 32) ptx::tmem_dealloc(tmem, 512);
}

template <int N, bool TS>
void run(int sms) {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  const int smem = 140 * 1024;
  cudaFuncSetAttribute(k_mma<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  k_mma<N, TS><<<sms, 128, smem>>>(10, d);
  k_mma<N, TS><<<sms, 128, smem>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double n = iters * 8.0;
  const double flops = 2.0 * 128 * N * 16;
  printf("%s N=%3d: issue %.1f cyc/mma, complete %.1f cyc/mma (%.0f flop/cyc/SM) %s\n", TS ? "TS" : "SS", N,
         h[0] / n, h[1] / n, flops / (h[1] / n), cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<64, false>(sms);
  run<128, false>(sms);
  run<256, false>(sms);
  run<64, true>(sms);
  run<128, true>(sms);
  run<256, true>(sms);
  run<64, false>(1);
  run<128, false>(1);
  return 0;
}
