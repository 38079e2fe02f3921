// Microbenchmark: MUFU.EX2 and FFMA2 throughput per SM on this GPU.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void ex2_kernel(float* out, int iters, long long* cycles) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

__global__ void ex2h2_kernel(float* out, int iters, long long* cycles) {
  unsigned a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 0xB800B800u + threadIdx.x + i;  // -0.5 f16 pairs
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i]));
  }
  __syncthreads();
  long long t1 = clock64();
  unsigned s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = float(s);
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

__global__ void ex2bh2_kernel(float* out, int iters, long long* cycles) {
  unsigned a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 0xBF00BF00u + threadIdx.x + i;  // -0.5 bf16 pairs
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i]));
  }
  __syncthreads();
  long long t1 = clock64();
  unsigned s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = float(s);
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

__global__ void ffma2_kernel(float* out, int iters, long long* cycles) {
  float2 a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = make_float2(0.001f * threadIdx.x, 0.002f * i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("{.reg .b64 r; mov.b64 r, {%0,%1}; fma.rn.f32x2 r, r, r, r; mov.b64 {%0,%1}, r;}"
                   : "+f"(a[i].x), "+f"(a[i].y));
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096;
  for (int warps : {1, 2, 4, 8, 16}) {
    for (int k = 0; k < 4; ++k) {
      long long h[148];
      if (k == 0) ex2_kernel<<<148, warps * 32>>>(out, iters, cyc);
      else if (k == 1) ffma2_kernel<<<148, warps * 32>>>(out, iters, cyc);
      else if (k == 2) ex2h2_kernel<<<148, warps * 32>>>(out, iters, cyc);
      else ex2bh2_kernel<<<148, warps * 32>>>(out, iters, cyc);
      cudaDeviceSynchronize();
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      double ops = double(warps) * 32 * iters * 8 * (k ? 2 : 1);
      const char* nm[4] = {"MUFU.EX2 f32", "FFMA2", "EX2 f16x2", "EX2 bf16x2"};
      printf("%s warps/SM=%2d: %.2f results/clk/SM (%.1f cycles per warp-instr per SMSP)\n",
             nm[k], warps, ops / h[0],
             double(h[0]) / (double(iters) * 8 * (warps >= 4 ? warps / 4.0 : 1.0)));
    }
  }
  return 0;
}
