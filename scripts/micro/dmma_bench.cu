// Microbenchmark: FP64 tensor-core (mma.sync m8n8k4 f64, "DMMA") vs FP64 FMA throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double c[8][2];
#pragma unroll
  for (int q = 0; q < 8; ++q) c[q][0] = c[q][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) dmma(c[q][0], c[q][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void k_fma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double c[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) c[q] = q;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 16; ++q) c[q] = fma(c[q], b, a);
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 16; ++q) s += c[q];
  if (s == 12345.0) out[0] = s;
}

// half the warps on DMMA, half on DFMA: do the two FP64 pipes overlap?
__global__ void k_mixed(double* out, int iters, int dfma_per_dmma) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double c[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) c[q] = q;
  if ((threadIdx.x >> 5) & 1) {
    for (int it = 0; it < iters * dfma_per_dmma; ++it) {
#pragma unroll
      for (int q = 0; q < 16; ++q) c[q] = fma(c[q], b, a);
    }
  } else {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int q = 0; q < 8; ++q) dmma(c[2 * q], c[2 * q + 1], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 16; ++q) s += c[q];
  if (s == 12345.0) out[0] = s;
}

// DMMA and DFMA interleaved in the same warp
__global__ void k_interleaved(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double c[8][2], f[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) c[q][0] = c[q][1] = f[q] = q;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      dmma(c[q][0], c[q][1], a, b);
      f[q] = fma(f[q], b, a);
      f[q] = fma(f[q], b, a);
    }
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1] + f[q];
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int warps = 4; warps <= 16; warps *= 2) {
    const int iters = 20000;
    k_dmma<<<sms * 2, 32 * warps>>>(out, 100);
    cudaEventRecord(a);
    k_dmma<<<sms * 2, 32 * warps>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double flops = 2.0 * 256 * 8 * (double)iters * sms * 2 * warps;
    printf("DMMA  warps/blk %2d: %.2f TFLOP/s\n", warps, flops / ms / 1e9);
    k_fma<<<sms * 2, 32 * warps>>>(out, 100);
    cudaEventRecord(a);
    k_fma<<<sms * 2, 32 * warps>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    flops = 2.0 * 16 * (double)iters * sms * 2 * warps * 32;
    printf("DFMA  warps/blk %2d: %.2f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  for (int ratio = 1; ratio <= 4; ratio *= 2) {
    const int iters = 20000, warps = 16;
    k_mixed<<<sms * 2, 32 * warps>>>(out, 100, ratio);
    cudaEventRecord(a);
    k_mixed<<<sms * 2, 32 * warps>>>(out, iters, ratio);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double fd = 2.0 * 256 * 8 * (double)iters * sms * 2 * (warps / 2);
    const double ff = 2.0 * 16 * (double)iters * ratio * sms * 2 * (warps / 2) * 32;
    printf("mixed (DFMA:DMMA iters %d): DMMA %.2f + DFMA %.2f = %.2f TFLOP/s\n", ratio, fd / ms / 1e9,
           ff / ms / 1e9, (fd + ff) / ms / 1e9);
  }
  {
    const int iters = 20000, warps = 8;
    k_interleaved<<<sms * 2, 32 * warps>>>(out, 100);
    cudaEventRecord(a);
    k_interleaved<<<sms * 2, 32 * warps>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double fd = 2.0 * 256 * 8 * (double)iters * sms * 2 * warps;
    const double ff = 2.0 * 16 * (double)iters * sms * 2 * warps * 32;
    printf("interleaved: DMMA %.2f + DFMA %.2f = %.2f TFLOP/s\n", fd / ms / 1e9, ff / ms / 1e9,
           (fd + ff) / ms / 1e9);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
