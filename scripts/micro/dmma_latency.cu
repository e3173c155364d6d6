// Microbenchmark: DMMA (mma.sync m8n8k4 f64) dependency latency and how many
// independent accumulation chains per SM sub-partition saturate the FP64 pipe.
// One CTA per SM; W warps per CTA; each warp runs C independent chains.
// Prints SM-cycles per DMMA per SMSP (issue interval) for each (W, C).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int C>
__global__ void k_chain(double* out, long long* cyc, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double c[C][2];
#pragma unroll
  for (int q = 0; q < C; ++q) c[q][0] = c[q][1] = 0.0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < C; ++q) dmma(c[q], a, b);
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < C; ++q) s += c[q][0] + c[q][1];
  __syncthreads();
  const long long t1 = clock64();
  if (s == 12345.0) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

template <int C>
void run(int warps, double* out, long long* cyc) {
  const int iters = 4096;
  k_chain<C><<<148, 32 * warps>>>(out, cyc, 16);
  k_chain<C><<<148, 32 * warps>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double per_smsp_warps = warps / 4.0 < 1 ? 1 : warps / 4.0;
  // cycles per DMMA per SMSP: total cycles / (DMMAs issued on the busiest SMSP)
  const double dmmas = (double)iters * C * per_smsp_warps;
  printf("warps/CTA %2d  chains/warp %d  cycles/iter/warp %7.2f  SMSP cycles per DMMA %6.2f\n", warps, C,
         (double)h / iters, (double)h / dmmas);
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 8);
  for (int w : {1, 4, 8, 12, 16}) {
    run<1>(w, out, cyc);
    run<2>(w, out, cyc);
    run<3>(w, out, cyc);
    run<4>(w, out, cyc);
    run<6>(w, out, cyc);
    run<8>(w, out, cyc);
  }
  return 0;
}
