// FP64 pipe microbenchmark: DFMA throughput vs independent chains per thread
// (ILP) and resident warps per SM.  Development tool (profiles/ evidence).
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void k(double* out, int iters, double b, double c) {
  double a[ILP];
#pragma unroll
  for (int q = 0; q < ILP; ++q) a[q] = threadIdx.x * 1e-3 + q;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < ILP; ++q) a[q] = fma(a[q], b, c);
  }
  double r = 0;
#pragma unroll
  for (int q = 0; q < ILP; ++q) r += a[q];
  if (r == 12345.678) out[0] = r;
}

template <int ILP>
void run(int warps_per_sm, int nsm, double* d) {
  const int threads = 32 * (warps_per_sm < 32 ? warps_per_sm : 32);
  const int blocks_per_sm = warps_per_sm * 32 / threads;
  const int iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<ILP><<<nsm * blocks_per_sm, threads>>>(d, 100, 1.0, 1e-9);
  cudaEventRecord(e0);
  k<ILP><<<nsm * blocks_per_sm, threads>>>(d, iters, 1.0 - 1e-12, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * ILP * (double)iters * nsm * blocks_per_sm * threads;
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double cycles = ms * 1e-3 * clk * 1e3;
  // DFMA warp-instructions per SM per cycle
  const double wipc = (double)ILP * iters * blocks_per_sm * threads / 32 / cycles;
  printf("ILP=%d warps/SM=%2d  %.2f TFLOP/s  %.3f DFMA warp-inst/clk/SM\n", ILP, warps_per_sm,
         flops / (ms * 1e-3) / 1e12, wipc);
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 8);
  for (int w : {4, 8, 12, 16, 32, 64}) {
    run<1>(w, nsm, d);
    run<2>(w, nsm, d);
    run<4>(w, nsm, d);
    run<8>(w, nsm, d);
  }
  return 0;
}
