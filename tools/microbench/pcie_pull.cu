// PCIe pull bandwidth from mapped pinned host memory: per-warp plain loads vs
// one cp.async.bulk (TMA bulk copy) per warp into shared memory.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pcie_pull pcie_pull.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void plain(const double* __restrict__ src, double* __restrict__ dst, int per_warp) {
  const int w = blockIdx.x, lane = threadIdx.x;
  const double* s = src + (size_t)w * per_warp;
  double* d = dst + (size_t)w * per_warp;
  double v[8];
  for (int e0 = 0; e0 < per_warp; e0 += 256) {
#pragma unroll
    for (int q = 0; q < 8; ++q) { int e = e0 + q * 32 + lane; v[q] = e < per_warp ? s[e] : 0.0; }
#pragma unroll
    for (int q = 0; q < 8; ++q) { int e = e0 + q * 32 + lane; if (e < per_warp) d[e] = v[q]; }
  }
}

__global__ void bulk(const double* __restrict__ src, double* __restrict__ dst, int per_warp) {
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) unsigned long long mbar;
  const int w = blockIdx.x, lane = threadIdx.x;
  const double* s = src + (size_t)w * per_warp;
  double* d = dst + (size_t)w * per_warp;
  const unsigned bytes = per_warp * 8;
  const unsigned mb = (unsigned)__cvta_generic_to_shared(&mbar);
  const unsigned sd = (unsigned)__cvta_generic_to_shared(sm);
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sd), "l"(s), "r"(bytes), "r"(mb) : "memory");
  }
  __syncwarp();
  unsigned ok = 0;
  while (!ok) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(mb) : "memory");
  }
  for (int e = lane; e < per_warp; e += 32) d[e] = sm[e];
}

int main() {
  const int warps = 1000, per_warp = 182;  // ~1.46 MB total (2000 atoms x 26 x 28 B)
  const size_t n = (size_t)warps * per_warp;
  double *h, *hd, *d;
  cudaHostAlloc(&h, n * 8, cudaHostAllocDefault);
  for (size_t i = 0; i < n; ++i) h[i] = (double)i;
  cudaHostGetDevicePointer(&hd, h, 0);
  cudaMalloc(&d, n * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    for (int k = 0; k < 2; ++k) {
      for (int it = 0; it < 3; ++it) {
        if (k == 0) plain<<<warps, 32>>>(hd, d, per_warp);
        else bulk<<<warps, 32, per_warp * 8>>>(hd, d, per_warp);
      }
      cudaEventRecord(a);
      for (int it = 0; it < 20; ++it) {
        if (k == 0) plain<<<warps, 32>>>(hd, d, per_warp);
        else bulk<<<warps, 32, per_warp * 8>>>(hd, d, per_warp);
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      double us = ms * 1e3 / 20;
      printf("%s: %.1f us per %.2f MB -> %.1f GB/s (%s)\n", k ? "bulk " : "plain", us, n * 8 / 1e6,
             n * 8 / (us * 1e-6) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  double chk = 0;
  cudaMemcpy(h, d, 8 * 16, cudaMemcpyDeviceToHost);
  for (int i = 0; i < 16; ++i) chk += h[i];
  printf("check %.0f (expect 120)\n", chk);
  return 0;
}
