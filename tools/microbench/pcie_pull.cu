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

// U2-prepass pattern: lane idx reads pair idx's three displacement components
// (24-byte stride across lanes); two iterations, serialized (loop) or with all
// loads issued first (hoisted)
template <bool HOIST>
__global__ void aos3(const double* __restrict__ src, double* __restrict__ dst, int per_warp) {
  const int w = blockIdx.x, lane = threadIdx.x;
  const int np = per_warp / 3;
  const double* s = src + (size_t)w * per_warp;
  double* d = dst + (size_t)w * per_warp;
  if (HOIST) {
    double v[2][3];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int idx = lane + 32 * q;
#pragma unroll
      for (int c = 0; c < 3; ++c) v[q][c] = idx < np ? s[idx * 3 + c] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int idx = lane + 32 * q;
      if (idx < np) d[idx] = v[q][0] + v[q][1] * v[q][2];
    }
  } else {
    for (int idx = lane; idx < np; idx += 32) {
      const double a = s[idx * 3], b = s[idx * 3 + 1], c = s[idx * 3 + 2];
      d[idx] = a + b * c;
    }
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
    for (int k = 0; k < 4; ++k) {
      for (int it = 0; it < 3; ++it) {
        if (k == 0) plain<<<warps, 32>>>(hd, d, per_warp);
        else if (k == 1) bulk<<<warps, 32, per_warp * 8>>>(hd, d, per_warp);
        else if (k == 2) aos3<false><<<warps, 32>>>(hd, d, 156);
        else aos3<true><<<warps, 32>>>(hd, d, 156);
      }
      cudaEventRecord(a);
      for (int it = 0; it < 20; ++it) {
        if (k == 0) plain<<<warps, 32>>>(hd, d, per_warp);
        else if (k == 1) bulk<<<warps, 32, per_warp * 8>>>(hd, d, per_warp);
        else if (k == 2) aos3<false><<<warps, 32>>>(hd, d, 156);
        else aos3<true><<<warps, 32>>>(hd, d, 156);
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      double us = ms * 1e3 / 20;
      const char* nm[4] = {"plain", "bulk ", "aos3 loop", "aos3 hoisted"};
      const double bytes = k < 2 ? n * 8.0 : warps * 156 * 8.0;
      printf("%s: %.1f us per %.2f MB -> %.1f GB/s (%s)\n", nm[k], us, bytes / 1e6,
             bytes / (us * 1e-6) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  plain<<<warps, 32>>>(hd, d, per_warp);  // the check reads the plain copy
  double chk = 0;
  cudaMemcpy(h, d, 8 * 16, cudaMemcpyDeviceToHost);
  for (int i = 0; i < 16; ++i) chk += h[i];
  printf("check %.0f (expect 120)\n", chk);
  return 0;
}
