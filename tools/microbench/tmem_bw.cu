// micro-benchmark: TMEM read (tcgen05.ld.32x32b.x32) throughput per SM vs warps
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "sm100_common.cuh"
using namespace sa;
__global__ void k(int iters, int nwarps, unsigned long long* out, float* sink) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&holder, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tb = holder;
  float acc = 0.f;
  unsigned long long t0 = clock64();
  if (warp < nwarps) {
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    for (int i = 0; i < iters; ++i) {
      uint32_t r[32];
      tmem_ld32(tb + lane_off + ((i * 32 + warp * 64) & 511), r);
      tmem_ld_wait();
#pragma unroll
      for (int c = 0; c < 32; ++c) acc += __uint_as_float(r[c]);
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc(tb, 512);
}
int main() {
  unsigned long long* out; float* sink;
  cudaMalloc(&out, 1024 * 8); cudaMalloc(&sink, 1024 * 1024 * 4);
  const int iters = 4096;
  for (int nw : {1, 2, 4, 8, 16}) {
    int threads = (nw < 4 ? 4 : nw) * 32;
    k<<<148, threads>>>(iters, nw, out, sink);
    cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, out, 148 * 8, cudaMemcpyDeviceToHost);
    double bytes = (double)iters * nw * 32 * 32 * 4;
    printf("warps %2d: %llu cyc  -> %.1f B/cyc/SM (%s)\n", nw, h[0], bytes / h[0], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
