// micro-benchmark: does tcgen05.ld traffic from other warps slow a tcgen05.mma
// chain on the same SM?  One CTA per SM: warp 0 issues SS (or TS) M=128 N=128
// K=16 MMAs into TMEM columns [0, 128); R reader warps (two per lane quarter
// at R = 8) loop tcgen05.ld.32x32b.x32 over columns [256, 384) until the MMAs
// are done.  Prints MMA cycles per instruction and the readers' TMEM bytes/clk.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include "sm100_common.cuh"
using namespace sa;
template <int MODE>
__global__ void k(int iters, int readers, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t holder;
  __shared__ uint64_t bar;
  __shared__ volatile int stop;
  __shared__ unsigned long long rbytes;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); stop = 0; rbytes = 0; }
  if (warp == 0) tmem_alloc(&holder, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tb = holder;
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  fence_proxy_async();
  __syncthreads();
  unsigned long long t0 = clock64();
  if (warp == 0) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16_f32(128, 128, 0, 0);
      const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
      if (MODE == 1)
        for (int kk = 0; kk < 8; ++kk) utccp_128x256b(tb + 384 + kk * 8, sdesc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024));
      for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          if (MODE == 0)
            mma_ss(tb, sdesc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                   sdesc_sw128(b + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), idesc, 1);
          else
            mma_ts(tb, tb + 384 + kk * 8, sdesc_sw128(b + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), idesc, 1);
        }
      }
      mma_commit(&bar);
      mbar_wait(&bar, 0);
      out[2 * blockIdx.x] = clock64() - t0;
      stop = 1;
    }
  } else if (warp >= 4 && warp < 4 + readers) {
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    unsigned long long n = 0;
    uint32_t r[32];
    uint32_t acc = 0;
    while (!stop) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        tmem_ld32(tb + lane_off + 256 + 32 * c, r);
        tmem_ld_wait();
        acc ^= r[c];
      }
      n += 4 * 32 * 32 * 4;  // bytes per warp per loop
    }
    if ((threadIdx.x & 31) == 0) atomicAdd(&rbytes, n);
    if (acc == 0x12345678u) out[1] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) out[2 * blockIdx.x + 1] = rbytes;
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc(tb, 512);
}
template <int MODE> void run(int readers, unsigned long long* out) {
  const int iters = 4096;
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304 + 1024);
  k<MODE><<<148, 384, 98304 + 1024>>>(iters, readers, out);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[2]; cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
  const double per = (double)h[0] / (iters * 8.0);
  printf("%s N=128, %d TMEM-reader warps: %.1f cyc/MMA, readers %.1f B/clk/SM %s\n", MODE ? "TS" : "SS", readers, per,
         (double)h[1] / (double)h[0], cudaGetErrorString(e));
}
int main() {
  unsigned long long* out; cudaMalloc(&out, 1024 * 8);
  for (int r : {0, 4, 8}) run<0>(r, out);
  for (int r : {0, 4, 8}) run<1>(r, out);
  return 0;
}
