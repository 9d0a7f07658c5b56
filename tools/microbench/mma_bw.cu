// micro-benchmark: tcgen05.mma issue rate for SS / TS operand modes and N
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include "sm100_common.cuh"
using namespace sa;
template <int MODE, int N, int M = 128>  // MODE 0: SS (A,B smem), 1: TS (A in TMEM)
__global__ void k(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t holder;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&holder, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tb = holder;
  // zero smem operands
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  fence_proxy_async();
  __syncthreads();
  unsigned long long t0 = clock64();
  if (warp == 0 && elect_one()) {
    constexpr uint32_t idesc = idesc_bf16_f32(M, N, 0, 0);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if (MODE == 0)
          mma_ss(tb, sdesc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                 sdesc_sw128(b + (kk >> 2) * (N * 128) + (kk & 3) * 32, 16, 1024), idesc, 1);
        else
          mma_ts(tb, tb + 256 + kk * 8, sdesc_sw128(b + (kk >> 2) * (N * 128) + (kk & 3) * 32, 16, 1024), idesc, 1);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc(tb, 512);
}
template <int MODE, int N, int M = 128> void run(const char* name, unsigned long long* out) {
  const int iters = 2048;
  cudaFuncSetAttribute(k<MODE, N, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304 + 1024);
  k<MODE, N, M><<<148, 128, 98304 + 1024>>>(iters, out);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h; cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  double per = (double)h / (iters * 8.0);
  double flops = 2.0 * M * N * 16;
  printf("%-10s M=%3d N=%3d: %.1f cyc/instr  (%.0f FLOP/clk/SM) %s\n", name, M, N, per, flops / per,
         cudaGetErrorString(e));
}
int main(int argc, char** argv) {
  unsigned long long* out; cudaMalloc(&out, 1024 * 8);
  const int which = argc > 1 ? atoi(argv[1]) : 0;
  if (which == 0) run<0, 64>("SS", out);
  if (which == 1) run<0, 128>("SS", out);
  if (which == 2) run<0, 256>("SS", out);
  if (which == 3) run<1, 64>("TS", out);
  if (which == 4) run<1, 128>("TS", out);
  if (which == 5) run<1, 256>("TS", out);
  if (which == 6) run<0, 64, 64>("SS", out);
  if (which == 7) run<0, 128, 64>("SS", out);
  if (which == 8) run<1, 64, 64>("TS", out);
  if (which == 9) run<1, 128, 64>("TS", out);
  return 0;
}
