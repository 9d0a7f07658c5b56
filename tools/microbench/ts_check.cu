// validate: S = Q K^T with A = Q from TMEM (tcgen05.cp 128x256b from SW128 smem) vs SS
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "sm100_common.cuh"
using namespace sa;
__device__ __forceinline__ void utccp_128x256b(uint32_t taddr, uint64_t desc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(desc) : "memory");
}
// element (r, d) of a [rows][128] bf16 matrix stored as two SW128 K-major halves of rows x 64
__device__ int sw_off(int r, int d, int rows) {
  const int half = d >> 6, dd = d & 63;
  const int chunk = dd >> 3, within = dd & 7;
  return half * rows * 128 + r * 128 + ((chunk ^ (r & 7)) << 4) + within * 2;
}
__global__ void k(float* out_ss, float* out_ts, int N) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t holder;
  __shared__ uint64_t bar;
  uint8_t* sQ = smem;            // 128 x 128
  uint8_t* sK = smem + 32768;    // N x 128
  const int warp = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < 128 * 128; e += blockDim.x) {
    const int r = e / 128, d = e % 128;
    *reinterpret_cast<__nv_bfloat16*>(sQ + sw_off(r, d, 128)) = __float2bfloat16((float)((r * 7 + d * 3) % 11 - 5));
  }
  for (int e = threadIdx.x; e < N * 128; e += blockDim.x) {
    const int r = e / 128, d = e % 128;
    *reinterpret_cast<__nv_bfloat16*>(sK + sw_off(r, d, N)) = __float2bfloat16((float)((r * 5 + d * 2) % 7 - 3));
  }
  fence_proxy_async();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&holder, 256);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tb = holder;
  const uint32_t qa = smem_u32(sQ), ka = smem_u32(sK);
  if (warp == 0 && elect_one()) {
    const uint32_t idesc = idesc_bf16_f32(128, N, 0, 0);
    // SS into cols [0, N)
    for (int kk = 0; kk < 8; ++kk)
      mma_ss(tb, sdesc_sw128(qa + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
             sdesc_sw128(ka + (kk >> 2) * (N * 128) + (kk & 3) * 32, 16, 1024), idesc, kk > 0);
    // Q -> TMEM cols [128, 192) via UTCCP, then TS into cols [64, 64 + N)
    for (int kk = 0; kk < 8; ++kk)
      utccp_128x256b(tb + 128 + kk * 8, sdesc_sw128(qa + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024));
    for (int kk = 0; kk < 8; ++kk)
      mma_ts(tb + 64, tb + 128 + kk * 8, sdesc_sw128(ka + (kk >> 2) * (N * 128) + (kk & 3) * 32, 16, 1024), idesc,
             kk > 0);
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc_fence_after();
  const uint32_t lo = static_cast<uint32_t>(warp * 32) << 16;
  uint32_t r1[32], r2[32];
  tmem_ld32(tb + lo, r1);
  tmem_ld32(tb + lo + 64, r2);
  tmem_ld_wait();
  const int row = threadIdx.x;
  for (int c = 0; c < N; ++c) {
    out_ss[row * N + c] = __uint_as_float(r1[c]);
    out_ts[row * N + c] = __uint_as_float(r2[c]);
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc(tb, 256);
}
int main() {
  const int N = 32;
  float *a, *b; cudaMalloc(&a, 128 * N * 4); cudaMalloc(&b, 128 * N * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  k<<<1, 128, 65536>>>(a, b, N);
  cudaError_t e = cudaDeviceSynchronize();
  float ha[128 * 32], hb[128 * 32];
  cudaMemcpy(ha, a, sizeof(ha), cudaMemcpyDeviceToHost);
  cudaMemcpy(hb, b, sizeof(hb), cudaMemcpyDeviceToHost);
  int bad_ss = 0, bad_ts = 0;
  for (int r = 0; r < 128; ++r)
    for (int c = 0; c < N; ++c) {
      double want = 0;
      for (int d = 0; d < 128; ++d) want += (double)((r * 7 + d * 3) % 11 - 5) * ((c * 5 + d * 2) % 7 - 3);
      bad_ss += ha[r * N + c] != (float)want;
      bad_ts += hb[r * N + c] != (float)want;
    }
  printf("%s: SS mismatches %d, TS(utccp) mismatches %d; sample ss %f ts %f\n", cudaGetErrorString(e), bad_ss, bad_ts,
         ha[5 * N + 3], hb[5 * N + 3]);
  return 0;
}
