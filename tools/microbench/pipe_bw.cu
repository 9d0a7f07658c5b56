// micro-benchmark: per-SM throughput of FFMA, FFMA2, FADD2, MUFU.EX2, FMNMX3 with 16 warps
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "sm100_common.cuh"
using namespace sa;
template <int OP>
__global__ void k(int iters, unsigned long long* out, float* sink, float s0) {
  float2 a[8], b = make_float2(s0, s0 * 0.5f), c = make_float2(0.999f, 0.998f);
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = make_float2(threadIdx.x * 1e-3f + j, j * 0.5f);
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) { a[j].x = fmaf(a[j].x, c.x, b.x); a[j].y = fmaf(a[j].y, c.y, b.y); }  // 2 FFMA
      if (OP == 1) a[j] = ffma2(a[j], c, b);                                             // 1 FFMA2
      if (OP == 2) a[j] = fadd2(a[j], b);                                                // 1 FADD2
      if (OP == 3) { a[j].x = fast_exp2(a[j].x); a[j].y = fast_exp2(a[j].y); }           // 2 MUFU
      if (OP == 4) { a[j].x = fmax3(a[j].x, b.x, c.x); a[j].y = fmax3(a[j].y, b.y, c.y); } // 2 FMNMX3
      if (OP == 5) { a[j].x = a[j].x + b.x; a[j].y = a[j].y + b.y; }                      // 2 FADD
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j].x + a[j].y;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int OP> void run(const char* name, unsigned long long* out, float* sink) {
  const int iters = 4096, threads = 512;
  k<OP><<<148, threads>>>(iters, out, sink, 1e-3f);
  cudaDeviceSynchronize();
  unsigned long long h; cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  double elems = (double)iters * 16 * threads;  // 16 float values per thread per iter
  printf("%-8s %8llu cyc: %.1f elem-ops/clk/SM (%.2f clk per warp-instr-equivalent of 32 elems per SMSP)\n",
         name, h, elems / h, h / (elems / 128.0));
}
int main() {
  unsigned long long* out; float* sink;
  cudaMalloc(&out, 1024 * 8); cudaMalloc(&sink, 1024 * 1024 * 4);
  run<0>("FFMA", out, sink); run<1>("FFMA2", out, sink); run<2>("FADD2", out, sink);
  run<3>("MUFU", out, sink); run<4>("FMNMX3", out, sink); run<5>("FADD", out, sink);
  return 0;
}
