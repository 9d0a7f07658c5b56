// util.cu — small device utilities of the host path: the input finiteness
// check of AttnMatrices (reference core.py:72-74) and a 2-D copy passthrough
// used to stream head-group outputs to the host.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "api_common.h"

namespace sa {

// bf16 is non-finite iff its exponent bits are all ones: (x & 0x7f80) == 0x7f80.
// 16-byte loads, grid-stride; one flag store per offending warp.
__global__ void check_finite_kernel(const uint4* __restrict__ x, long long n16, const uint16_t* tail,
                                    int ntail, int32_t* flag) {
  bool bad = false;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) {
    const uint4 v = __ldg(x + i);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      bad |= (w[k] & 0x7f80u) == 0x7f80u;
      bad |= (w[k] & 0x7f800000u) == 0x7f800000u;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < ntail) bad |= (tail[threadIdx.x] & 0x7f80u) == 0x7f80u;
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *flag = 1;
}

}  // namespace sa

extern "C" int sa_check_finite_bf16(const void* x, long long count, int32_t* flag, void* stream) {
  using namespace sa;
  if (count < 0 || !flag || (count > 0 && !x)) return fail(SA_ERR_DIMENSION, "bad finiteness-check arguments");
  if (count == 0) return SA_OK;
  const uintptr_t p = reinterpret_cast<uintptr_t>(x);
  if (p % 16 != 0) return fail(SA_ERR_DIMENSION, "finiteness check needs a 16-byte aligned buffer");
  const long long n16 = count / 8;
  const int ntail = (int)(count % 8);
  const int threads = 256;
  long long blocks = (n16 + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  check_finite_kernel<<<(int)blocks, threads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const uint4*>(x), n16, reinterpret_cast<const uint16_t*>(x) + n16 * 8, ntail, flag);
  return check_launch("check_finite_kernel");
}

extern "C" int sa_memcpy2d_async(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                                 size_t height, void* stream) {
  using namespace sa;
  const cudaError_t e = cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDefault,
                                          reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(SA_ERR_CUDA, "cudaMemcpy2DAsync: %s", cudaGetErrorString(e));
  return SA_OK;
}
