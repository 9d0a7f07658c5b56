// util.cu — small device utilities of the host path: the input finiteness
// check of AttnMatrices (reference core.py:72-74) and a 2-D copy passthrough
// used to stream head-group outputs to the host.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "api_common.h"
#include "internal.h"

namespace sa {

// bf16 is non-finite iff its exponent bits are all ones: (x & 0x7f80) == 0x7f80.
// 16-byte loads, grid-stride; one flag store per offending warp.
__global__ void check_finite_kernel(const uint4* __restrict__ x, long long n16, const uint16_t* tail,
                                    int ntail, int32_t* flag) {
  bool bad = false;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  // four independent 16-byte loads in flight per thread (a small grid still
  // streams near HBM rate, leaving SMs to the kernels it runs beside)
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldcs(x + i + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        bad |= (w[k] & 0x7f80u) == 0x7f80u;
        bad |= (w[k] & 0x7f800000u) == 0x7f800000u;
      }
    }
  }
  for (; i < n16; i += stride) {
    const uint4 v = __ldcs(x + i);
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

// AttnMatrices' finiteness scan of q, k, v fused with the KvCache fill
// (runtime.py:197): one pass reads q, k and v once (16-byte streaming loads,
// four in flight per thread) and writes k / v into the cache rows
// [hk, 0..rows) of a cache with `cap` rows per head.  A grid-stride loop over
// a small grid, so it streams beside the compute-bound estimator kernels.
__device__ __forceinline__ bool bf16x8_bad(const uint4& v) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  bool bad = false;
#pragma unroll
  for (int k = 0; k < 4; ++k) bad |= ((w[k] & 0x7f80u) == 0x7f80u) | ((w[k] & 0x7f800000u) == 0x7f800000u);
  return bad;
}
__global__ void scan_fill_kernel(const uint4* __restrict__ q, long long nq16, const uint4* __restrict__ k,
                                 const uint4* __restrict__ v, long long nkv16, long long row16, uint4* ck,
                                 uint4* cv, long long cap16, int32_t* flag) {
  bool bad = false;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  // k / v: rows of (head, n * 8 uint4); cache rows of cap16 uint4 per head
  for (long long i = t0; i < nkv16; i += stride) {
    const uint4 a = __ldcs(k + i), b = __ldcs(v + i);
    bad |= bf16x8_bad(a) | bf16x8_bad(b);
    if (ck) {
      const long long h = i / row16, r = i - h * row16, o = h * cap16 + r;
      ck[o] = a;
      cv[o] = b;
    }
  }
  long long i = t0;
  for (; i + 3 * stride < nq16; i += 4 * stride) {
    uint4 x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = __ldcs(q + i + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) bad |= bf16x8_bad(x[u]);
  }
  for (; i < nq16; i += stride) bad |= bf16x8_bad(__ldcs(q + i));
  if (flag && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *flag = 1;
}

// Chunked variant (one 16 KB piece of q, or 8 KB of k + 8 KB of v, per
// CTA): short-lived CTAs that fill whatever an SM has left beside a
// persistent kernel (the attention kernel leaves room for one per SM).
constexpr int kScanU = 8;
constexpr int kScanT = 128;  // 128 x 48 registers: fits beside two attention CTAs
__global__ void __launch_bounds__(kScanT) scan_fill_chunk_kernel(
    const uint4* __restrict__ q, long long nq16, const uint4* __restrict__ k, const uint4* __restrict__ v,
    long long nkv16, long long row16, uint4* ck, uint4* cv, long long cap16, int32_t* flag, int kv_blocks) {
  bool bad = false;
  if ((int)blockIdx.x < kv_blocks) {
    const long long base = (long long)blockIdx.x * (kScanT * kScanU / 2) + threadIdx.x;
    uint4 a[kScanU / 2], b[kScanU / 2];
#pragma unroll
    for (int u = 0; u < kScanU / 2; ++u) {
      const long long i = base + u * kScanT;
      if (i < nkv16) a[u] = __ldcs(k + i), b[u] = __ldcs(v + i);
    }
#pragma unroll
    for (int u = 0; u < kScanU / 2; ++u) {
      const long long i = base + u * kScanT;
      if (i < nkv16) {
        bad |= bf16x8_bad(a[u]) | bf16x8_bad(b[u]);
        if (ck) {
          const long long h = i / row16, r = i - h * row16, o = h * cap16 + r;
          __stcs(ck + o, a[u]);
          __stcs(cv + o, b[u]);
        }
      }
    }
  } else {
    const long long base = (long long)(blockIdx.x - kv_blocks) * (kScanT * kScanU) + threadIdx.x;
    uint4 x[kScanU];
#pragma unroll
    for (int u = 0; u < kScanU; ++u) {
      const long long i = base + u * kScanT;
      if (i < nq16) x[u] = __ldcs(q + i);
    }
#pragma unroll
    for (int u = 0; u < kScanU; ++u)
      if (base + u * kScanT < nq16) bad |= bf16x8_bad(x[u]);
  }
  if (flag && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *flag = 1;
}

int launch_scan_fill(const void* q, long long nq, const void* k, const void* v, long long nkv, long long row,
                     void* cache_k, void* cache_v, long long cap, int32_t* flag, cudaStream_t st, bool chunked) {
  if ((nq | nkv | row | cap) % 8 != 0) return fail(SA_ERR_DIMENSION, "scan/fill needs 16-byte rows");
  if (chunked) {
    const long long kv_blocks = (nkv / 8 + kScanT * kScanU / 2 - 1) / (kScanT * kScanU / 2);
    const long long q_blocks = (nq / 8 + kScanT * kScanU - 1) / (kScanT * kScanU);
    if (kv_blocks + q_blocks == 0) return SA_OK;
    scan_fill_chunk_kernel<<<(unsigned)(kv_blocks + q_blocks), kScanT, 0, st>>>(
        reinterpret_cast<const uint4*>(q), nq / 8, reinterpret_cast<const uint4*>(k),
        reinterpret_cast<const uint4*>(v), nkv / 8, row / 8, reinterpret_cast<uint4*>(cache_k),
        reinterpret_cast<uint4*>(cache_v), cap / 8, flag, (int)kv_blocks);
    return check_launch("scan_fill_chunk_kernel");
  }
  static const int cap_blocks = [] {
    const char* e = getenv("SA_SCAN_BLOCKS");  // A/B: grid of the fused scan / cache fill
    return e ? atoi(e) : 296;
  }();
  scan_fill_kernel<<<cap_blocks, 256, 0, st>>>(
      reinterpret_cast<const uint4*>(q), nq / 8, reinterpret_cast<const uint4*>(k),
      reinterpret_cast<const uint4*>(v), nkv / 8, row / 8, reinterpret_cast<uint4*>(cache_k),
      reinterpret_cast<uint4*>(cache_v), cap / 8, flag);
  return check_launch("scan_fill_kernel");
}

}  // namespace sa

namespace sa {
int launch_check_finite(const void* x, long long count, int32_t* flag, cudaStream_t st);
}

extern "C" int sa_check_finite_bf16(const void* x, long long count, int32_t* flag, void* stream) {
  return sa::launch_check_finite(x, count, flag, reinterpret_cast<cudaStream_t>(stream));
}

int sa::launch_check_finite(const void* x, long long count, int32_t* flag, cudaStream_t st) {
  using namespace sa;
  if (count < 0 || !flag || (count > 0 && !x)) return fail(SA_ERR_DIMENSION, "bad finiteness-check arguments");
  if (count == 0) return SA_OK;
  const uintptr_t p = reinterpret_cast<uintptr_t>(x);
  if (p % 16 != 0) return fail(SA_ERR_DIMENSION, "finiteness check needs a 16-byte aligned buffer");
  const long long n16 = count / 8;
  const int ntail = (int)(count % 8);
  const int threads = 256;
  long long blocks = (n16 + threads - 1) / threads;
  static const int cap = [] {
    const char* e = getenv("SA_CHECK_BLOCKS");  // A/B: grid cap of the scan
    return e ? atoi(e) : 148;
  }();
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  check_finite_kernel<<<(int)blocks, threads, 0, st>>>(
      reinterpret_cast<const uint4*>(x), n16, reinterpret_cast<const uint16_t*>(x) + n16 * 8, ntail, flag);
  return check_launch("check_finite_kernel");
}

// ---------------------------------------------------- fp32 <-> bf16 staging
namespace sa {
// fp32 -> bf16 (round to nearest even) with the finiteness flag of the fp32
// input (exponent all ones): the AttnMatrices check (core.py:72-74) on the
// rows as given; 32-byte loads, grid-stride.
__global__ void f32_to_bf16_kernel(const float4* __restrict__ x, uint2* __restrict__ y, long long n4,
                                   const float* tail, __nv_bfloat16* ytail, int ntail, int32_t* flag) {
  bool bad = false;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 v = __ldcs(x + i);
    bad |= !isfinite(v.x) | !isfinite(v.y) | !isfinite(v.z) | !isfinite(v.w);
    const __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    y[i] = make_uint2(*reinterpret_cast<const uint32_t*>(&a), *reinterpret_cast<const uint32_t*>(&b));
  }
  if (blockIdx.x == 0 && threadIdx.x < ntail) {
    bad |= !isfinite(tail[threadIdx.x]);
    ytail[threadIdx.x] = __float2bfloat16_rn(tail[threadIdx.x]);
  }
  if (flag && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *flag = 1;
}

__global__ void bf16_to_f32_kernel(const uint2* __restrict__ x, float4* __restrict__ y, long long n4,
                                   const __nv_bfloat16* tail, float* ytail, int ntail) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const uint2 v = __ldcs(x + i);
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.y));
    __stcs(y + i, make_float4(a.x, a.y, b.x, b.y));
  }
  if (blockIdx.x == 0 && threadIdx.x < ntail) ytail[threadIdx.x] = __bfloat162float(tail[threadIdx.x]);
}
}  // namespace sa

extern "C" int sa_f32_to_bf16(const float* x, void* y, long long count, int32_t* flag, void* stream) {
  using namespace sa;
  if (count < 0 || (count > 0 && (!x || !y))) return fail(SA_ERR_DIMENSION, "bad conversion arguments");
  if ((reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(y) & 7))
    return fail(SA_ERR_DIMENSION, "conversion buffers must be 16-byte (fp32) / 8-byte (bf16) aligned");
  if (count == 0) return SA_OK;
  const long long n4 = count / 4;
  const int ntail = (int)(count - n4 * 4);
  const int grid = (int)std::min<long long>(std::max<long long>((n4 + 255) / 256, 1), 4LL * device_sm_count());
  f32_to_bf16_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const float4*>(x), reinterpret_cast<uint2*>(y), n4, x + n4 * 4,
      reinterpret_cast<__nv_bfloat16*>(y) + n4 * 4, ntail, flag);
  return check_launch("f32_to_bf16_kernel");
}

extern "C" int sa_bf16_to_f32(const void* x, float* y, long long count, void* stream) {
  using namespace sa;
  if (count < 0 || (count > 0 && (!x || !y))) return fail(SA_ERR_DIMENSION, "bad conversion arguments");
  if ((reinterpret_cast<uintptr_t>(x) & 7) || (reinterpret_cast<uintptr_t>(y) & 15))
    return fail(SA_ERR_DIMENSION, "conversion buffers must be 8-byte (bf16) / 16-byte (fp32) aligned");
  if (count == 0) return SA_OK;
  const long long n4 = count / 4;
  const int ntail = (int)(count - n4 * 4);
  const int grid = (int)std::min<long long>(std::max<long long>((n4 + 255) / 256, 1), 4LL * device_sm_count());
  bf16_to_f32_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const uint2*>(x), reinterpret_cast<float4*>(y), n4,
      reinterpret_cast<const __nv_bfloat16*>(x) + n4 * 4, y + n4 * 4, ntail);
  return check_launch("bf16_to_f32_kernel");
}

extern "C" int sa_memcpy2d_async(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                                 size_t height, void* stream) {
  using namespace sa;
  const cudaError_t e = cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDefault,
                                          reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(SA_ERR_CUDA, "cudaMemcpy2DAsync: %s", cudaGetErrorString(e));
  return SA_OK;
}

// ------------------------------------------------------------ peer barrier
namespace sa {

struct PeerFlags {
  int32_t* peer[8];
};

__global__ void peer_barrier_kernel(int32_t* flags, PeerFlags pf, int rank, int world, long long timeout_ns) {
  if (threadIdx.x != 0) return;
  const int e = flags[world] + 1;
  flags[world] = e;
  // earlier work on this stream (the epilogue's peer stores) before the flags
  asm volatile("fence.sc.sys;" ::: "memory");
  for (int p = 0; p < world - 1; ++p)
    asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(pf.peer[p] + rank), "r"(e) : "memory");
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int r = 0; r < world; ++r) {
    if (r == rank) continue;
    for (;;) {
      int v;
      asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(flags + r) : "memory");
      if (v - e >= 0) break;
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if ((long long)(t - t0) > timeout_ns) __trap();
      __nanosleep(200);
    }
  }
}

}  // namespace sa

extern "C" int sa_peer_barrier(int32_t* flags, void* const* peer_flags, int rank, int world, int timeout_ms,
                               void* stream) {
  using namespace sa;
  if (world < 1 || world > 8 || rank < 0 || rank >= world || !flags || (world > 1 && !peer_flags) ||
      timeout_ms < 1)
    return fail(SA_ERR_DIMENSION, "sa_peer_barrier: bad arguments (world must be in [1, 8])");
  PeerFlags pf;
  memset(&pf, 0, sizeof(pf));
  for (int p = 0; p < world - 1; ++p) {
    pf.peer[p] = reinterpret_cast<int32_t*>(peer_flags[p]);
    if (!pf.peer[p]) return fail(SA_ERR_DIMENSION, "sa_peer_barrier: null peer flag buffer");
  }
  peer_barrier_kernel<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(flags, pf, rank, world,
                                                                           (long long)timeout_ms * 1000000ll);
  return check_launch("peer_barrier_kernel");
}
