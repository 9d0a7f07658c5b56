// decode.cu — one decode step on device: the new token's queries attend over
// the whole KV cache (reference runtime.py:209-242 decode_step: dense
// attention of the appended row over every cached position).
//
// A GEMV-shaped, HBM-bound problem (each cached K/V byte is used by the g = H/HK
// query heads of its group once), so it runs on CUDA cores as a split-K pass:
//   decode_partial_kernel: CTA (batch * kv head, key chunk of 256) — scores of
//     the group's g heads against its keys (thread per key), chunk softmax
//     statistics (warp per head), P·V with coalesced V rows (thread per
//     column pair and key quarter); writes (max2, sum, o[d]) per head.
//   decode_combine_kernel: CTA per (batch, query head) folds the chunks in order.
// K and V are read once per kv head, in place in the cache's
// [B, HK, capacity, d] layout (no staging copy).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "api_common.h"
#include "internal.h"

namespace sa {

constexpr int kDecChunkMax = 1024;  // keys per CTA: 256 .. 1024, about 2048 CTAs per call
constexpr int kDecThreads = 256;
constexpr int kDecMaxG = 4;       // query heads per kv head and pass (registers: 4 x 8 accumulators)
constexpr int kDecMaxD = 128;

template <class T>
__device__ __forceinline__ float ld1(const T* p);
template <>
__device__ __forceinline__ float ld1<float>(const float* p) { return __ldg(p); }
template <>
__device__ __forceinline__ float ld1<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(__ldg(p)); }
// W consecutive elements (W = 2: even offset; W = 8: 16-byte aligned)
template <class T, int W>
__device__ __forceinline__ void ldw(const T* p, float (&v)[W]) {
  if constexpr (W == 8) {
    if constexpr (sizeof(T) == 4) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(p));
      const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
      v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
      const uint4 a = __ldg(reinterpret_cast<const uint4*>(p));
      const uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 x = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
        v[2 * i] = x.x;
        v[2 * i + 1] = x.y;
      }
    }
  } else if constexpr (W == 2) {
    if constexpr (sizeof(T) == 4) {
      const float2 x = __ldg(reinterpret_cast<const float2*>(p));
      v[0] = x.x;
      v[1] = x.y;
    } else {
      const float2 x = __bfloat1622float2(__ldg(reinterpret_cast<const __nv_bfloat162*>(p)));
      v[0] = x.x;
      v[1] = x.y;
    }
  } else {
    v[0] = ld1<T>(p);
  }
}

// part layout: [B * HK, nsplit, g, d + 2] floats: (max2, sum, o[0..d)).
// W = 8 (d % 8 == 0): 16-byte loads; W = 2 (even d): pairs; W = 1 otherwise.
template <class T, int W>
__global__ void __launch_bounds__(kDecThreads, 3) decode_partial_kernel(const float* __restrict__ q, const T* __restrict__ kc,
                                                                     const T* __restrict__ vc, int heads, int kv_heads, int n,
                                                                     int d, int cap, float scale_log2, int h_off, int g,
                                                                     int chunk, float* __restrict__ part) {
  // this pass: query heads [h_off, h_off + g) of each kv group (g <= kDecMaxG)
  const int bkh = blockIdx.x, split = blockIdx.y, nsplit = gridDim.y;
  const int gt = heads / kv_heads;
  const int b = bkh / kv_heads, kh = bkh % kv_heads;
  const int c0 = split * chunk, len = min(chunk, n - c0);
  constexpr int kCols = kDecMaxD / W;           // column groups of a V row
  constexpr int kKq = kDecThreads / kCols;      // key interleave of the P·V pass
  // partial P·V slots: one per key interleave, or per warp when W = 8 (two
  // interleaves per warp are folded with a shuffle first)
  constexpr int kSlots = W == 8 ? kDecThreads / 32 : kKq;
  __shared__ float qs[kDecMaxG][kDecMaxD];
  __shared__ float sc[kDecMaxG][kDecChunkMax];
  __shared__ float stat[kDecMaxG][2];
  __shared__ float po[kSlots][kDecMaxG][kDecMaxD];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < g * kDecMaxD; i += kDecThreads) {
    const int h = i / kDecMaxD, c = i % kDecMaxD;
    qs[h][c] = c < d ? q[((size_t)b * heads + kh * gt + h_off + h) * d + c] * scale_log2 : 0.f;
  }
  __syncthreads();
  const size_t base = ((size_t)bkh * cap) * d;
  // 1. scores (log2 domain), thread per key
  for (int key = tid; key < len; key += kDecThreads) {
    const T* kr = kc + base + (size_t)(c0 + key) * d;
    float acc[kDecMaxG];
#pragma unroll
    for (int h = 0; h < kDecMaxG; ++h) acc[h] = 0.f;
    if constexpr (W == 8) {
      // 8 x 16-byte loads of the row in flight, then the dot products
      constexpr int E = 16 / (int)sizeof(T);
      for (int cb = 0; cb < d; cb += 8 * E) {
        uint4 raw[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          raw[u] = cb + u * E < d ? __ldg(reinterpret_cast<const uint4*>(kr + cb + u * E)) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          float kv[E];
          if constexpr (E == 8) {
            const uint32_t w4[4] = {raw[u].x, raw[u].y, raw[u].z, raw[u].w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float2 x = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w4[i]));
              kv[2 * i] = x.x;
              kv[2 * i + 1] = x.y;
            }
          } else {
            kv[0] = __uint_as_float(raw[u].x);
            kv[1] = __uint_as_float(raw[u].y);
            kv[2] = __uint_as_float(raw[u].z);
            kv[3] = __uint_as_float(raw[u].w);
          }
          const int c = cb + u * E;
          if (c < d) {
#pragma unroll
            for (int h = 0; h < kDecMaxG; ++h)
              if (h < g) {
#pragma unroll
                for (int e = 0; e < E; ++e) acc[h] += qs[h][c + e] * kv[e];
              }
          }
        }
      }
    } else {
      for (int c = 0; c < d; c += W) {
        float kv[W];
        ldw<T, W>(kr + c, kv);
#pragma unroll
        for (int h = 0; h < kDecMaxG; ++h)
          if (h < g) {
#pragma unroll
            for (int w = 0; w < W; ++w) acc[h] += qs[h][c + w] * kv[w];
          }
      }
    }
#pragma unroll
    for (int h = 0; h < kDecMaxG; ++h)
      if (h < g) sc[h][key] = acc[h];
  }
  __syncthreads();
  // 2. chunk max / exp / sum per head (warp per head)
  for (int h = warp; h < g; h += kDecThreads / 32) {
    float m = -INFINITY;
    for (int t = lane; t < len; t += 32) m = fmaxf(m, sc[h][t]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float s = 0.f;
    for (int t = lane; t < len; t += 32) {
      const float p = exp2f(sc[h][t] - m);
      sc[h][t] = p;
      s += p;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      stat[h][0] = m;
      stat[h][1] = s;
    }
  }
  __syncthreads();
  // 3. o = P V: thread (column group cg, key interleave kq); V rows read coalesced
  const int cg = tid % kCols, kq = tid / kCols;
  float acc[kDecMaxG][W];
#pragma unroll
  for (int h = 0; h < kDecMaxG; ++h)
#pragma unroll
    for (int w = 0; w < W; ++w) acc[h][w] = 0.f;
  if (cg * W < d) {
    // 4 rows' loads in flight per step
    for (int t0 = kq; t0 < len; t0 += 4 * kKq) {
      float vv[4][W];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int t = t0 + u * kKq;
        if (t < len) {
          ldw<T, W>(vc + base + (size_t)(c0 + t) * d + cg * W, vv[u]);
        } else {
#pragma unroll
          for (int w = 0; w < W; ++w) vv[u][w] = 0.f;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int t = min(t0 + u * kKq, len - 1);  // rows past len carry v = 0
#pragma unroll
        for (int h = 0; h < kDecMaxG; ++h)
          if (h < g) {
            const float p = sc[h][t];
#pragma unroll
            for (int w = 0; w < W; ++w) acc[h][w] += p * vv[u][w];
          }
      }
    }
  }
  if constexpr (W == 8) {
#pragma unroll
    for (int h = 0; h < kDecMaxG; ++h)
#pragma unroll
      for (int w = 0; w < W; ++w) acc[h][w] += __shfl_xor_sync(0xffffffffu, acc[h][w], 16);
  }
  if (W != 8 || lane < 16) {
    const int slot = W == 8 ? warp : kq;
#pragma unroll
    for (int h = 0; h < kDecMaxG; ++h)
      if (h < g) {
#pragma unroll
        for (int w = 0; w < W; ++w) po[slot][h][cg * W + w] = acc[h][w];
      }
  }
  __syncthreads();
  float* dst = part + ((size_t)bkh * nsplit + split) * g * (d + 2);
  for (int i = tid; i < g * (d + 2); i += kDecThreads) {
    const int h = i / (d + 2), c = i % (d + 2);
    float v;
    if (c == 0) {
      v = stat[h][0];
    } else if (c == 1) {
      v = stat[h][1];
    } else {
      v = 0.f;
#pragma unroll
      for (int k = 0; k < kSlots; ++k) v += po[k][h][c - 2];
    }
    dst[i] = v;
  }
}

// out[b, h, c] = sum_s 2^(m_s - M) o_s[c] / sum_s 2^(m_s - M) l_s over the
// chunks s.  All chunk statistics are read in parallel (the weights land in
// shared memory), then thread c sums column c over the chunks with 8 loads in
// flight.
constexpr int kDecMaxSplit = 8192;  // chunks per kv head: up to 8M cached rows at 1024 keys per chunk

// keys per CTA for n cached rows over `groups` = batch * kv_heads
static int dec_chunk(int n, int groups) {
  int c = 256;
  while (c < kDecChunkMax && (long long)n * groups / c > 2048) c *= 2;
  return c;
}
__global__ void __launch_bounds__(128) decode_combine_kernel(const float* __restrict__ part, int heads, int kv_heads,
                                                             int d, int nsplit, int h_off, int g, float* __restrict__ out) {
  // CTA (batch * kv head, head of this pass)
  const int bkh = blockIdx.x / g, hg = blockIdx.x % g;
  const int gt = heads / kv_heads;
  const int b = bkh / kv_heads, kh = bkh % kv_heads;
  const int bh = b * heads + kh * gt + h_off + hg;
  const float* p = part + (size_t)bkh * nsplit * g * (d + 2) + (size_t)hg * (d + 2);
  const size_t sstride = (size_t)g * (d + 2);
  __shared__ float wsm[kDecMaxSplit];
  __shared__ float red[4];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float m = -INFINITY;
  for (int s = tid; s < nsplit; s += 128) m = fmaxf(m, p[s * sstride]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) red[warp] = m;
  __syncthreads();
  const float M = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
  __syncthreads();
  float den = 0.f;
  for (int s = tid; s < nsplit; s += 128) {
    const float w = exp2f(p[s * sstride] - M);
    wsm[s] = w;
    den += w * p[s * sstride + 1];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
  if (lane == 0) red[warp] = den;
  __syncthreads();
  den = (red[0] + red[1]) + (red[2] + red[3]);
  for (int c = tid; c < d; c += 128) {
    float num[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    int s = 0;
    for (; s + 8 <= nsplit; s += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) num[u] += wsm[s + u] * p[(s + u) * sstride + 2 + c];
    }
    for (; s < nsplit; ++s) num[0] += wsm[s] * p[s * sstride + 2 + c];
    out[(size_t)bh * d + c] = (((num[0] + num[1]) + (num[2] + num[3])) + ((num[4] + num[5]) + (num[6] + num[7]))) / den;
  }
}

}  // namespace sa

extern "C" size_t sa_decode_workspace(int batch, int heads, int kv_heads, int n, int d) {
  if (batch < 1 || heads < 1 || kv_heads < 1 || n < 1 || d < 1) return 0;
  const int chunk = sa::dec_chunk(n, batch * kv_heads);
  const size_t nsplit = (size_t)(n + chunk - 1) / chunk;
  const size_t g = (size_t)(heads / kv_heads < sa::kDecMaxG ? heads / kv_heads : sa::kDecMaxG);
  return (size_t)batch * kv_heads * g * nsplit * (d + 2) * sizeof(float);
}

extern "C" int sa_decode_attn(int batch, int heads, int kv_heads, int n, int d, int capacity, float scale,
                              const float* q, const void* k_cache, const void* v_cache, int kv_dtype, float* out,
                              void* ws, size_t ws_bytes, void* stream) {
  using namespace sa;
  if (batch < 1 || heads < 1 || kv_heads < 1 || n < 1 || heads % kv_heads)
    return fail(SA_ERR_DIMENSION, "bad decode shape (batch %d, heads %d, kv_heads %d, n %d)", batch, heads, kv_heads, n);
  if (d < 1 || d > kDecMaxD) return fail(SA_ERR_DIMENSION, "decode head_dim must be in [1, 128], got %d", d);
  if (capacity < n) return fail(SA_ERR_DIMENSION, "cache capacity %d below length %d", capacity, n);
  if ((long long)n > (long long)kDecMaxSplit * kDecChunkMax)
    return fail(SA_ERR_DIMENSION, "decode supports up to %lld cached rows", (long long)kDecMaxSplit * kDecChunkMax);
  if (!(scale > 0.f) || !std::isfinite(scale)) return fail(SA_ERR_DIMENSION, "bad scale");
  if (!q || !k_cache || !v_cache || !out || !ws) return fail(SA_ERR_DIMENSION, "null pointer argument");
  if (ws_bytes < sa_decode_workspace(batch, heads, kv_heads, n, d)) return fail(SA_ERR_DIMENSION, "decode workspace too small");
  const int chunk = dec_chunk(n, batch * kv_heads);
  const int nsplit = (n + chunk - 1) / chunk;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const float sl2 = scale * 1.4426950408889634f;
  dim3 grid(batch * kv_heads, nsplit);
  float* part = reinterpret_cast<float*>(ws);
  const int gt = heads / kv_heads;
  int rc;
  for (int h_off = 0; h_off < gt; h_off += kDecMaxG) {  // query-head passes of <= kDecMaxG per kv head
    const int g = gt - h_off < kDecMaxG ? gt - h_off : kDecMaxG;
    const bool al16 = ((reinterpret_cast<uintptr_t>(k_cache) | reinterpret_cast<uintptr_t>(v_cache)) & 15) == 0;
    const int w = (d % 8 == 0 && al16) ? 8 : (d % 2 == 0 ? 2 : 1);
#define SA_DEC(T, W)                                                                                          \
  decode_partial_kernel<T, W><<<grid, kDecThreads, 0, st>>>(q, reinterpret_cast<const T*>(k_cache),         \
                                                            reinterpret_cast<const T*>(v_cache), heads,       \
                                                            kv_heads, n, d, capacity, sl2, h_off, g, chunk, part)
    if (kv_dtype == 0) {
      if (w == 8) SA_DEC(float, 8); else if (w == 2) SA_DEC(float, 2); else SA_DEC(float, 1);
    } else if (kv_dtype == 1) {
      if (w == 8) SA_DEC(__nv_bfloat16, 8); else if (w == 2) SA_DEC(__nv_bfloat16, 2); else SA_DEC(__nv_bfloat16, 1);
    } else {
      return fail(SA_ERR_DIMENSION, "kv_dtype must be 0 (fp32) or 1 (bf16)");
    }
    if ((rc = check_launch("decode_partial_kernel"))) return rc;
    decode_combine_kernel<<<batch * kv_heads * g, 128, 0, st>>>(part, heads, kv_heads, d, nsplit, h_off, g, out);
    if ((rc = check_launch("decode_combine_kernel"))) return rc;
  }
#undef SA_DEC
  return SA_OK;
}
