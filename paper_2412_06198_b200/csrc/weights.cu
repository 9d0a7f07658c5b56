// weights.cu — dense n x n attention weights of a realised index (the
// need_weights=True return of patterns.py:422-434 / 466-467 and core.py:152),
// plus an fp32 block_mean for the per-head API (patterns.py:279-287).
//
// Weights are a debug/selection-size path (typically n <= 4096, search.DENSE_EVAL_CAP):
// w[i, j] = exp(q_i . k_j * scale - lse_i) on the index, 0 elsewhere, with the
// row log-sum-exp taken from the attention kernel so rows match its softmax.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "api_common.h"
#include "internal.h"
#include "sa_types.h"

namespace sa {

__device__ __forceinline__ bool index_allows(const sa_head_index& ix, int hh, int n, int i, int j) {
  const int fam = ix.family[hh];
  if (fam == FAM_DENSE_NC) return true;
  if (j > i) return false;
  if (fam == FAM_DENSE) return true;
  if (fam == FAM_TRI) return (i - j < ix.tri_window[hh]) || (j < ix.tri_sinks[hh]) || i == j;
  if (fam == FAM_VS || fam == FAM_VS_NOEYE) {
    if (i == j && fam == FAM_VS) return true;
    const uint32_t* cb = ix.colbits + (size_t)hh * ix.vs_words;
    const uint32_t* dr = ix.diagrev + (size_t)hh * ix.vs_words;
    const int p = n + 127 - (i - j);
    return ((cb[j >> 5] >> (j & 31)) & 1u) || ((dr[p >> 5] >> (p & 31)) & 1u);
  }
  const int b = ix.blk_b[hh];
  const int32_t* ro = ix.blk_row_off + (size_t)hh * ix.blk_row_stride;
  const int gq = i / b, gk = j / b;
  for (int k = ro[gq]; k < ro[gq + 1]; ++k) {
    const int v = ix.blk_idx[k];
    if (v == gk) return true;
    if (v > gk) break;
  }
  return false;
}

__global__ void weights_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k,
                               const float* __restrict__ lse, sa_head_index ix, int hh, int hkv, int n,
                               float scale, float* __restrict__ w) {
  __shared__ float qs[16][129];
  __shared__ float ks[16][129];
  const int i0 = blockIdx.y * 16, j0 = blockIdx.x * 16;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 16 x 16
  for (int e = ty * 16 + tx; e < 16 * kHeadDim; e += 256) {
    const int r = e / kHeadDim, d = e % kHeadDim;
    qs[r][d] = (i0 + r < n) ? __bfloat162float(q[((size_t)hh * n + i0 + r) * kHeadDim + d]) : 0.f;
    ks[r][d] = (j0 + r < n) ? __bfloat162float(k[((size_t)hkv * n + j0 + r) * kHeadDim + d]) : 0.f;
  }
  __syncthreads();
  const int i = i0 + ty, j = j0 + tx;
  if (i >= n || j >= n) return;
  float out = 0.f;
  if (index_allows(ix, hh, n, i, j)) {
    float acc = 0.f;
    for (int d = 0; d < kHeadDim; ++d) acc = fmaf(qs[ty][d], ks[tx][d], acc);
    out = expf(acc * scale - lse[(size_t)hh * n + i]);
  }
  w[(size_t)i * n + j] = out;
}

__global__ void mean_f32_kernel(const float* __restrict__ x, int n, int d, int b, float* __restrict__ out) {
  const int blk = blockIdx.x;
  const int r0 = blk * b, r1 = min(n, r0 + b);
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float acc = 0.f;
    for (int r = r0; r < r1; ++r) acc += x[(size_t)r * d + c];
    out[(size_t)blk * d + c] = acc / (float)(r1 - r0);
  }
}

}  // namespace sa

// w: [n, n] fp32 for head hh (batch-folded index), lse from sa_attn_sparse.
extern "C" int sa_attn_weights(int heads, int kv_heads, int n, int hh, float scale, const void* q,
                               const void* k, const float* lse, const sa_head_index* index,
                               float* w, void* stream) {
  using namespace sa;
  // the dense n x n result is what the reference returns (numpy, any n); the
  // only limit here is the 16-row grid (y < 65536 blocks)
  if (n < 1 || n > 65535 * 16) return fail(SA_ERR_DIMENSION, "weights path supports 1 <= n <= %d", 65535 * 16);
  if (heads < 1 || kv_heads < 1 || heads % kv_heads) return fail(SA_ERR_DIMENSION, "bad head layout");
  if (!q || !k || !lse || !index || !w) return fail(SA_ERR_DIMENSION, "null pointer argument");
  const int b = hh / heads, h = hh % heads;
  const int hkv = b * kv_heads + h / (heads / kv_heads);
  dim3 grid((n + 15) / 16, (n + 15) / 16), block(16, 16);
  weights_kernel<<<grid, block, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const __nv_bfloat16*>(q), reinterpret_cast<const __nv_bfloat16*>(k), lse,
      *index, hh, hkv, n, scale, w);
  return check_launch("weights_kernel");
}

extern "C" int sa_block_mean_f32(const float* x, int n, int d, int b, float* out, void* stream) {
  using namespace sa;
  if (n < 1 || d < 1) return fail(SA_ERR_DIMENSION, "bad block_mean shape");
  if (b < 1) return fail(SA_ERR_PATTERN_PARAM, "block side must be >= 1, got %d", b);
  if (!x || !out) return fail(SA_ERR_DIMENSION, "null pointer argument");
  const int nb = (n + b - 1) / b;
  mean_f32_kernel<<<nb, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(x, n, d, b, out);
  return check_launch("mean_f32_kernel");
}
