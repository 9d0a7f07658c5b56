// estimate_block.cu — the block-sparse (Block-Cluster) pattern estimator.
//
// Reference: patterns.py:279-287 (block_mean) and patterns.py:290-321
// (build_block_index): pooled logits qb . kb^T * scale over block-causal
// pairs, row softmax, per query block the top-min(k_b, gq+1) key blocks (ties
// to the lower block id) plus the forced diagonal block.
//
// Softmax is strictly increasing within a row, so the top-k of the weights is
// the top-k of the logits; the estimator therefore selects on logits and never
// exponentiates (single GEMM pass, no row statistics).  Pooled means are fp32
// (not bf16-representable), so the GEMM runs on tcgen05 with a split-bf16
// operand: x = hi + lo (hi = bf16(x), lo = bf16(x - hi)), and
//     qb . kb ~= qhi.khi + qlo.khi + qhi.klo   (three K=128 passes)
// which keeps ~16 mantissa bits per product (DESIGN.md §Block estimator).  The
// query operand is stored [qhi | qlo | qhi] (384 wide), the key operand
// [khi | klo] (256 wide); khi feeds two passes from one shared-memory stage.
//
// Epilogue modes: FUSED keeps a per-row top-K list in registers (K = k_b <= 8,
// which covers the auto-selected Block(8, 1)); MATERIALIZE writes the masked
// fp32 logits for a segmented stable top-k (topk.cu) when k_b is large.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstring>

#include "api_common.h"
#include "internal.h"
#include "sa_types.h"
#include "sm100_common.cuh"

namespace sa {

constexpr int kSplitQ = 384;  // query operand [hi | lo | hi]
constexpr int kSplitKey = 256;  // key operand [hi | lo]

// One half-warp per (group, block): lane l pools d = 8 (l % 16) .. + 7 over the
// block's rows in order (fp32, like np.add.reduceat) with 16-byte loads (a
// coalesced 256-byte row per half-warp step, 8 rows in flight).
// out: side 0 -> [G, nb, 384] = [hi | lo | hi]; side 1 -> [G, nb, 256] = [hi | lo].
__global__ void block_pool_kernel(const __nv_bfloat16* __restrict__ x, int G, int n, int b,
                                  int side, __nv_bfloat16* __restrict__ out, float* mean_out,
                                  const int32_t* gate, int gate_val) {
  const int nb = (n + b - 1) / b;
  const long long gid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 4;  // (g, block)
  const int hl = threadIdx.x & 15;
  if (gid >= (long long)G * nb) return;
  const int g = (int)(gid / nb), blk = (int)(gid % nb);
  if (gate && gate[g] != gate_val) return;
  const int r0 = blk * b, r1 = min(n, r0 + b);
  const uint4* src = reinterpret_cast<const uint4*>(x + ((long long)g * n + r0) * kHeadDim) + hl;
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  auto add = [&](const uint4& v) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
      acc[2 * i] += f2.x;
      acc[2 * i + 1] += f2.y;
    }
  };
  int r = r0;
  for (; r + 8 <= r1; r += 8) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(src + (size_t)(r - r0 + u) * (kHeadDim / 8));
#pragma unroll
    for (int u = 0; u < 8; ++u) add(v[u]);
  }
  for (; r < r1; ++r) add(__ldg(src + (size_t)(r - r0) * (kHeadDim / 8)));
  const float inv_cnt = 1.0f / (float)(r1 - r0);
  __nv_bfloat16 hi[8], lo[8];
  float mean[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    mean[u] = acc[u] * inv_cnt;
    hi[u] = __float2bfloat16_rn(mean[u]);
    lo[u] = __float2bfloat16_rn(mean[u] - __bfloat162float(hi[u]));
  }
  const int width = side == 0 ? kSplitQ : kSplitKey;
  __nv_bfloat16* o = out + ((long long)g * nb + blk) * width + 8 * hl;
  *reinterpret_cast<uint4*>(o) = *reinterpret_cast<uint4*>(hi);
  *reinterpret_cast<uint4*>(o + 128) = *reinterpret_cast<uint4*>(lo);
  if (side == 0) *reinterpret_cast<uint4*>(o + 256) = *reinterpret_cast<uint4*>(hi);
  if (mean_out) {
    float* mo = mean_out + ((long long)g * nb + blk) * kHeadDim + 8 * hl;
    *reinterpret_cast<float4*>(mo) = make_float4(mean[0], mean[1], mean[2], mean[3]);
    *reinterpret_cast<float4*>(mo + 4) = make_float4(mean[4], mean[5], mean[6], mean[7]);
  }
}

struct BlockScoreArgs {
  CUtensorMap tmap_qp;  // [HH, nb, 384]
  CUtensorMap tmap_kp;  // [HK, nb, 256]
  int nb, heads, kv_heads, hh_total;
  int nqt;  // ceil(nb / 128)
  float scale;
  int k_b;
  int b;                 // block side (stored in the index)
  // FUSED output: fixed-stride rows of (k_b + 1) slots, INT32_MAX padded
  int32_t* blk_idx;      // per head at hh * head_stride: [nb, k_b + 1]
  int32_t* blk_row_off;  // per head at hh * row_stride: [nb + 1] (absolute offsets into blk_idx); FUSED
                         // rows write their own (no separate row-offset kernel)
  long long head_stride;
  int row_stride;
  // MATERIALIZE output
  float* logits;         // [HH_group, nb, logits_ld] (row-major), indexed by hh - hh_base
  int logits_ld;         // nb rounded up to 4: 16-byte aligned rows for the float4 stores
  int hh_base, hh_count;
  const int32_t* gate;
  int gate_val;
};

constexpr int kBsThreads = 192;
// Two CTAs per SM (one's prologue and epilogue under the other's MMAs):
//   A: [qhi d0-63 | qhi d64-127 | qlo d0-63 | qlo d64-127], 4 x 16 KB (the
//      third product reuses qhi, so the 384-wide operand's last third is not
//      loaded);
//   B: a ring of 3 x 16 KB key chunks, per key tile in the order khi d0, klo d0,
//      khi d1, klo d1, each released right after its MMAs:
//      (qhi.khi + qlo.khi) on a khi chunk, qhi.klo on a klo chunk.
constexpr int kBsSmemA = 0;
constexpr int kBsSmemB = 65536;
constexpr int kBsRing = 3;
constexpr int kBsSmemBar = kBsSmemB + kBsRing * 16384;  // 114688
constexpr int kBsSmemBytes = kBsSmemBar + 256;            // base must be 1024-aligned

enum BBar { BB_A = 0, BB_KF0, BB_KE0 = BB_KF0 + kBsRing, BB_SF0 = BB_KE0 + kBsRing, BB_SF1, BB_SE0, BB_SE1, BB_NUM };

template <int K, bool FUSED>
__global__ void __launch_bounds__(kBsThreads, 2) block_score_kernel(const __grid_constant__ BlockScoreArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if ((smem_u32(smem) & 1023u) != 0u) __trap();  // SWIZZLE_128B tiles need 1024-byte alignment
  // grid (heads, query tiles): every head's heaviest tile is dispatched first
  const int hh = a.hh_base + blockIdx.x;
  if (a.gate && a.gate[hh] != a.gate_val) return;
  const int qt = a.nqt - 1 - blockIdx.y;
  const int cnt = qt + 1;                  // causal key tiles
  uint8_t* sA = smem + kBsSmemA;
  uint8_t* sB = smem + kBsSmemB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBsSmemBar);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + BB_NUM);
  const int warp = warp_id();
  const int bidx = hh / a.heads;
  const int h = hh % a.heads;
  const int hkv = bidx * a.kv_heads + h / (a.heads / a.kv_heads);

  if (threadIdx.x == 0) {
    mbar_init(&bars[BB_A], 1);
    for (int s = 0; s < kBsRing; ++s) {
      mbar_init(&bars[BB_KF0 + s], 1);
      mbar_init(&bars[BB_KE0 + s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bars[BB_SF0 + s], 1);
      mbar_init(&bars[BB_SE0 + s], 128);
    }
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc(tmem_holder, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_holder;

  if (warp == 4) {
    if (elect_one()) {
      mbar_arrive_expect_tx(&bars[BB_A], 65536);
      for (int c = 0; c < 4; ++c) tma_load_3d(sA + c * 16384, &a.tmap_qp, &bars[BB_A], 64 * c, qt * kTile, hh);
      // key chunks of tile j at ring positions 4 j + c: khi d0, klo d0, khi d1, klo d1
      constexpr int kCol[4] = {0, 128, 64, 192};
      for (int j = 0; j < cnt; ++j) {
        for (int c = 0; c < 4; ++c) {
          const int g = 4 * j + c, slot = g % kBsRing;
          if (g >= kBsRing) mbar_wait(&bars[BB_KE0 + slot], ((g / kBsRing) - 1) & 1);
          mbar_arrive_expect_tx(&bars[BB_KF0 + slot], 16384);
          tma_load_3d(sB + slot * 16384, &a.tmap_kp, &bars[BB_KF0 + slot], kCol[c], j * kTile, hkv);
        }
      }
    }
  } else if (warp == 5) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16_f32(128, 128, 0, 0);
      const uint32_t a_addr = smem_u32(sA);
      mbar_wait(&bars[BB_A], 0);
      for (int j = 0; j < cnt; ++j) {
        const int buf = j & 1;
        if (j >= 2) mbar_wait(&bars[BB_SE0 + buf], ((j >> 1) - 1) & 1);
        for (int c = 0; c < 4; ++c) {
          const int g = 4 * j + c, slot = g % kBsRing;
          const int dh = c >> 1;           // d-half of this chunk
          const bool lo = (c & 1) != 0;    // klo chunk
          mbar_wait(&bars[BB_KF0 + slot], (g / kBsRing) & 1);
          tc_fence_after();
          const uint32_t b_addr = smem_u32(sB + slot * 16384);
          // khi chunk: qhi.khi then qlo.khi; klo chunk: qhi.klo
          for (int pass = 0; pass < (lo ? 1 : 2); ++pass) {
            const uint32_t a_chunk = a_addr + (pass ? 32768u : 0u) + dh * 16384u;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_ss(tbase + buf * 128, sdesc_sw128(a_chunk + kk * 32, 16, 1024), sdesc_sw128(b_addr + kk * 32, 16, 1024),
                     idesc, (c > 0 || pass > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&bars[BB_KE0 + slot]);
        }
        mma_commit(&bars[BB_SF0 + buf]);
      }
    }
  } else {
    const int t = threadIdx.x;
    const int gq = qt * kTile + t;
    const bool valid = gq < a.nb;
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    float bv[K];
    int bi[K];
#pragma unroll
    for (int q = 0; q < K; ++q) {
      bv[q] = -INFINITY;
      bi[q] = -1;
    }
    for (int j = 0; j < cnt; ++j) {
      const int buf = j & 1;
      mbar_wait(&bars[BB_SF0 + buf], (j >> 1) & 1);
      tc_fence_after();
      uint32_t s[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(tbase + lane_off + buf * 128 + 32 * c, s[c]);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&bars[BB_SE0 + buf]);
      if (!valid) continue;
      const int g0 = j * kTile;
      const int lim = gq - g0;  // block-causal: gk <= gq
      if (FUSED && K == 1) {
        // tile max by an FMNMX3 tree, then the first column holding it (lowest
        // id wins ties, as does the strict > against the running best)
        float v[128];
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int u = 0; u < 32; ++u)
            v[32 * c + u] = (32 * c + u <= lim) ? __uint_as_float(s[c][u]) * a.scale : -INFINITY;
        float m8[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float m = v[16 * q];
#pragma unroll
          for (int u = 1; u < 16; u += 2) m = fmax3(m, v[16 * q + u], v[16 * q + u + 1 < 16 * q + 16 ? 16 * q + u + 1 : 16 * q + u]);
          m8[q] = m;
        }
        const float tm = fmax3(fmax3(m8[0], m8[1], m8[2]), fmax3(m8[3], m8[4], m8[5]), fmaxf(m8[6], m8[7]));
        if (tm > bv[0]) {
          int first = 127;
#pragma unroll
          for (int c = 127; c >= 0; --c) first = (v[c] == tm) ? c : first;
          bv[0] = tm;
          bi[0] = g0 + first;
        }
      } else if (FUSED) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int u = 0; u < 32; ++u) {
            const int cc = 32 * c + u;
            if (cc <= lim) {
              const float v = __uint_as_float(s[c][u]) * a.scale;
              if (v > bv[K - 1]) {  // strictly greater: ties keep the lower id
                int p = K - 1;
#pragma unroll
                for (int q = K - 1; q > 0; --q) {
                  if (v > bv[q - 1]) {
                    bv[q] = bv[q - 1];
                    bi[q] = bi[q - 1];
                    p = q - 1;
                  }
                }
                bv[p] = v;
                bi[p] = g0 + cc;
              }
            }
          }
      } else {
        float* row = a.logits + ((size_t)(hh - a.hh_base) * a.nb + gq) * a.logits_ld + g0;
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int u = 0; u < 32; u += 4) {
            const int cc = 32 * c + u;
            if (g0 + cc < a.nb) {
              float4 v;
              v.x = (cc + 0 <= lim) ? __uint_as_float(s[c][u + 0]) * a.scale : -INFINITY;
              v.y = (cc + 1 <= lim) ? __uint_as_float(s[c][u + 1]) * a.scale : -INFINITY;
              v.z = (cc + 2 <= lim) ? __uint_as_float(s[c][u + 2]) * a.scale : -INFINITY;
              v.w = (cc + 3 <= lim) ? __uint_as_float(s[c][u + 3]) * a.scale : -INFINITY;
              if (g0 + cc + 3 < a.nb) {
                *reinterpret_cast<float4*>(row + cc) = v;
              } else {
                row[cc] = v.x;
                if (g0 + cc + 1 < a.nb) row[cc + 1] = v.y;
                if (g0 + cc + 2 < a.nb) row[cc + 2] = v.z;
              }
            }
          }
      }
    }
    if (FUSED && valid) {
      // selected ids + forced diagonal block, ascending, INT32_MAX padded
      int ids[K + 1];
      int m = 0;
      bool has_diag = false;
#pragma unroll
      for (int q = 0; q < K; ++q) {
        if (q < a.k_b && bi[q] >= 0) {
          ids[m++] = bi[q];
          has_diag |= (bi[q] == gq);
        }
      }
      if (!has_diag) ids[m++] = gq;
      // insertion sort (m <= K + 1 <= 9)
      for (int x = 1; x < m; ++x) {
        const int v = ids[x];
        int y = x - 1;
        while (y >= 0 && ids[y] > v) {
          ids[y + 1] = ids[y];
          --y;
        }
        ids[y + 1] = v;
      }
      const int stride = a.k_b + 1;
      int32_t* dst = a.blk_idx + (size_t)hh * a.head_stride + (size_t)gq * stride;
      for (int q = 0; q < stride; ++q) dst[q] = q < m ? ids[q] : INT_MAX;
      int32_t* ro = a.blk_row_off + (size_t)hh * a.row_stride;
      ro[gq] = (int32_t)(hh * a.head_stride + (long long)gq * stride);
      if (gq == a.nb - 1) ro[a.nb] = (int32_t)(hh * a.head_stride + (long long)a.nb * stride);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) tmem_dealloc(tbase, 256);
}

__global__ void fixed_row_off_kernel(int32_t* row_off, int hh_total, int nb, int stride,
                                     int row_stride, long long head_stride, const int32_t* gate,
                                     int gate_val) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)hh_total * (nb + 1)) return;
  const int hh = (int)(t / (nb + 1)), g = (int)(t % (nb + 1));
  if (gate && gate[hh] != gate_val) return;
  row_off[(long long)hh * row_stride + g] = (int32_t)(hh * head_stride + (long long)g * stride);
}

int launch_fixed_row_off(int32_t* row_off, int hh_total, int nb, int stride, int row_stride, long long head_stride,
                         const int32_t* gate, int gate_val, cudaStream_t st) {
  const long long tot = (long long)hh_total * (nb + 1);
  fixed_row_off_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(row_off, hh_total, nb, stride, row_stride,
                                                                       head_stride, gate, gate_val);
  return check_launch("fixed_row_off_kernel");
}

// MATERIALIZE: per row, fold the stable top-k output (ascending ids) and the
// forced diagonal into the fixed-stride row.
__global__ void merge_diag_kernel(const int32_t* topk, int k_b, int nb, int32_t* blk_idx,
                                  long long head_stride, int hh_base, int hh_count,
                                  const int32_t* gate, int gate_val) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)hh_count * nb) return;
  const int hl = (int)(t / nb), gq = (int)(t % nb);
  const int hh = hh_base + hl;
  if (gate && gate[hh] != gate_val) return;
  const int keff = min(k_b, gq + 1);
  const int32_t* src = topk + t * (long long)k_b;
  int32_t* dst = blk_idx + hh * head_stride + (long long)gq * (k_b + 1);
  int w = 0;
  bool placed = false;
  for (int q = 0; q < keff; ++q) {
    const int v = src[q];
    if (!placed && gq < v) {
      dst[w++] = gq;
      placed = true;
    }
    if (v == gq) placed = true;
    dst[w++] = v;
  }
  if (!placed) dst[w++] = gq;
  for (; w < k_b + 1; ++w) dst[w] = INT_MAX;
}

}  // namespace sa

// ------------------------------------------------------------------ C ABI
#include "sparseattn_b200.h"

namespace sa {
__global__ void seg_lens_kernel(int32_t* lens, int32_t* ks, int rows, int nb, int k_b) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= rows) return;
  const int gq = t % nb;
  lens[t] = gq + 1;
  ks[t] = min(k_b, gq + 1);
}
}  // namespace sa

namespace sa {

int launch_block_pool(int groups, int n, int b, int side, const void* x, void* split_out,
                      float* mean_out, const int32_t* gate, int gate_val, cudaStream_t st) {
  if (groups < 1 || n < 1) return fail(SA_ERR_DIMENSION, "bad pool shape");
  if (b < 1 || b > n) return fail(SA_ERR_PATTERN_PARAM, "b must be in [1, %d], got %d", n, b);
  const int nb = (n + b - 1) / b;
  const long long items = (long long)groups * nb;  // one half-warp each
  const long long grid = (items * 16 + 255) / 256;
  block_pool_kernel<<<(unsigned)grid, 256, 0, st>>>(
      reinterpret_cast<const __nv_bfloat16*>(x), groups, n, b, side,
      reinterpret_cast<__nv_bfloat16*>(split_out), mean_out, gate, gate_val);
  return check_launch("block_pool_kernel");
}

// MATERIALIZE path: logits of up to kMatHeads heads at a time (<= ~1 GB).
static int logits_ld(int nb) { return (nb + 3) & ~3; }

static int mat_heads(int nb, int hh_total) {
  const long long per = (long long)nb * logits_ld(nb) * 4 + (long long)nb * 64;
  long long g = (1ll << 30) / per;
  if (g < 1) g = 1;
  if (g > hh_total) g = hh_total;
  return (int)g;
}

size_t block_select_ws(int n, int b, int k_b, int hh_total) {
  const int nb = (n + b - 1) / b;
  if (k_b <= 8) return 256;
  const long long g = mat_heads(nb, hh_total);
  return (size_t)g * ((size_t)nb * logits_ld(nb) * 4 + (size_t)nb * k_b * 4 + (size_t)nb * 8) + 1024;
}

int launch_block_select(int batch, int heads, int kv_heads, int n, int b, int k_b, float scale,
                        const void* qp, const void* kp, int32_t* blk_idx, long long head_stride,
                        int32_t* blk_row_off, int row_stride, const int32_t* gate, int gate_val,
                        void* ws, size_t ws_bytes, cudaStream_t st) {
  if (batch < 1 || heads < 1 || kv_heads < 1 || heads % kv_heads)
    return fail(SA_ERR_DIMENSION, "bad head layout");
  if (b < 1 || b > n) return fail(SA_ERR_PATTERN_PARAM, "b must be in [1, %d], got %d", n, b);
  const int nb = (n + b - 1) / b;
  if (k_b < 1 || k_b > nb) return fail(SA_ERR_PATTERN_PARAM, "k_b must be in [1, %d], got %d", nb, k_b);
  if (row_stride < nb + 1 || head_stride < (long long)nb * (k_b + 1))
    return fail(SA_ERR_DIMENSION, "block index strides too small");
  BlockScoreArgs a;
  memset(&a, 0, sizeof(a));
  int rc;
  const int hh_total = batch * heads;
  if ((rc = make_tmap_3d_bf16(&a.tmap_qp, qp, kSplitQ, nb, hh_total, kTile))) return rc;
  if ((rc = make_tmap_3d_bf16(&a.tmap_kp, kp, kSplitKey, nb, batch * kv_heads, kTile))) return rc;
  a.nb = nb;
  a.heads = heads;
  a.kv_heads = kv_heads;
  a.hh_total = hh_total;
  a.nqt = (nb + kTile - 1) / kTile;
  a.scale = scale;
  a.k_b = k_b;
  a.b = b;
  a.blk_idx = blk_idx;
  a.blk_row_off = blk_row_off;
  a.head_stride = head_stride;
  a.row_stride = row_stride;
  a.gate = gate;
  a.gate_val = gate_val;
  if (k_b > 8 && (rc = launch_fixed_row_off(blk_row_off, hh_total, nb, k_b + 1, row_stride, head_stride, gate,
                                              gate_val, st)))
    return rc;  // (the fused k_b <= 8 kernel writes its rows' offsets itself)
  static std::atomic<uint64_t> attr_done{0};
  once_per_device(attr_done, [] {
    cudaFuncSetAttribute(block_score_kernel<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBsSmemBytes);
    cudaFuncSetAttribute(block_score_kernel<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBsSmemBytes);
    cudaFuncSetAttribute(block_score_kernel<4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBsSmemBytes);
    cudaFuncSetAttribute(block_score_kernel<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBsSmemBytes);
    cudaFuncSetAttribute(block_score_kernel<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBsSmemBytes);
  });
  if (k_b <= 8) {
    a.hh_base = 0;
    a.hh_count = hh_total;
    dim3 grid(hh_total, a.nqt);
    if (k_b == 1) block_score_kernel<1, true><<<grid, kBsThreads, kBsSmemBytes, st>>>(a);
    else if (k_b == 2) block_score_kernel<2, true><<<grid, kBsThreads, kBsSmemBytes, st>>>(a);
    else if (k_b <= 4) block_score_kernel<4, true><<<grid, kBsThreads, kBsSmemBytes, st>>>(a);
    else block_score_kernel<8, true><<<grid, kBsThreads, kBsSmemBytes, st>>>(a);
    return check_launch("block_score_kernel<fused>");
  }
  // MATERIALIZE, heads in groups of G through the workspace
  const int G = mat_heads(nb, hh_total);
  const size_t need = block_select_ws(n, b, k_b, hh_total);
  if (!ws || ws_bytes < need) return fail(SA_ERR_DIMENSION, "block_select workspace too small");
  char* p = reinterpret_cast<char*>(ws);
  float* logits = reinterpret_cast<float*>(p);
  if ((reinterpret_cast<uintptr_t>(logits) & 15) != 0) return fail(SA_ERR_DIMENSION, "workspace not 16-byte aligned");
  p += (size_t)G * nb * logits_ld(nb) * 4;
  int32_t* topk = reinterpret_cast<int32_t*>(p);
  p += (size_t)G * nb * k_b * 4;
  int32_t* lens = reinterpret_cast<int32_t*>(p);
  int32_t* ks = lens + (size_t)G * nb;
  seg_lens_kernel<<<(G * nb + 255) / 256, 256, 0, st>>>(lens, ks, G * nb, nb, k_b);
  a.logits = logits;
  a.logits_ld = logits_ld(nb);
  for (int h0 = 0; h0 < hh_total; h0 += G) {
    const int cnt = std::min(G, hh_total - h0);
    a.hh_base = h0;
    a.hh_count = cnt;
    dim3 grid(cnt, a.nqt);
    block_score_kernel<1, false><<<grid, kBsThreads, kBsSmemBytes, st>>>(a);
    if ((rc = check_launch("block_score_kernel<materialize>"))) return rc;
    TopkArgs t{};
    t.scores = logits;
    t.ld = a.logits_ld;
    t.rows = cnt * nb;
    t.n = nb;
    t.lens = lens;
    t.ks = ks;
    t.idx_out = topk;
    t.out_ld = k_b;
    t.gate = gate ? gate + h0 : nullptr;
    t.gate_div = nb;  // row r belongs to head h0 + r / nb
    t.gate_val = gate_val;
    if ((rc = launch_topk(t, st))) return rc;
    merge_diag_kernel<<<(cnt * nb + 255) / 256, 256, 0, st>>>(topk, k_b, nb, blk_idx, head_stride, h0,
                                                              cnt, gate, gate_val);
    if ((rc = check_launch("merge_diag_kernel"))) return rc;
  }
  return SA_OK;
}

}  // namespace sa

extern "C" int sa_block_pool(int groups, int n, int b, int side, const void* x, void* split_out,
                             float* mean_out, void* stream) {
  return sa::launch_block_pool(groups, n, b, side, x, split_out, mean_out, nullptr, 0,
                               reinterpret_cast<cudaStream_t>(stream));
}

extern "C" size_t sa_block_select_workspace(int n, int b, int k_b) {
  return sa::block_select_ws(n, b, k_b, 1);
}

extern "C" int sa_block_select(int batch, int heads, int kv_heads, int n, int b, int k_b,
                               float scale, const void* qp, const void* kp, int32_t* blk_idx,
                               int32_t* blk_row_off, void* ws, size_t ws_bytes, void* stream) {
  const int nb = (n + b - 1) / b;
  return sa::launch_block_select(batch, heads, kv_heads, n, b, k_b, scale, qp, kp, blk_idx,
                                 (long long)nb * (k_b + 1), blk_row_off, nb + 1, nullptr, 0, ws,
                                 ws_bytes, reinterpret_cast<cudaStream_t>(stream));
}

// build_block_index's selection on given fp32 block weights (patterns.py:309-321):
// row gq keeps the stable top-min(k_b, gq + 1) of w[gq, :gq + 1] plus gq itself,
// ascending, in fixed-stride rows of k_b + 1 padded with INT32_MAX.
extern "C" size_t sa_block_topk_workspace(int nb, int k_b) {
  if (nb < 1 || k_b < 1) return 0;
  return ((size_t)nb * (2 + (size_t)k_b)) * 4 + 256;
}

extern "C" int sa_block_topk_f32(const float* w, int nb, long long ld, int k_b, int32_t* blk_out, void* ws,
                                 size_t ws_bytes, void* stream) {
  using namespace sa;
  if (nb < 1 || ld < nb) return fail(SA_ERR_DIMENSION, "bad block weight shape");
  if (k_b < 1 || k_b > nb) return fail(SA_ERR_PATTERN_PARAM, "k_b must be in [1, %d], got %d", nb, k_b);
  if (!w || !blk_out || !ws || ws_bytes < sa_block_topk_workspace(nb, k_b))
    return fail(SA_ERR_DIMENSION, "null pointer or workspace too small");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int32_t* lens = reinterpret_cast<int32_t*>(ws);
  int32_t* ks = lens + nb;
  int32_t* topk = ks + nb;
  seg_lens_kernel<<<(nb + 255) / 256, 256, 0, st>>>(lens, ks, nb, nb, k_b);
  int rc;
  if ((rc = check_launch("seg_lens_kernel"))) return rc;
  TopkArgs t{};
  t.scores = w;
  t.ld = ld;
  t.rows = nb;
  t.n = nb;
  t.lens = lens;
  t.ks = ks;
  t.idx_out = topk;
  t.out_ld = k_b;
  if ((rc = launch_topk(t, st))) return rc;
  merge_diag_kernel<<<(nb + 255) / 256, 256, 0, st>>>(topk, k_b, nb, blk_out, (long long)nb * (k_b + 1), 0, 1,
                                                     nullptr, 0);
  return check_launch("merge_diag_kernel");
}
