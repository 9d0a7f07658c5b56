// block_screen.cu — the Block-Cluster index for small k_b (<= 8, the auto
// search's Block(8, 1)) by fp16 tensor passes and an exact refine.  Opt-in
// inside sa_prefill (SA_BLOCK_SCREEN=1) and the sa_block_index_bf16 entry
// point: at 32K both variants measured slower than the split-bf16 GEMM they
// would replace: for 2 <= k_b <= 8 the one-pass screen's top-T
// tracking epilogue is issue/latency-bound; for k_b = 1 the two-pass top-1
// (block_top1_kernel) runs its GEMM ~13% faster than the split GEMM, but the
// second read of every logit from TMEM, the exact refine and the fp16 pooling
// give the gain back.
//
// Reference: patterns.py:279-287 (block_mean) and patterns.py:290-321
// (build_block_index): per query block, the top-min(k_b, gq+1) causal key
// blocks by pooled logit (softmax is monotone in a row), ties to the lower id,
// plus the forced diagonal block.
//
// The split-bf16 GEMM of estimate_block.cu spends three K=128 tensor passes per
// logit to get ~16 mantissa bits everywhere, although only the few logits near
// each row's cut decide anything.  Here:
//   1. block_pool16_kernel pools each block in fp32 (true division by the row
//      count, as np.add.reduceat / counts) and writes the mean and its L2 norm;
//      query blocks also get an fp16 copy normalised by their own power of two
//      2^e (max |x 2^-e| in [2^13, 2^14): no overflow, no relative loss to
//      subnormals); key blocks share ONE power of two per kv head (the head's
//      largest block, key_f16_kernel), so the screened logit needs no
//      per-column rescaling;
//   2. block_screen_kernel runs ONE fp16 tcgen05 pass per (query tile, key
//      tile): acc is the row's logit up to a per-row power of two (irrelevant
//      to the order), within
//          E = (2^-9 + 2^-15) |x~| |y~|max + 2^-21 (|x~| + |y~|max) + 2^-40
//      of the exact pooled product (two fp16 roundings of 2^-11 and fp32
//      accumulation, the 7 low mantissa bits that carry the column index,
//      subnormal terms).  Per row it keeps the T = k_b + 3 largest CHUNK maxima
//      (32 columns; the column rides in the low mantissa bits, so a max tree
//      yields its argmax) and U = the largest value not tracked (every chunk's
//      second largest, every evicted or rejected chunk max);
//   3. block_refine_kernel decides per row: the cut is certain when the k-th
//      tracked value beats max(the (k+1)-th, U) by more than 2E; otherwise, if
//      U is below the cut, every tracked candidate within 2E of the k-th is
//      re-scored exactly (fp64 dot of the fp32 means) — anything else is at
//      most U, so at least k blocks beat it exactly; rows whose untracked
//      values reach the cut (massive near-ties: zeros, repeated blocks) go to
//      block_rescan_kernel, a CTA per row re-scoring every causal block.
// The chosen set equals the exact top-k of the fp32 pooled logits (fp64
// products), which is the reference's selection up to its own fp32 rounding.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
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

// pooled block layout of one side (Q or K) in the workspace:
//   f16  [G, nb, 128] half   normalised copy (TMA operand)
//   mean [G, nb, 128] float  exact fp32 means (refine)
//   aux  [G, nb]      float2 (|x~|_2 of the normalised copy, 2^e: the block's own scale for q, the head's for k)
//   head [G]          int2   k only: (max biased exponent, max |y~|_2 as float bits)
static size_t al256(size_t x) { return (x + 255) & ~size_t(255); }
size_t pool16_bytes(int groups, int nb) {
  const size_t gb = (size_t)groups * nb;
  return gb * 256 + gb * 512 + al256(gb * 8) + al256((size_t)groups * 8);
}
struct Pool16View {
  __half* f16;
  float* mean;
  float2* aux;
  int2* head;
};
static Pool16View pool16_view(void* base, int groups, int nb) {
  char* p = reinterpret_cast<char*>(base);
  const size_t gb = (size_t)groups * nb;
  return Pool16View{reinterpret_cast<__half*>(p), reinterpret_cast<float*>(p + gb * 256),
                    reinterpret_cast<float2*>(p + gb * 768), reinterpret_cast<int2*>(p + gb * 768 + al256(gb * 8))};
}
constexpr int kExpBias = 256;

// max of non-negative ints into base[2 g + comp] for the CTA's half-warps:
// the CTA's first two groups reduce in shared memory first (one global atomic
// each instead of one per block: thousands of same-address atomics per head
// serialise in L2).  Every thread of the CTA must call it.
__device__ __forceinline__ void cta_group_max(int* base, int comp, int g, int g0, bool on, int v) {
  __shared__ int sm[2];
  if (threadIdx.x < 2) sm[threadIdx.x] = 0;
  __syncthreads();
  if (on) {
    if (g - g0 < 2)
      atomicMax(&sm[g - g0], v);
    else
      atomicMax(base + 2 * g + comp, v);
  }
  __syncthreads();
  if (threadIdx.x < 2 && sm[threadIdx.x] > 0) atomicMax(base + 2 * (g0 + threadIdx.x) + comp, sm[threadIdx.x]);
}

// One half-warp per (group, block); lane l pools dims 8 (l % 16) .. + 7 over
// the block's rows in order (fp32), like block_pool_kernel.  Query side
// (head == nullptr): fp16 copy at the block's own scale.  Key side: only the
// mean and norm here; the head's largest exponent / norm go to head[g]
// (zeroed by the caller) and key_f16_kernel writes the fp16 copy.
__global__ void block_pool16_kernel(const __nv_bfloat16* __restrict__ x, int G, int n, int b, __half* f16,
                                    float* mean_out, float2* aux, int2* head, const int32_t* gate, int gate_val) {
  const int nb = (n + b - 1) / b;
  const long long gid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 4;
  const int hl = threadIdx.x & 15;
  const bool live = gid < (long long)G * nb;
  const int g = live ? (int)(gid / nb) : 0, blk = live ? (int)(gid % nb) : 0;
  const bool on = live && !(gate && gate[g] != gate_val);
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const int r0 = blk * b, r1 = min(n, r0 + b);
  if (on) {
    const uint4* src = reinterpret_cast<const uint4*>(x + ((long long)g * n + r0) * kHeadDim) + hl;
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
  }
  const float cntf = on ? (float)(r1 - r0) : 1.f;
  float mean[8], amax = 0.f;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    mean[u] = __fdiv_rn(acc[u], cntf);
    amax = fmaxf(amax, fabsf(mean[u]));
  }
#pragma unroll
  for (int o = 8; o > 0; o >>= 1)  // the half-warp's 16 lanes (xor < 16 stays inside)
    amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  // 2^-e * max in [2^13, 2^14); e clamped so 2^e stays a normal float
  int E = -1000;
  if (amax > 0.f) frexpf(amax, &E);  // amax in [2^(E-1), 2^E)
  const int ex = amax > 0.f ? max(E - 14, -120) : 0;
  // the norm of the normalised copy (its squares cannot underflow the way the
  // raw means' squares can: the bound E of the screens is taken from it)
  float ss = 0.f;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const float y = ldexpf(mean[u], -ex);
    ss = fmaf(y, y, ss);
  }
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const long long row = (long long)g * nb + blk;
  if (on) {
    float* mo = mean_out + row * kHeadDim + 8 * hl;
    *reinterpret_cast<float4*>(mo) = make_float4(mean[0], mean[1], mean[2], mean[3]);
    *reinterpret_cast<float4*>(mo + 4) = make_float4(mean[4], mean[5], mean[6], mean[7]);
  }
  if (head != nullptr) {  // key side: the head's exponent now, the fp16 copy and |y~| in key_f16_kernel
    const int g0 = (int)(((long long)blockIdx.x * blockDim.x >> 4) / nb);
    cta_group_max(reinterpret_cast<int*>(head), 0, g, g0, on && hl == 0 && amax > 0.f, E + kExpBias);
    return;
  }
  if (!on) return;
  __align__(16) __half h[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) h[u] = __float2half_rn(ldexpf(mean[u], -ex));
  *reinterpret_cast<uint4*>(f16 + row * kHeadDim + 8 * hl) = *reinterpret_cast<uint4*>(h);
  if (hl == 0) aux[row] = make_float2(sqrtf(ss), ldexpf(1.f, ex));  // (|x~|, 2^e)
}

// Key side, second pass: fp16 copy of every block at its kv head's common
// scale; head[g].y = max |y~| over the head (as float bits, zeroed by the caller).
__global__ void key_f16_kernel(int G, int nb, const float* __restrict__ mean, __half* f16, float2* aux,
                               int2* head) {
  const long long gid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 4;
  const int hl = threadIdx.x & 15;
  const bool live = gid < (long long)G * nb;
  const int g = live ? (int)(gid / nb) : 0;
  float ss = 0.f;
  if (live) {
    const int hx = head[g].x;
    const int ex = hx > 0 ? max(hx - kExpBias - 14, -120) : 0;
    const float4* mi = reinterpret_cast<const float4*>(mean + gid * kHeadDim + 8 * hl);
    const float4 m0 = __ldg(mi), m1 = __ldg(mi + 1);
    const float m[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
    __align__(16) __half h[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float y = ldexpf(m[u], -ex);
      h[u] = __float2half_rn(y);
      ss = fmaf(y, y, ss);
    }
    *reinterpret_cast<uint4*>(f16 + gid * kHeadDim + 8 * hl) = *reinterpret_cast<uint4*>(h);
    if (hl == 0) aux[gid].y = ldexpf(1.f, ex);
  }
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);  // xor < 16: inside the half-warp
  const float yn = sqrtf(ss);
  if (live && hl == 0) aux[gid].x = yn;  // |y~|
  const int g0 = (int)(((long long)blockIdx.x * blockDim.x >> 4) / nb);
  cta_group_max(reinterpret_cast<int*>(head), 1, g, g0, live && hl == 0, __float_as_int(yn));  // floats >= 0 order as ints
}

struct ScreenArgs {
  CUtensorMap tmap_q;  // q16 [HH, nb, 128] (2-byte elements), box {64, 128}
  CUtensorMap tmap_k;  // k16 [HK, nb, 128]
  const float2* qaux;  // [HH, nb] (|x~|, 2^e_q): the normalised copy's norm
  const float2* kaux;  // [HK, nb] (|y~|, 2^e_head)
  const int2* khead;   // [HK] (max biased exponent, max |y~| bits)
  int nb, heads, kv_heads, nqt, k_b;
  float* tv;           // [HH, nb, T] tracked chunk maxima (raw units), -inf padded
  float* t2;           // [HH, nb, T] each tracked chunk's second largest value
  int32_t* ti;         // [HH, nb, T] their key block ids
  float* terr;         // [HH, nb] bound E
  float* tu;           // [HH, nb] U: the largest value outside the tracked chunks
  const int32_t* gate;
  int gate_val;
};

constexpr int kScThreads = 192;
constexpr int kScRing = 4;
constexpr int kScSmemA = 0;                           // q16 tile: 2 x 16 KB (d halves)
constexpr int kScSmemB = 32768;                       // ring of 16 KB key chunks (d halves)
constexpr int kScSmemBar = kScSmemB + kScRing * 16384;
constexpr int kScSmemBytes = kScSmemBar + 256;
enum SBar { SB_A = 0, SB_KF0, SB_KE0 = SB_KF0 + kScRing, SB_SF0 = SB_KE0 + kScRing, SB_SF1, SB_SE0, SB_SE1, SB_NUM };

// kind::f16 with fp16 operands (a_format = b_format = F16 = 0)
__host__ __device__ constexpr uint32_t idesc_f16_f32(int M, int N) {
  return (1u << 4) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}

template <int T>
__global__ void __launch_bounds__(kScThreads, 2) block_screen_kernel(const __grid_constant__ ScreenArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if ((smem_u32(smem) & 1023u) != 0u) __trap();
  const int hh = blockIdx.x;
  if (a.gate && a.gate[hh] != a.gate_val) return;
  const int qt = a.nqt - 1 - blockIdx.y;  // heaviest query tiles first
  const int cnt = qt + 1;
  uint8_t* sA = smem + kScSmemA;
  uint8_t* sB = smem + kScSmemB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kScSmemBar);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + SB_NUM);
  const int warp = warp_id();
  const int bidx = hh / a.heads;
  const int hkv = bidx * a.kv_heads + (hh % a.heads) / (a.heads / a.kv_heads);

  if (threadIdx.x == 0) {
    mbar_init(&bars[SB_A], 1);
    for (int s = 0; s < kScRing; ++s) {
      mbar_init(&bars[SB_KF0 + s], 1);
      mbar_init(&bars[SB_KE0 + s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bars[SB_SF0 + s], 1);
      mbar_init(&bars[SB_SE0 + s], 128);
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
      mbar_arrive_expect_tx(&bars[SB_A], 32768);
      for (int c = 0; c < 2; ++c) tma_load_3d(sA + c * 16384, &a.tmap_q, &bars[SB_A], 64 * c, qt * kTile, hh);
      for (int j = 0; j < cnt; ++j)
        for (int c = 0; c < 2; ++c) {
          const int g = 2 * j + c, slot = g % kScRing;
          if (g >= kScRing) mbar_wait_backoff<256>(&bars[SB_KE0 + slot], ((g / kScRing) - 1) & 1);
          mbar_arrive_expect_tx(&bars[SB_KF0 + slot], 16384);
          tma_load_3d(sB + slot * 16384, &a.tmap_k, &bars[SB_KF0 + slot], 64 * c, j * kTile, hkv);
        }
    }
  } else if (warp == 5) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_f16_f32(128, 128);
      const uint32_t a_addr = smem_u32(sA);
      mbar_wait(&bars[SB_A], 0);
      for (int j = 0; j < cnt; ++j) {
        const int buf = j & 1;
        if (j >= 2) mbar_wait_backoff<128>(&bars[SB_SE0 + buf], ((j >> 1) - 1) & 1);
        for (int c = 0; c < 2; ++c) {
          const int g = 2 * j + c, slot = g % kScRing;
          mbar_wait_backoff<64>(&bars[SB_KF0 + slot], (g / kScRing) & 1);
          tc_fence_after();
          const uint32_t b_addr = smem_u32(sB + slot * 16384);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_ss(tbase + buf * 128, sdesc_sw128(a_addr + c * 16384 + kk * 32, 16, 1024),
                   sdesc_sw128(b_addr + kk * 32, 16, 1024), idesc, (c > 0 || kk > 0) ? 1u : 0u);
          mma_commit(&bars[SB_KE0 + slot]);
        }
        mma_commit(&bars[SB_SF0 + buf]);
      }
    }
  } else {
    const int t = threadIdx.x;  // 0..127: query block row of the tile
    const int gq = qt * kTile + t;
    const bool valid = gq < a.nb;
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    float bv[T], b2[T];  // tracked chunk maxima and each chunk's second largest value
    int bi[T];
#pragma unroll
    for (int q = 0; q < T; ++q) {
      bv[q] = -INFINITY;
      b2[q] = -INFINITY;
      bi[q] = -1;
    }
    float U = -INFINITY;  // every value outside the tracked chunks is <= U
    for (int j = 0; j < cnt; ++j) {
      const int buf = j & 1;
      const int g0 = j * kTile;
      const int lim = gq - g0;  // block-causal: key block g0 + c <= gq
      const bool diag = j == cnt - 1;  // the only tile with block-causal cuts
      mbar_wait(&bars[SB_SF0 + buf], (j >> 1) & 1);
      tc_fence_after();
      // 32 columns at a time (tcgen05.ld is warp-collective: every lane loads,
      // rows past nb are masked); the column index rides in the 7 low mantissa
      // bits, so the chunk's max tree also yields its argmax.  Chunk c + 1's
      // TMEM load is in flight while chunk c is processed; the S buffer is
      // released as soon as the last chunk is in registers.
      auto process = [&](const uint32_t (&s)[32], int c) {
        float x[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) x[u] = __uint_as_float((s[u] & ~127u) | (uint32_t)(32 * c + u));
        if (diag || !valid) {
#pragma unroll
          for (int u = 0; u < 32; ++u) x[u] = (valid && 32 * c + u <= lim) ? x[u] : -INFINITY;
        }
        // top-2 of the chunk: pairwise (max, min), then merges
        float h1[16], h2[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          h1[u] = fmaxf(x[2 * u], x[2 * u + 1]);
          h2[u] = fminf(x[2 * u], x[2 * u + 1]);
        }
#pragma unroll
        for (int w = 8; w > 0; w >>= 1) {
#pragma unroll
          for (int u = 0; u < w; ++u) {
            const float a1 = h1[u], b1 = h1[u + w];
            h1[u] = fmaxf(a1, b1);
            h2[u] = fmax3(fminf(a1, b1), h2[u], h2[u + w]);
          }
        }
        const float c1 = h1[0], c2 = h2[0];
        if (c1 > bv[T - 1]) {
          U = fmaxf(U, bv[T - 1]);  // the evicted chunk (its second value is below its max)
          int p = T - 1;
#pragma unroll
          for (int q = T - 1; q > 0; --q) {
            if (c1 > bv[q - 1]) {
              bv[q] = bv[q - 1];
              b2[q] = b2[q - 1];
              bi[q] = bi[q - 1];
              p = q - 1;
            }
          }
          const int id = g0 + (int)(__float_as_uint(c1) & 127u);
#pragma unroll
          for (int q = 0; q < T; ++q)
            if (q == p) {
              bv[q] = c1;
              b2[q] = c2;
              bi[q] = id;
            }
        } else {
          U = fmaxf(U, c1);
        }
      };
      uint32_t s0[32], s1[32];
      const uint32_t col = tbase + lane_off + buf * 128;
      tmem_ld32(col, s0);
      tmem_ld_wait();
      tmem_ld32(col + 32, s1);
      process(s0, 0);
      tmem_ld_wait();
      tmem_ld32(col + 64, s0);
      process(s1, 1);
      tmem_ld_wait();
      tmem_ld32(col + 96, s1);
      process(s0, 2);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&bars[SB_SE0 + buf]);
      process(s1, 3);
    }
    if (valid) {
      const float2 qa = a.qaux[(size_t)hh * a.nb + gq];
      const int2 kh = a.khead[hkv];
      const float xn = qa.x;                 // |x~|
      const float yn = __int_as_float(kh.y);  // |y~|max
      const float E = (ldexpf(1.f, -9) + ldexpf(1.f, -15)) * xn * yn + ldexpf(xn + yn, -21) + ldexpf(1.f, -40);
      const size_t r = (size_t)hh * a.nb + gq;
#pragma unroll
      for (int q = 0; q < T; ++q) {
        a.tv[r * T + q] = bv[q];
        a.t2[r * T + q] = b2[q];
        a.ti[r * T + q] = bi[q];
      }
      a.terr[r] = E * 1.0001f;
      a.tu[r] = U;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) tmem_dealloc(tbase, 256);
}

// ---------------------------------------------------------------- k_b = 1
// The auto search's Block(8, 1) needs only each row's argmax, so k_b = 1 runs
// the fp16 GEMM TWICE per CTA instead of tracking candidates in one pass:
//   pass A: every key tile's logits reduce to the row max M~ (a max tree: ~0.5
//           instructions per logit, far below the tensor time of the tile);
//   pass B: the same MMAs again (bit-identical values); every logit with
//           s~ >= M~ - 2E is a candidate (the exact argmax is one of them:
//           s >= M >= M~ - E and s~ >= s - E), appended per row (few: the
//           argmax and whatever lies within the fp16 error of it).
// A row with one candidate is decided at once; rows with 2..kTop1Cand go to
// block_top1_refine_kernel (exact fp64 dots of the fp32 means), rows with
// more to the CTA-per-row rescan (massive exact ties only).  A zero query block (or an all-zero key head) has all logits
// exactly 0 and takes block 0.  Two fp16 passes are 16 MMAs per 128 x 128
// tile against the split-bf16 GEMM's 24.
constexpr int kTop1Cand = 16;  // candidates kept per row (global slots; more go to the rescan)
__device__ __forceinline__ void write_block_row(int32_t* dst, int gq, const int (&sel)[8], int K, int stride);

struct Top1Args {
  CUtensorMap tmap_q;
  CUtensorMap tmap_k;
  const float2* qaux;
  const int2* khead;
  int nb, heads, kv_heads, nqt;
  int32_t* blk_idx;  // per head at hh * head_stride: [nb, 2]
  long long head_stride;
  int32_t* blk_row_off;  // per head at hh * row_stride: [nb + 1]
  int row_stride;
  int32_t* cand;    // [HH * nb, kTop1Cand] candidate slots
  int32_t* ccount;  // [HH * nb] candidates of the rows sent to the refine
  int* refine;      // [count, rows...]: 2..kTop1Cand candidates
  int* rescan;      // [count, rows...]: more than kTop1Cand
  const int32_t* gate;
  int gate_val;
};

__device__ __forceinline__ float max32(const float (&x)[32]) {
  float m[11];
#pragma unroll
  for (int i = 0; i < 10; ++i) m[i] = fmax3(x[3 * i], x[3 * i + 1], x[3 * i + 2]);
  m[10] = fmaxf(x[30], x[31]);
  const float a = fmax3(m[0], m[1], m[2]), b = fmax3(m[3], m[4], m[5]), c = fmax3(m[6], m[7], m[8]);
  return fmax3(fmax3(a, b, c), m[9], m[10]);
}


// The MMAs read the query operand from TMEM (copied once per CTA with
// tcgen05.cp) and only the key chunk from shared memory: an SS MMA reads both
// operands (8 KB per M=128 N=128 K=16 MMA = the 128 B/clk shared-memory port
// by itself), which with the TMA fills left the tensor pipe ~60% busy.  TMEM
// (256 columns per CTA, two CTAs per SM): q [0, 64), three 64-column S
// buffers (one per 64-key chunk, N = 64 runs at the full rate from TMEM).
constexpr int kT1ColS = 64;
constexpr int kT1Threads = 320;  // 8 epilogue warps (two per TMEM lane quarter), producer, MMA issuer
enum T1Bar { T1_A = 0, T1_KF0, T1_KE0 = T1_KF0 + kScRing, T1_SF0 = T1_KE0 + kScRing, T1_SE0 = T1_SF0 + 3, T1_NUM = T1_SE0 + 3 };

// The two epilogue warps of a lane quarter take alternate 64-key chunks (warp
// set p = warp / 4 takes chunks u = p, p + 2, ...), so each has two MMA chunk
// times to finish one; they meet twice, through shared memory: the row max
// after pass A, and the candidate counts at the end (set p appends into slots
// [8 p, 8 p + 8) of the row's kTop1Cand).
__global__ void __launch_bounds__(kT1Threads, 2) block_top1_kernel(const __grid_constant__ Top1Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if ((smem_u32(smem) & 1023u) != 0u) __trap();
  const int hh = blockIdx.x;
  if (a.gate && a.gate[hh] != a.gate_val) return;
  const int qt = a.nqt - 1 - blockIdx.y;  // heaviest query tiles first
  const int cnt = qt + 1;                 // causal key tiles per pass
  uint8_t* sA = smem + kScSmemA;
  uint8_t* sB = smem + kScSmemB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kScSmemBar);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + T1_NUM);
  __shared__ float sM[128];
  __shared__ int sN[128];
  const int warp = warp_id();
  const int bidx = hh / a.heads;
  const int hkv = bidx * a.kv_heads + (hh % a.heads) / (a.heads / a.kv_heads);

  if (threadIdx.x == 0) {
    mbar_init(&bars[T1_A], 1);
    for (int s = 0; s < kScRing; ++s) {
      mbar_init(&bars[T1_KF0 + s], 1);
      mbar_init(&bars[T1_KE0 + s], 1);
    }
    for (int s = 0; s < 3; ++s) {
      mbar_init(&bars[T1_SF0 + s], 1);
      mbar_init(&bars[T1_SE0 + s], 128);
    }
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc(tmem_holder, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_holder;

  if (warp == 8) {
    if (elect_one()) {
      mbar_arrive_expect_tx(&bars[T1_A], 32768);
      for (int c = 0; c < 2; ++c) tma_load_3d(sA + c * 16384, &a.tmap_q, &bars[T1_A], 64 * c, qt * kTile, hh);
      // the key tiles' d-halves, once per pass (pass B's are L2 hits: nb x 256 B per kv head)
      for (int j = 0; j < 2 * cnt; ++j) {
        const int jt = j < cnt ? j : j - cnt;
        for (int c = 0; c < 2; ++c) {
          const int g = 2 * j + c, slot = g % kScRing;
          if (g >= kScRing) mbar_wait_backoff<256>(&bars[T1_KE0 + slot], ((g / kScRing) - 1) & 1);
          mbar_arrive_expect_tx(&bars[T1_KF0 + slot], 16384);
          tma_load_3d(sB + slot * 16384, &a.tmap_k, &bars[T1_KF0 + slot], 64 * c, jt * kTile, hkv);
        }
      }
    }
  } else if (warp == 9) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_f16_f32(128, 64);
      const uint32_t a_addr = smem_u32(sA);
      const uint32_t b_addr = smem_u32(sB);
      mbar_wait(&bars[T1_A], 0);
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        utccp_128x256b(tbase + kk * 8, sdesc_sw128(a_addr + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024));
      for (int j = 0; j < 2 * cnt; ++j) {
        const int s0 = (2 * j) % kScRing, s1 = (2 * j + 1) % kScRing;
        mbar_wait(&bars[T1_KF0 + s0], ((2 * j) / kScRing) & 1);
        mbar_wait(&bars[T1_KF0 + s1], ((2 * j + 1) / kScRing) & 1);
        for (int h = 0; h < 2; ++h) {  // 64-key chunk h of the tile (keys 64 h .. 64 h + 63: +8 KB in SW128)
          const int u = 2 * j + h, buf = u % 3;
          if (u >= 3) mbar_wait(&bars[T1_SE0 + buf], ((u / 3) - 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const int slot = (kk >> 2) ? s1 : s0;
            mma_ts(tbase + kT1ColS + 64 * buf, tbase + kk * 8,
                   sdesc_sw128(b_addr + slot * 16384 + h * 8192 + (kk & 3) * 32, 16, 1024), idesc, kk > 0 ? 1u : 0u);
          }
          mma_commit(&bars[T1_SF0 + buf]);
        }
        mma_commit(&bars[T1_KE0 + s0]);
        mma_commit(&bars[T1_KE0 + s1]);
      }
    }
  } else {
    const int t = threadIdx.x & 127;  // query block row of the tile (TMEM lane)
    const int p = warp >> 2;          // warp set: chunks u = p, p + 2, ...
    const int gq = qt * kTile + t;
    const bool valid = gq < a.nb;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const size_t r = (size_t)hh * a.nb + (valid ? gq : 0);
    float M = -INFINITY;     // pass A: max over this set's chunks of the row (raw units)
    float theta = INFINITY;  // pass B: candidate threshold M~ - 2E
    int nc = 0;
    int32_t* cand = a.cand + r * kTop1Cand + 8 * p;  // this set's 8 slots (written only for candidates)
    for (int u = p; u < 4 * cnt; u += 2) {  // 64-key chunks: pass A, then pass B
      const int j = u >> 1;
      const bool pb = j >= cnt;
      const int jt = pb ? j - cnt : j;
      const int buf = u % 3;
      const int g0 = jt * kTile + (u & 1) * 64;
      const int lim = gq - g0;          // block-causal: key block g0 + c <= gq
      const bool diag = jt == cnt - 1;  // the only tile with block-causal cuts
      if (u == 2 * cnt + p) {  // first pass-B chunk: the row max over both sets
        if (p == 1) sM[t] = M;
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (p == 0) sM[t] = fmaxf(M, sM[t]);
        asm volatile("bar.sync 1, 256;" ::: "memory");
        M = sM[t];
        if (valid) {
          // E bounds |s~ - s| in raw units (block_screen_kernel's bound)
          const float xn = a.qaux[r].x, yn = __int_as_float(a.khead[hkv].y);  // |x~|, |y~|max
          const float E = (ldexpf(1.f, -9) + ldexpf(1.f, -15)) * xn * yn + ldexpf(xn + yn, -21) + ldexpf(1.f, -40);
          theta = M - 2.0002f * E;
        }
      }
      mbar_wait(&bars[T1_SF0 + buf], (u / 3) & 1);
      tc_fence_after();
      // both halves in flight, then the buffer goes straight back to the MMA warp
      uint32_t s0[32], s1[32];
      const uint32_t col = tbase + lane_off + kT1ColS + 64 * buf;
      tmem_ld32(col, s0);
      tmem_ld32(col + 32, s1);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&bars[T1_SE0 + buf]);
      auto process = [&](const uint32_t (&s)[32], int c) {
        float x[32];
#pragma unroll
        for (int v = 0; v < 32; ++v) x[v] = __uint_as_float(s[v]);
        if (diag || !valid) {
#pragma unroll
          for (int v = 0; v < 32; ++v) x[v] = (valid && 32 * c + v <= lim) ? x[v] : -INFINITY;
        }
        // maxima of the four 8-column groups, then of the 32
        float gm[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          gm[q] = fmax3(fmax3(x[8 * q], x[8 * q + 1], x[8 * q + 2]), fmax3(x[8 * q + 3], x[8 * q + 4], x[8 * q + 5]),
                        fmaxf(x[8 * q + 6], x[8 * q + 7]));
        const float m = fmaxf(fmax3(gm[0], gm[1], gm[2]), gm[3]);
        if (!pb) {
          M = fmaxf(M, m);
        } else if (__any_sync(0xffffffffu, m >= theta)) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (gm[q] >= theta) {  // rare per lane: scan the group
#pragma unroll
              for (int v = 0; v < 8; ++v) {
                if (x[8 * q + v] >= theta) {
                  if (nc < 8) cand[nc] = g0 + 32 * c + 8 * q + v;
                  ++nc;
                }
              }
            }
          }
        }
      };
      process(s0, 0);
      process(s1, 1);
    }
    // both sets' counts meet; set 0 finishes the row
    if (p == 1) sN[t] = nc;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    if (p == 0 && valid) {
      const int n1 = sN[t];
      int32_t* c0 = a.cand + r * kTop1Cand;
      int32_t* ro = a.blk_row_off + (size_t)hh * a.row_stride;
      ro[gq] = (int32_t)(hh * a.head_stride + (long long)gq * 2);
      if (gq == a.nb - 1) ro[a.nb] = (int32_t)(hh * a.head_stride + (long long)a.nb * 2);
      // a zero query block (or an all-zero key head) makes every logit exactly
      // 0: the lowest id wins, like the reference's stable top-k
      const bool zero = a.qaux[r].x == 0.f || a.khead[hkv].y == 0;
      const int tot = nc + n1;
      if (zero || tot == 1) {
        int sel[8] = {zero ? 0 : (nc == 1 ? c0[0] : c0[8]), -1, -1, -1, -1, -1, -1, -1};
        write_block_row(a.blk_idx + (size_t)hh * a.head_stride + (size_t)gq * 2, gq, sel, 1, 2);
      } else if (nc <= 8 && n1 <= 8) {
        for (int c = 0; c < n1; ++c) c0[nc + c] = c0[8 + c];  // pack set 1's slots after set 0's
        a.ccount[r] = tot;
        a.refine[1 + atomicAdd(a.refine, 1)] = (int)r;
      } else {
        a.rescan[1 + atomicAdd(a.rescan, 1)] = (int)r;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) tmem_dealloc(tbase, 256);
}

__device__ __forceinline__ double warp_sum_d(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// chosen ids + forced diagonal block, ascending, INT32_MAX padded (K <= 8)
__device__ __forceinline__ void write_block_row(int32_t* dst, int gq, const int (&sel)[8], int K, int stride) {
  int ids[9];
  int m = 0;
  bool has_diag = false;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    if (q < K && sel[q] >= 0) {
      ids[m++] = sel[q];
      has_diag |= sel[q] == gq;
    }
  }
  if (!has_diag) ids[m++] = gq;
  for (int x = 1; x < m; ++x) {
    const int y0 = ids[x];
    int y = x - 1;
    while (y >= 0 && ids[y] > y0) {
      ids[y + 1] = ids[y];
      --y;
    }
    ids[y + 1] = y0;
  }
  for (int q = 0; q < stride; ++q) dst[q] = q < m ? ids[q] : INT_MAX;
}

// running top-K by (exact value desc, id asc) in registers (K <= 8)
struct TopK8 {
  double v[8];
  int i[8];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      v[q] = -INFINITY;
      i[q] = INT_MAX;
    }
  }
  __device__ __forceinline__ void offer(double x, int g, int K) {
    int p = 0;  // entries ranked ahead of (x, g)
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < K && (v[q] > x || (v[q] == x && i[q] < g))) p = q + 1;
    if (p >= K) return;
#pragma unroll
    for (int q = 7; q > 0; --q)
      if (q > p && q < K) {
        v[q] = v[q - 1];
        i[q] = i[q - 1];
      }
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q == p) {
        v[q] = x;
        i[q] = g;
      }
  }
};

// fp64 dot of a query row staged in shared memory (32 float4) with one key row
__device__ __forceinline__ double dot_row(const float4* sq, const float4* kr) {
  double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
#pragma unroll 8
  for (int c = 0; c < 32; ++c) {
    const float4 kx = __ldg(kr + c);
    const float4 qx = sq[c];
    d0 = fma((double)qx.x, (double)kx.x, d0);
    d1 = fma((double)qx.y, (double)kx.y, d1);
    d2 = fma((double)qx.z, (double)kx.z, d2);
    d3 = fma((double)qx.w, (double)kx.w, d3);
  }
  return (d0 + d1) + (d2 + d3);
}

// K times, the best head over the warp's lane-local lists (value desc, id asc)
// is popped into `out` (warp-uniform); ids are unique, so one lane pops
__device__ __forceinline__ void warp_merge_topk(TopK8& mine, TopK8& out, int K) {
  out.init();
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    if (t >= K) break;
    double wv = mine.v[0];
    int wi = mine.i[0];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, wv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, wi, o);
      if (ov > wv || (ov == wv && oi < wi)) {
        wv = ov;
        wi = oi;
      }
    }
    out.v[t] = wv;
    out.i[t] = wi;
    if (mine.i[0] == wi && wi != INT_MAX) {
#pragma unroll
      for (int q = 0; q < 7; ++q) {
        mine.v[q] = mine.v[q + 1];
        mine.i[q] = mine.i[q + 1];
      }
      mine.v[7] = -INFINITY;
      mine.i[7] = INT_MAX;
    }
  }
}

// One warp per 32 rows of a head (lane = row).  Every value of a row lies in a
// tracked chunk (its max v[q] is tracked, the rest are <= its second value
// s2[q]) or is <= U.  Certain rows (the k-th tracked max beats the (k+1)-th,
// every s2 and U by > 2E) take the tracked top-k; if only U is below the cut
// the candidates are the tracked maxima within 2E plus every block of the
// tracked chunks whose second value is within 2E, re-scored exactly (fp64 dots
// of the fp32 means: a chunk's 32 blocks one per lane); rows where U reaches
// the cut are queued for block_rescan_kernel.
template <int T>
__global__ void __launch_bounds__(256) block_refine_kernel(
    const float* __restrict__ tv, const float* __restrict__ t2, const int32_t* __restrict__ ti,
    const float* __restrict__ terr, const float* __restrict__ tu, const float* __restrict__ qmean,
    const float* __restrict__ kmean, int hh_total, int heads, int kv_heads, int nb, int k_b, int32_t* blk_idx,
    long long head_stride, int* rescan, const int32_t* gate, int gate_val) {
  __shared__ float4 sqw[8][32];  // per warp: the query row being re-scored
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long long wid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int wpr = (nb + 31) / 32;  // warps per head
  if (wid >= (long long)hh_total * wpr) return;
  const int hh = (int)(wid / wpr);
  if (gate && gate[hh] != gate_val) return;
  const int gq = (int)(wid % wpr) * 32 + lane;
  const bool valid = gq < nb;
  const int hkv = (hh / heads) * kv_heads + (hh % heads) / (heads / kv_heads);
  const size_t r = (size_t)hh * nb + (valid ? gq : 0);
  float v[T], v2[T];
  int id[T];
#pragma unroll
  for (int q = 0; q < T; ++q) {
    v[q] = valid ? tv[r * T + q] : -INFINITY;
    v2[q] = valid ? t2[r * T + q] : -INFINITY;
    id[q] = valid ? ti[r * T + q] : -1;
  }
  const float E2 = valid ? 2.f * terr[r] : 0.f;
  const float U = valid ? tu[r] : -INFINITY;
  const int K = min(k_b, gq + 1);
  int sel[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) sel[q] = q < K ? (K == gq + 1 ? q : (q < T ? id[q] : -1)) : -1;  // K == gq + 1: all
  // 0 = certain, 1 = re-score candidates, 2 = re-score the whole row
  int mode = 0;
  float cut = -INFINITY;
  if (valid && K < gq + 1) {  // more causal blocks than K: a cut to decide
    const float vk = K - 1 < T ? v[K - 1] : -INFINITY;
    float nxt = fmaxf(K < T ? v[K] : -INFINITY, U);
#pragma unroll
    for (int q = 0; q < T; ++q) nxt = fmaxf(nxt, v2[q]);
    if (vk == -INFINITY) {
      mode = 2;
    } else if (!(vk - nxt > E2)) {
      cut = vk - E2;
      mode = U >= cut ? 2 : 1;
    }
  }
  if (mode == 2) {
    const int slot = atomicAdd(rescan, 1);
    rescan[1 + slot] = (int)r;
  }
  float4* sq = sqw[wib];
  uint32_t todo = __ballot_sync(0xffffffffu, mode == 1);
  while (todo) {
    const int src = __ffs(todo) - 1;
    todo &= todo - 1;
    const int rgq = (int)(wid % wpr) * 32 + src;
    const int rK = __shfl_sync(0xffffffffu, K, src);
    const float rcut = __shfl_sync(0xffffffffu, cut, src);
    __syncwarp();
    sq[lane] = __ldg(reinterpret_cast<const float4*>(qmean + ((size_t)hh * nb + rgq) * kHeadDim) + lane);
    __syncwarp();
    const float4* kbase = reinterpret_cast<const float4*>(kmean + (size_t)hkv * nb * kHeadDim);
    TopK8 mine;
    mine.init();
    uint32_t whole = 0u;  // tracked chunks re-scored block by block
#pragma unroll
    for (int q = 0; q < T; ++q) {
      const float c2 = __shfl_sync(0xffffffffu, v2[q], src);
      const int cg = __shfl_sync(0xffffffffu, id[q], src);
      if (cg >= 0 && c2 >= rcut) {  // warp-uniform: the chunk's 32 blocks, one per lane
        whole |= 1u << q;
        const int g = (cg & ~31) + lane;
        if (g <= rgq) mine.offer(dot_row(sq, kbase + (size_t)g * 32), g, rK);
      }
    }
    // tracked maxima within the cut whose chunk was not re-scored whole: lane q takes candidate q
    int mycand = -1;
#pragma unroll
    for (int q = 0; q < T; ++q) {
      const float cv = __shfl_sync(0xffffffffu, v[q], src);
      const int cg = __shfl_sync(0xffffffffu, id[q], src);
      if (lane == q && cg >= 0 && cv >= rcut && !(whole & (1u << q))) mycand = cg;
    }
    if (mycand >= 0) mine.offer(dot_row(sq, kbase + (size_t)mycand * 32), mycand, rK);
    TopK8 best;
    warp_merge_topk(mine, best, rK);
    if (lane == src) {
#pragma unroll
      for (int q = 0; q < 8; ++q) sel[q] = q < rK ? best.i[q] : -1;
    }
  }
  if (!valid || mode == 2) return;
  write_block_row(blk_idx + (size_t)hh * head_stride + (size_t)gq * (k_b + 1), gq, sel, K, k_b + 1);
}

// Rows queued by the refine (list[0] = count, then hh * nb + gq): a CTA per row
// re-scores every causal key block exactly.  Thread t takes blocks t, t + 256,
// ...: a full 128-dim fp64 dot per block (the query row is read from shared
// memory as a broadcast, each thread's key rows stream through L1), eight
// blocks' loads in flight per thread; per-thread top-k lists merge through
// warp shuffles and then across the eight warps.
constexpr int kRescanThreads = 256;
__device__ __forceinline__ void rescan_rows(const int* __restrict__ list, const float* __restrict__ qmean,
                                            const float* __restrict__ kmean, int heads, int kv_heads, int nb,
                                            int k_b, int32_t* blk_idx, long long head_stride) {
  __shared__ float4 sq[32];
  __shared__ double sv[8][8];
  __shared__ int si[8][8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cnt = list[0];
  for (int it = blockIdx.x; it < cnt; it += gridDim.x) {
    const int r = list[1 + it];
    const int hh = r / nb, gq = r % nb;
    const int hkv = (hh / heads) * kv_heads + (hh % heads) / (heads / kv_heads);
    const int K = min(k_b, gq + 1);
    if (threadIdx.x < 32) sq[threadIdx.x] = __ldg(reinterpret_cast<const float4*>(qmean + (size_t)r * kHeadDim) + threadIdx.x);
    __syncthreads();
    const float4* kbase = reinterpret_cast<const float4*>(kmean + (size_t)hkv * nb * kHeadDim);
    TopK8 best;
    best.init();
    for (int g = threadIdx.x; g <= gq; g += kRescanThreads) best.offer(dot_row(sq, kbase + (size_t)g * 32), g, K);
    TopK8 wl;
    warp_merge_topk(best, wl, K);
    if (lane == 0) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        sv[warp][q] = wl.v[q];
        si[warp][q] = wl.i[q];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      TopK8 all;
      all.init();
      for (int w = 0; w < 8; ++w)
        for (int q = 0; q < K; ++q)
          if (si[w][q] != INT_MAX) all.offer(sv[w][q], si[w][q], K);
      int sel[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) sel[q] = q < K ? all.i[q] : -1;
      write_block_row(blk_idx + (size_t)hh * head_stride + (size_t)gq * (k_b + 1), gq, sel, K, k_b + 1);
    }
    __syncthreads();
  }
}
__global__ void __launch_bounds__(kRescanThreads) block_rescan_kernel(
    const int* __restrict__ list, const float* __restrict__ qmean, const float* __restrict__ kmean, int heads,
    int kv_heads, int nb, int k_b, int32_t* blk_idx, long long head_stride) {
  rescan_rows(list, qmean, kmean, heads, kv_heads, nb, k_b, blk_idx, head_stride);
}

// k_b = 1 rows with 2..kTop1Cand candidates: a warp per row, lane l holds
// dims 4l..4l+3 of the query mean and of each candidate's key mean; fp64
// products summed across the warp and taken from lane 0, so every lane
// compares the same values; the largest exact logit wins, ties to the lower
// id.  Then the CTAs re-score the rescan rows (rescan_rows, k_b = 1).
__global__ void __launch_bounds__(kRescanThreads) block_top1_refine_kernel(
    const int* __restrict__ refine, const int32_t* __restrict__ cand, const int32_t* __restrict__ ccount,
    const int* __restrict__ rescan, const float* __restrict__ qmean, const float* __restrict__ kmean, int heads,
    int kv_heads, int nb, int32_t* blk_idx, long long head_stride) {
  const int lane = threadIdx.x & 31;
  const int nwarps = gridDim.x * (kRescanThreads / 32);
  const int cnt = refine[0];
  for (int it = (int)((blockIdx.x * kRescanThreads + threadIdx.x) >> 5); it < cnt; it += nwarps) {
    const int r = refine[1 + it];
    const int hh = r / nb, gq = r % nb;
    const int hkv = (hh / heads) * kv_heads + (hh % heads) / (heads / kv_heads);
    const float4 qx = __ldg(reinterpret_cast<const float4*>(qmean + (size_t)r * kHeadDim) + lane);
    const int nc = ccount[r];
    double best = -INFINITY;
    int bi = INT_MAX;
    for (int c = 0; c < nc; ++c) {
      const int g = cand[(size_t)r * kTop1Cand + c];
      const float4 kx = __ldg(reinterpret_cast<const float4*>(kmean + ((size_t)hkv * nb + g) * kHeadDim) + lane);
      double d = (double)qx.x * (double)kx.x;
      d = fma((double)qx.y, (double)kx.y, d);
      d = fma((double)qx.z, (double)kx.z, d);
      d = fma((double)qx.w, (double)kx.w, d);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
      d = __shfl_sync(0xffffffffu, d, 0);
      if (d > best || (d == best && g < bi)) {
        best = d;
        bi = g;
      }
    }
    if (lane == 0) {
      int sel[8] = {bi, -1, -1, -1, -1, -1, -1, -1};
      write_block_row(blk_idx + (size_t)hh * head_stride + (size_t)gq * 2, gq, sel, 1, 2);
    }
  }
  rescan_rows(rescan, qmean, kmean, heads, kv_heads, nb, 1, blk_idx, head_stride);
}


int launch_block_pool16(int groups, int n, int b, const void* x, void* pooled, bool key_side, const int32_t* gate,
                        int gate_val, cudaStream_t st) {
  if (groups < 1 || n < 1) return fail(SA_ERR_DIMENSION, "bad pool shape");
  if (b < 1 || b > n) return fail(SA_ERR_PATTERN_PARAM, "b must be in [1, %d], got %d", n, b);
  const int nb = (n + b - 1) / b;
  Pool16View v = pool16_view(pooled, groups, nb);
  const long long items = (long long)groups * nb;
  const unsigned grid = (unsigned)((items * 16 + 255) / 256);
  if (key_side) cudaMemsetAsync(v.head, 0, (size_t)groups * sizeof(int2), st);
  block_pool16_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(x), groups, n, b, v.f16, v.mean,
                                            v.aux, key_side ? v.head : nullptr, gate, gate_val);
  int rc;
  if ((rc = check_launch("block_pool16_kernel"))) return rc;
  if (!key_side) return SA_OK;
  key_f16_kernel<<<grid, 256, 0, st>>>(groups, nb, v.mean, v.f16, v.aux, v.head);
  return check_launch("key_f16_kernel");
}

// tracked candidates per row: k_b + 3, rounded to the kernel instantiations
// (k_b = 1: the top-1 path's candidate slots, kTop1Cand per row, in the tv region)
static int screen_T(int k_b) { return k_b <= 1 ? kTop1Cand : k_b == 2 ? 5 : k_b <= 4 ? 7 : 11; }

size_t block_screen_ws(int nb, int k_b, int hh_total) {
  const size_t rows = (size_t)hh_total * nb;
  const size_t T = (size_t)screen_T(k_b);
  return al256(rows * T * 4) * 3 + al256(rows * 4) * 2 + al256((rows + 1) * 4) + 256;
}

template <int T>
static int run_screen(const ScreenArgs& a, int hh_total, int nqt, cudaStream_t st) {
  static std::atomic<uint64_t> attr_done{0};
  once_per_device(attr_done, [] {
    cudaFuncSetAttribute(block_screen_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, kScSmemBytes);
  });
  block_screen_kernel<T><<<dim3(hh_total, nqt), kScThreads, kScSmemBytes, st>>>(a);
  return check_launch("block_screen_kernel");
}

template <int T>
static int run_refine(const ScreenArgs& a, const float* qmean, const float* kmean, int hh_total, int32_t* blk_idx,
                      long long head_stride, int* rescan, cudaStream_t st) {
  const long long warps = (long long)hh_total * ((a.nb + 31) / 32);
  block_refine_kernel<T><<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(
      a.tv, a.t2, a.ti, a.terr, a.tu, qmean, kmean, hh_total, a.heads, a.kv_heads, a.nb, a.k_b, blk_idx, head_stride,
      rescan, a.gate, a.gate_val);
  int rc;
  if ((rc = check_launch("block_refine_kernel"))) return rc;
  block_rescan_kernel<<<2 * device_sm_count(), kRescanThreads, 0, st>>>(rescan, qmean, kmean, a.heads, a.kv_heads,
                                                                        a.nb, a.k_b, blk_idx, head_stride);
  return check_launch("block_rescan_kernel");
}

// Pooled q (per head) and k (per kv head) from launch_block_pool16 -> fixed-stride
// block rows (k_b <= 8) and their row offsets.
int launch_block_screen(int batch, int heads, int kv_heads, int n, int b, int k_b, const void* qpool,
                        const void* kpool, int32_t* blk_idx, long long head_stride, int32_t* blk_row_off,
                        int row_stride, const int32_t* gate, int gate_val, void* ws, size_t ws_bytes,
                        cudaStream_t st) {
  if (batch < 1 || heads < 1 || kv_heads < 1 || heads % kv_heads)
    return fail(SA_ERR_DIMENSION, "bad head layout");
  if (b < 1 || b > n) return fail(SA_ERR_PATTERN_PARAM, "b must be in [1, %d], got %d", n, b);
  const int nb = (n + b - 1) / b;
  if (k_b < 1 || k_b > nb) return fail(SA_ERR_PATTERN_PARAM, "k_b must be in [1, %d], got %d", nb, k_b);
  if (k_b > 8) return fail(SA_ERR_DIMENSION, "block screen handles k_b <= 8");
  if (row_stride < nb + 1 || head_stride < (long long)nb * (k_b + 1))
    return fail(SA_ERR_DIMENSION, "block index strides too small");
  const int hh_total = batch * heads, hk_total = batch * kv_heads;
  if (!ws || ws_bytes < block_screen_ws(nb, k_b, hh_total))
    return fail(SA_ERR_DIMENSION, "block screen workspace too small");
  Pool16View qv = pool16_view(const_cast<void*>(qpool), hh_total, nb);
  Pool16View kv = pool16_view(const_cast<void*>(kpool), hk_total, nb);
  ScreenArgs a;
  memset(&a, 0, sizeof(a));
  int rc;
  if ((rc = make_tmap_3d_bf16(&a.tmap_q, qv.f16, kHeadDim, nb, hh_total, kTile))) return rc;
  if ((rc = make_tmap_3d_bf16(&a.tmap_k, kv.f16, kHeadDim, nb, hk_total, kTile))) return rc;
  a.qaux = qv.aux;
  a.kaux = kv.aux;
  a.khead = kv.head;
  a.nb = nb;
  a.heads = heads;
  a.kv_heads = kv_heads;
  a.nqt = (nb + kTile - 1) / kTile;
  a.k_b = k_b;
  const size_t rows = (size_t)hh_total * nb;
  const size_t T = (size_t)screen_T(k_b);
  char* p = reinterpret_cast<char*>(ws);
  a.tv = reinterpret_cast<float*>(p);
  p += al256(rows * T * 4);
  a.ti = reinterpret_cast<int32_t*>(p);
  p += al256(rows * T * 4);
  a.t2 = reinterpret_cast<float*>(p);
  p += al256(rows * T * 4);
  a.terr = reinterpret_cast<float*>(p);
  p += al256(rows * 4);
  a.tu = reinterpret_cast<float*>(p);
  p += al256(rows * 4);
  int* rescan = reinterpret_cast<int*>(p);  // [count, rows...]
  a.gate = gate;
  a.gate_val = gate_val;
  if (k_b > 1 &&
      (rc = launch_fixed_row_off(blk_row_off, hh_total, nb, k_b + 1, row_stride, head_stride, gate, gate_val, st)))
    return rc;
  cudaMemsetAsync(rescan, 0, sizeof(int), st);
  switch (k_b) {
    case 1: {
      // two fp16 passes (block_top1_kernel); the tracked-maxima workspace holds
      // the candidate slots (tv), the refine list (ti) and counts (terr)
      Top1Args t;
      memset(&t, 0, sizeof(t));
      t.tmap_q = a.tmap_q;
      t.tmap_k = a.tmap_k;
      t.qaux = a.qaux;
      t.khead = a.khead;
      t.nb = nb;
      t.heads = heads;
      t.kv_heads = kv_heads;
      t.nqt = a.nqt;
      t.blk_idx = blk_idx;
      t.head_stride = head_stride;
      t.blk_row_off = blk_row_off;
      t.row_stride = row_stride;
      t.cand = reinterpret_cast<int32_t*>(a.tv);
      t.ccount = reinterpret_cast<int32_t*>(a.terr);
      t.refine = reinterpret_cast<int*>(a.ti);
      t.rescan = rescan;
      t.gate = gate;
      t.gate_val = gate_val;
      cudaMemsetAsync(t.refine, 0, sizeof(int), st);
      static std::atomic<uint64_t> attr_done{0};
      once_per_device(attr_done, [] {
        cudaFuncSetAttribute(block_top1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kScSmemBytes);
      });
      block_top1_kernel<<<dim3(hh_total, a.nqt), kT1Threads, kScSmemBytes, st>>>(t);
      if ((rc = check_launch("block_top1_kernel"))) return rc;
      block_top1_refine_kernel<<<16 * device_sm_count(), kRescanThreads, 0, st>>>(
          t.refine, t.cand, t.ccount, rescan, qv.mean, kv.mean, heads, kv_heads, nb, blk_idx, head_stride);
      return check_launch("block_top1_refine_kernel");
    }
    case 2:
      if ((rc = run_screen<5>(a, hh_total, a.nqt, st))) return rc;
      return run_refine<5>(a, qv.mean, kv.mean, hh_total, blk_idx, head_stride, rescan, st);
    case 3:
    case 4:
      if ((rc = run_screen<7>(a, hh_total, a.nqt, st))) return rc;
      return run_refine<7>(a, qv.mean, kv.mean, hh_total, blk_idx, head_stride, rescan, st);
    default:
      if ((rc = run_screen<11>(a, hh_total, a.nqt, st))) return rc;
      return run_refine<11>(a, qv.mean, kv.mean, hh_total, blk_idx, head_stride, rescan, st);
  }
}

}  // namespace sa

// Block-Cluster index straight from bf16 q / k (pool16 + fp16 passes + refine):
// sa_prefill's path for k_b <= 8 under SA_BLOCK_SCREEN=1.  Workspace:
// sa_block_index_workspace.
extern "C" size_t sa_block_index_workspace(int batch, int heads, int kv_heads, int n, int b, int k_b) {
  if (batch < 1 || heads < 1 || kv_heads < 1 || n < 1 || b < 1 || b > n || k_b < 1) return 0;
  const int nb = (n + b - 1) / b;
  return sa::pool16_bytes(batch * heads, nb) + sa::pool16_bytes(batch * kv_heads, nb) +
         sa::block_screen_ws(nb, k_b, batch * heads) + 1024;
}

extern "C" int sa_block_index_bf16(int batch, int heads, int kv_heads, int n, int b, int k_b, const void* q,
                                   const void* k, int32_t* blk_idx, int32_t* blk_row_off, void* ws,
                                   size_t ws_bytes, void* stream) {
  using namespace sa;
  if (batch < 1 || heads < 1 || kv_heads < 1 || n < 1 || heads % kv_heads)
    return fail(SA_ERR_DIMENSION, "bad head layout");
  if (b < 1 || b > n) return fail(SA_ERR_PATTERN_PARAM, "b must be in [1, %d], got %d", n, b);
  const int nb = (n + b - 1) / b;
  if (k_b < 1 || k_b > nb) return fail(SA_ERR_PATTERN_PARAM, "k_b must be in [1, %d], got %d", nb, k_b);
  if (k_b > 8) return fail(SA_ERR_DIMENSION, "sa_block_index_bf16 handles k_b <= 8 (use sa_block_select)");
  if (!q || !k || !blk_idx || !blk_row_off || !ws) return fail(SA_ERR_DIMENSION, "null pointer");
  if (ws_bytes < sa_block_index_workspace(batch, heads, kv_heads, n, b, k_b))
    return fail(SA_ERR_DIMENSION, "workspace too small");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  char* p = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(ws) + 1023) & ~uintptr_t(1023));
  void* qpool = p;
  p += pool16_bytes(batch * heads, nb);
  void* kpool = p;
  p += pool16_bytes(batch * kv_heads, nb);
  int rc;
  if ((rc = launch_block_pool16(batch * heads, n, b, q, qpool, false, nullptr, 0, st))) return rc;
  if ((rc = launch_block_pool16(batch * kv_heads, n, b, k, kpool, true, nullptr, 0, st))) return rc;
  return launch_block_screen(batch, heads, kv_heads, n, b, k_b, qpool, kpool, blk_idx, (long long)nb * (k_b + 1),
                             blk_row_off, nb + 1, nullptr, 0, p, block_screen_ws(nb, k_b, batch * heads), st);
}
