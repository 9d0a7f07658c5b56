// estimate_vs.cu — the vertical-slash pattern estimator on tcgen05.
//
// Reference: patterns.py:165-202 (_tail_weights, _column_scores,
// _diagonal_scores) and patterns.py:237-259 (build_vertical_slash_index).
// For each selected head, the last R (<= 64 per launch) query rows
// [r_lo, r_hi) are scored against every causal key:
//     w[i, j] = softmax_row(q_i . k_j * scale) over j <= i
//     col[j]  = sum_i w[i, j]            (column mass)
//     diag[o] = sum_i w[i, i - o]        (diagonal mass, o >= 0).
//
// One persistent kernel does the whole estimator.  A *unit* is up to four
// selected heads of one kv head (two 128-row slots: rows 0-63 of a slot are one
// head's tail, rows 64-127 the next head's), so every K tile staged in shared
// memory feeds four heads.  Row statistics need every key before any weight is
// final, so each unit runs two passes over its K:
//   pass 1 (S = Q K^T, rows on TMEM lanes): per (row, key chunk) online
//     (max, sum); the CTA finishing the last chunk of a 16-chunk group merges
//     the group, the one finishing the last group merges the groups into the
//     rows' log2-sum-exp (fixed merge order: deterministic) and releases the
//     unit's pass 2;
//   pass 2 (S^T = K Q^T, keys on TMEM lanes): w = exp2(s c - lse2[row]); each
//     key's column sum is a register sum; the diagonal sums go through a
//     32-row x 128-key shared-memory block read back along rotated rows (every
//     thread sums exactly one element per row for two diagonals, bank-conflict
//     free), and each (tile, head, diagonal) partial is added to the zeroed
//     output with one red.add — a diagonal touches at most two key tiles and
//     0 + a + b == 0 + b + a, so the result is deterministic.
// Schedule: units run in waves of W (W units' K fit in L2 together: 64 MB);
// within a wave each unit owns grid / W CTAs and each CTA one contiguous range
// of key tiles, which it streams for pass 1 and again (from L2) for pass 2, so
// K is read from HBM about once.  A CTA keeps its unit's Q in shared memory for
// both passes; 16 softmax warps (four groups of four, two per 128-row slot)
// hide the TMEM / shared-memory / MUFU latencies.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "api_common.h"
#include "internal.h"
#include "sa_types.h"
#include "sm100_common.cuh"

namespace sa {

constexpr int kVsSoftWarps = 16;
constexpr int kVsSoft = kVsSoftWarps * 32;       // 512 softmax threads
constexpr int kVsThreads = kVsSoft + 64;         // + warp 16 TMA producer, warp 17 MMA issuer
constexpr int kVsKSlots = 2;
constexpr int kVsGroup = 16;                     // pass-1 chunks merged per first-level group
constexpr int kVsMaxCta = 16 * kVsGroup;         // CTAs per unit (two-level merge)
constexpr size_t kVsWaveBytes = 64ull << 20;     // K bytes of one wave (L2-resident between passes)
// shared memory: Q [64 KB] | K [2 slots][32 KB] | D [16 warps][16 rows][kDw] f32 (skewed
// diagonal blocks) | C2 [4 groups][191 diagonals][9] f32 | misc (barriers, flags, -lse2, merge exchange)
constexpr int kDw = 50;                          // D row stride: conflict-free skewed writes and half-column reads
constexpr int kC2Floats = 191 * 9 + 1;
constexpr int kVsOffK = 65536;
constexpr int kVsOffD = kVsOffK + kVsKSlots * 32768;
constexpr int kVsOffC = kVsOffD + kVsSoftWarps * 16 * kDw * 4;
constexpr int kVsOffMisc = kVsOffC + ((4 * kC2Floats * 4 + 1023) & ~1023);
constexpr int kVsOffNl = kVsOffMisc + 256;       // [4 groups][64] -lse2 of the group's rows
constexpr int kVsOffX = kVsOffNl + 1024;         // [256] float2 merge exchange
constexpr int kVsSmemBytes = kVsOffX + 2048 + 1024;

enum VBar {
  V_QF = 0,    // Q loaded
  V_QE = 1,    // MMAs of a wave done with Q
  V_KF = 2,    // [3] K slot loaded
  V_KE = 5,    // [3] MMAs done with a K slot
  V_SF = 8,    // [slot * 2 + buf] S ready
  V_SE = 12,   // [slot * 2 + buf] S consumed (256 arrivals: two groups)
  V_NUM = 16
};

struct TailArgs {
  CUtensorMap tmap_q;  // [HH, n, 128], box {64, 64 rows}
  CUtensorMap tmap_k;  // [HK, n, 128], box {64, 128 rows}
  int n, heads, kv_heads, hh_total;
  int r_lo, r_hi;      // scored rows, r_hi - r_lo <= 64
  int qrow0;           // global row of Q box row 0 (r_hi - 64, may be negative)
  int nkt;             // key tiles with a causal key: ceil(r_hi / 128)
  int wave_units;      // most units per wave
  int min_tiles;       // fewest key tiles per CTA (small launches leave SMs to the concurrent block chain)
  float scale_log2;
  float2* stats;       // [U, kVsMaxCta, 2 key halves, 256] per-(chunk, row) (max2, sum)
  float2* stats2;      // [U, 16, 256] per-(group, row)
  float* lse2;         // [U, 256] log2-sum-exp per row (+inf: no weight)
  int* grp_done;       // [U, 16]
  int* unit_done;      // [U]
  int* ready;          // [U] pass 2 may start
  float* col_out;      // [HH, n]
  float* diag_dst;     // [HH, n] zeroed by pass 1, red.add by pass 2
  int accumulate;      // col_out += (diag goes to a scratch buffer, added afterwards)
  const int4* units;
  const int32_t* unit_count;
  unsigned long long* trace;  // optional [grid, 64] globaltimer stamps (tools/vs_trace.py)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void vs_stamp(const TailArgs& a, int v, int e) {
  if (a.trace && v < 8) a.trace[blockIdx.x * 64 + v * 8 + e] = gtimer();
}
// per-tile clock stamps of CTA 0, wave 0 (tools/vs_trace.py): [gridDim.x * 64 + tile * 8 + e]
__device__ __forceinline__ void vs_tstamp(const TailArgs& a, int v, int tile, int e) {
  if (a.trace && v == 0 && blockIdx.x == 0 && tile < 32) a.trace[gridDim.x * 64 + tile * 8 + e] = clock64();
}

// 2^x for a pair on the FMA pipe: x = j + f (j = rint x by the 1.5*2^23 magic
// add), 2^f by a degree-5 fit on [-0.5, 0.5] (max relative error 2.4e-7 in
// fp32, the accuracy of ex2.approx), 2^j added into the exponent field;
// x < -125 (masked / unscored) gives exactly 0 like ex2.approx.ftz.
__device__ __forceinline__ float2 exp2_poly5(float2 x) {
  const float2 xc = make_float2(fmaxf(x.x, -125.f), fmaxf(x.y, -125.f));
  const float2 t = fadd2(xc, make_float2(12582912.f, 12582912.f));
  const float2 j = fadd2(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = ffma2(j, make_float2(-1.f, -1.f), xc);
  float2 p = ffma2(make_float2(0.0013277214f, 0.0013277214f), f, make_float2(0.0096755475f, 0.0096755475f));
  p = ffma2(p, f, make_float2(0.0555071086f, 0.0555071086f));
  p = ffma2(p, f, make_float2(0.2402212024f, 0.2402212024f));
  p = ffma2(p, f, make_float2(0.6931469440f, 0.6931469440f));
  p = ffma2(p, f, make_float2(1.0000001192f, 1.0000001192f));
  float2 r = make_float2(__uint_as_float(__float_as_uint(p.x) + (__float_as_uint(t.x) << 23)),
                         __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(t.y) << 23)));
  r.x = x.x < -125.f ? 0.f : r.x;
  r.y = x.y < -125.f ? 0.f : r.y;
  return r;
}

// pair p of a row block on the FMA pipe when (p & 7) < POLY8, else on MUFU
template <int POLY8>
__device__ __forceinline__ float2 exp2_mix(float2 x, int p) {
  if ((p & 7) < POLY8) return exp2_poly5(x);
  return make_float2(fast_exp2(x.x), fast_exp2(x.y));
}

// for sums only: x < -125 (masked) contributes 2^-125 instead of 0, which no
// row sum (>= 1, the maximum's own term) can notice
__device__ __forceinline__ float2 exp2_poly5_sum(float2 x) {
  const float2 xc = make_float2(fmaxf(x.x, -125.f), fmaxf(x.y, -125.f));
  const float2 t = fadd2(xc, make_float2(12582912.f, 12582912.f));
  const float2 j = fadd2(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = ffma2(j, make_float2(-1.f, -1.f), xc);
  float2 p = ffma2(make_float2(0.0013277214f, 0.0013277214f), f, make_float2(0.0096755475f, 0.0096755475f));
  p = ffma2(p, f, make_float2(0.0555071086f, 0.0555071086f));
  p = ffma2(p, f, make_float2(0.2402212024f, 0.2402212024f));
  p = ffma2(p, f, make_float2(0.6931469440f, 0.6931469440f));
  p = ffma2(p, f, make_float2(1.0000001192f, 1.0000001192f));
  return make_float2(__uint_as_float(__float_as_uint(p.x) + (__float_as_uint(t.x) << 23)),
                     __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(t.y) << 23)));
}
template <int POLY8>
__device__ __forceinline__ float2 exp2_mix_sum(float2 x, int p) {
  if ((p & 7) < POLY8) return exp2_poly5_sum(x);
  return make_float2(fast_exp2(x.x), fast_exp2(x.y));
}

__device__ __forceinline__ float2 merge_stat(float2 a, float2 b) {
  const float m = fmaxf(a.x, b.x);
  if (m == -INFINITY) return make_float2(-INFINITY, 0.f);
  return make_float2(m, a.y * fast_exp2(a.x - m) + b.y * fast_exp2(b.x - m));
}

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add(float* p, float v) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

// this CTA's place in the wave schedule (identical in every role)
struct VsPlace {
  int U, W, cpu, ws, rank, t_lo, t_hi, nwaves;
};
__device__ __forceinline__ VsPlace vs_place(const TailArgs& a) {
  VsPlace p;
  p.U = *a.unit_count;
  p.W = min(p.U, a.wave_units);
  p.cpu = p.W > 0 ? min((int)gridDim.x / p.W, min((a.nkt + a.min_tiles - 1) / a.min_tiles, kVsMaxCta)) : 0;
  p.ws = p.cpu > 0 ? (int)blockIdx.x / p.cpu : 0;
  p.rank = p.cpu > 0 ? (int)blockIdx.x % p.cpu : 0;
  p.t_lo = p.cpu > 0 ? (int)(((long long)p.rank * a.nkt) / p.cpu) : 0;
  p.t_hi = p.cpu > 0 ? (int)(((long long)(p.rank + 1) * a.nkt) / p.cpu) : 0;
  p.nwaves = p.W > 0 ? (p.U + p.W - 1) / p.W : 0;
  return p;
}

// P1POLY / P2POLY: pairs (of every 8) whose exp runs on the FMA pipe in pass 1 / 2
template <int P1POLY, int P2POLY>
__global__ void __launch_bounds__(kVsThreads, 1) vs_estimator_kernel(const __grid_constant__ TailArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem;
  uint8_t* sK = smem + kVsOffK;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kVsOffMisc);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + V_NUM);
  volatile int* flag = reinterpret_cast<volatile int*>(tmem_holder + 4);
  const int warp = warp_id();
  const VsPlace pl = vs_place(a);
  if (pl.W == 0 || pl.ws >= pl.W) return;  // idle CTA (uniform exit)

  if (threadIdx.x == 0) {
    mbar_init(&bars[V_QF], 1);
    mbar_init(&bars[V_QE], 1);
    for (int s = 0; s < kVsKSlots; ++s) {
      mbar_init(&bars[V_KF + s], 1);
      mbar_init(&bars[V_KE + s], 1);
    }
    for (int s = 0; s < 4; ++s) {
      mbar_init(&bars[V_SF + s], 1);
      mbar_init(&bars[V_SE + s], 256);
    }
    fence_barrier_init();
  }
  if (warp == kVsSoftWarps + 1) tmem_alloc(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_holder;

  if (warp == kVsSoftWarps) {
    // ------------------------------------------------------------ producer
    if (elect_one()) {
      int kj = 0;
      for (int v = 0; v < pl.nwaves; ++v) {
        const int u = v * pl.W + pl.ws;
        if (u >= pl.U) break;
        const int4 un = a.units[u];
        if (v > 0) mbar_wait_backoff<64>(&bars[V_QE], (v - 1) & 1);  // previous wave's MMAs read Q
        const int nslot = un.z >= 0 ? 2 : 1;
        mbar_arrive_expect_tx(&bars[V_QF], 32768 * nslot);
        for (int s = 0; s < nslot; ++s) {
          const int h0 = s ? un.z : un.x;
          const int h1r = s ? un.w : un.y;
          const int h1 = h1r >= 0 ? h1r : h0;  // a lone head fills both halves (rows inactive)
#pragma unroll
          for (int dh = 0; dh < 2; ++dh) {
            tma_load_3d(sQ + dh * 32768 + s * 16384, &a.tmap_q, &bars[V_QF], 64 * dh, a.qrow0, h0);
            tma_load_3d(sQ + dh * 32768 + s * 16384 + 8192, &a.tmap_q, &bars[V_QF], 64 * dh, a.qrow0, h1);
          }
        }
        const int hkv = (un.x / a.heads) * a.kv_heads + (un.x % a.heads) / (a.heads / a.kv_heads);
        // the whole K range of this CTA into L2 first: the two-slot ring then
        // waits for L2 latency instead of DRAM latency (pass 2 re-reads it from L2)
        for (int kt = pl.t_lo; kt < pl.t_hi; ++kt) {
          tma_prefetch_l2_3d(&a.tmap_k, 0, kt * kTile, hkv);
          tma_prefetch_l2_3d(&a.tmap_k, 64, kt * kTile, hkv);
        }
        for (int pass = 0; pass < 2; ++pass)
          for (int kt = pl.t_lo; kt < pl.t_hi; ++kt, ++kj) {
            const int ks = kj % kVsKSlots;
            if (kj >= kVsKSlots) mbar_wait_backoff<32>(&bars[V_KE + ks], ((kj / kVsKSlots) - 1) & 1);
            uint8_t* dst = sK + ks * 32768;
            mbar_arrive_expect_tx(&bars[V_KF + ks], 32768);
            tma_load_3d(dst, &a.tmap_k, &bars[V_KF + ks], 0, kt * kTile, hkv);
            tma_load_3d(dst + 16384, &a.tmap_k, &bars[V_KF + ks], 64, kt * kTile, hkv);
          }
      }
    }
  } else if (warp == kVsSoftWarps + 1) {
    // ------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc1 = idesc_bf16_f32(128, 128, 0, 0);
      constexpr uint32_t idesc2a = idesc_bf16_f32(128, 128, 0, 0);
      constexpr uint32_t idesc2b = idesc_bf16_f32(128, 256, 0, 0);
      const uint32_t q_addr = smem_u32(sQ);
      int kj = 0, jt = 0;
      for (int v = 0; v < pl.nwaves; ++v) {
        const int u = v * pl.W + pl.ws;
        if (u >= pl.U) break;
        const bool sb = a.units[u].z >= 0;
        mbar_wait(&bars[V_QF], v & 1);
        tc_fence_after();
        for (int pass = 1; pass <= 2; ++pass)
          for (int kt = pl.t_lo; kt < pl.t_hi; ++kt, ++kj, ++jt) {
            const int ks = kj % kVsKSlots, b = jt & 1;
            mbar_wait(&bars[V_KF + ks], (kj / kVsKSlots) & 1);
            if (pass == 1) vs_tstamp(a, v, kt - pl.t_lo, 4);
            if (jt >= 2) {
              mbar_wait(&bars[V_SE + b], ((jt >> 1) - 1) & 1);
              mbar_wait(&bars[V_SE + 2 + b], ((jt >> 1) - 1) & 1);
            }
            if (pass == 1) vs_tstamp(a, v, kt - pl.t_lo, 3);
            tc_fence_after();
            const uint32_t k_addr = smem_u32(sK + ks * 32768);
            const uint32_t d0 = tbase + b * 256;
            if (pass == 1) {
              // S[slot] = Q_slot K^T: rows on lanes, keys on columns
#pragma unroll
              for (int s = 0; s < 2; ++s) {
                if (s == 1 && !sb) break;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                  mma_ss(d0 + s * 128,
                         sdesc_sw128(q_addr + (kk >> 2) * 32768 + s * 16384 + (kk & 3) * 32, 16, 1024),
                         sdesc_sw128(k_addr + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), idesc1, kk > 0);
              }
            } else {
              // S^T = K Q^T over both slots' rows (N = 256): keys on lanes
#pragma unroll
              for (int kk = 0; kk < 8; ++kk)
                mma_ss(d0, sdesc_sw128(k_addr + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                       sdesc_sw128(q_addr + (kk >> 2) * 32768 + (kk & 3) * 32, 16, 1024), sb ? idesc2b : idesc2a,
                       kk > 0);
            }
            mma_commit(&bars[V_KE + ks]);
            mma_commit(&bars[V_SF + b]);
            mma_commit(&bars[V_SF + 2 + b]);
          }
        mma_commit(&bars[V_QE]);
      }
    }
  } else {
    // ------------------------------------------------------------ softmax warps
    const int grp = warp >> 2;      // 0..3
    const int slot = grp >> 1;      // 128-row slot
    const int sub = grp & 1;        // pass 1: key half of the tile; pass 2: head of the slot
    const int q4 = warp & 3;        // TMEM lane quarter
    const int t = threadIdx.x & 127;
    const int lane = threadIdx.x & 31;
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const float sl2 = a.scale_log2;
    float* Dw = reinterpret_cast<float*>(smem + kVsOffD) + warp * (16 * kDw);      // [16 rows][kDw] skewed
    float* C2 = reinterpret_cast<float*>(smem + kVsOffC) + grp * kC2Floats;         // [191 ops][9]
    float* nl = reinterpret_cast<float*>(smem + kVsOffNl) + grp * 64;               // -lse2 of the group's rows
    float2* xch = reinterpret_cast<float2*>(smem + kVsOffX);
    const int ng = (pl.cpu + kVsGroup - 1) / kVsGroup;
    int jt = 0;
    // zero the never-written parts of this warp's skewed buffer and of the
    // group's C2 (the written positions are the same for every tile)
    for (int x = lane; x < 16 * kDw; x += 32) Dw[x] = 0.f;
    for (int x = t; x < kC2Floats; x += 128) C2[x] = 0.f;
    named_bar_sync(2 + grp, 128);
    for (int v = 0; v < pl.nwaves; ++v) {
      const int u = v * pl.W + pl.ws;
      if (u >= pl.U) break;
      const int4 un = a.units[u];
      const int ha = slot ? un.z : un.x, hb = slot ? un.w : un.y;
      const bool on = ha >= 0;
      // ---------------------------------------------------- pass 1 (thread = row, half the keys)
      if (threadIdx.x == 0) vs_stamp(a, v, 0);
      {
        const int hrow = (t < 64) ? ha : hb;
        const int i = a.qrow0 + (t & 63);
        const bool active = on && hrow >= 0 && i >= a.r_lo && i < a.r_hi;
        float m = -INFINITY, ssum = 0.f;
        for (int kt = pl.t_lo; kt < pl.t_hi; ++kt, ++jt) {
          const int b = jt & 1;
          mbar_wait(&bars[V_SF + slot * 2 + b], (jt >> 1) & 1);
          if (threadIdx.x == 0) vs_tstamp(a, v, kt - pl.t_lo, 0);
          if (on) {
            tc_fence_after();
            uint32_t s[64];
            tmem_ld32(tbase + lane_off + b * 256 + slot * 128 + 64 * sub, *reinterpret_cast<uint32_t(*)[32]>(s));
            tmem_ld32(tbase + lane_off + b * 256 + slot * 128 + 64 * sub + 32,
                      *reinterpret_cast<uint32_t(*)[32]>(s + 32));
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(&bars[V_SE + slot * 2 + b]);
            if (threadIdx.x == 0) vs_tstamp(a, v, kt - pl.t_lo, 1);
            const int lim = i - (kt * kTile + 64 * sub);  // keep columns c <= lim
            const bool diag_tile = __any_sync(0xffffffffu, active && lim < 63);  // warp-uniform
            if (active) {
              if (diag_tile) {
#pragma unroll
                for (int c = 0; c < 64; ++c)
                  if (c > lim) s[c] = __float_as_uint(-INFINITY);
              }
              float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
              for (int c = 0; c < 64; c += 8) {
                m4[0] = fmax3(m4[0], __uint_as_float(s[c]), __uint_as_float(s[c + 1]));
                m4[1] = fmax3(m4[1], __uint_as_float(s[c + 2]), __uint_as_float(s[c + 3]));
                m4[2] = fmax3(m4[2], __uint_as_float(s[c + 4]), __uint_as_float(s[c + 5]));
                m4[3] = fmax3(m4[3], __uint_as_float(s[c + 6]), __uint_as_float(s[c + 7]));
              }
              const float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
              if (mx != -INFINITY) {
                const float mn = fmaxf(m, mx * sl2);
                const float2 sc2 = make_float2(sl2, sl2), mo2 = make_float2(-mn, -mn);
                float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                                 make_float2(0.f, 0.f)};
#pragma unroll
                for (int c = 0; c < 64; c += 2) {
                  const float2 x = ffma2(make_float2(__uint_as_float(s[c]), __uint_as_float(s[c + 1])), sc2, mo2);
                  acc[(c >> 1) & 3] = fadd2(acc[(c >> 1) & 3], exp2_mix_sum<P1POLY>(x, c >> 1));
                }
                const float2 a01 = fadd2(acc[0], acc[1]), a23 = fadd2(acc[2], acc[3]);
                ssum = ssum * fast_exp2(m - mn) + ((a01.x + a01.y) + (a23.x + a23.y));
                m = mn;
              }
            }
            if (threadIdx.x == 0) vs_tstamp(a, v, kt - pl.t_lo, 2);
          } else {
            mbar_arrive(&bars[V_SE + slot * 2 + b]);
          }
        }
        // per-(chunk, key half, row) statistics (unscored rows: (-inf, 0))
        a.stats[(((size_t)u * kVsMaxCta + pl.rank) * 2 + sub) * 256 + slot * 128 + t] = make_float2(m, ssum);
        // zero this chunk's range of the diagonal output (and the column tail
        // beyond the scored keys) for the unit's heads: pass 2 adds into them
        {
          const int o_lo = pl.t_lo * kTile;
          const int o_hi = pl.t_hi == a.nkt ? a.n : min(a.n, pl.t_hi * kTile);
          const int tid = threadIdx.x;
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            const int h = qq == 0 ? un.x : (qq == 1 ? un.y : (qq == 2 ? un.z : un.w));
            if (h < 0) continue;
            float* dd = a.diag_dst + (size_t)h * a.n;
            for (int o = o_lo + tid; o < o_hi; o += kVsSoft) dd[o] = 0.f;
            if (!a.accumulate && pl.t_hi == a.nkt) {
              float* cc = a.col_out + (size_t)h * a.n;
              for (int j = a.nkt * kTile + tid; j < a.n; j += kVsSoft) cc[j] = 0.f;
            }
          }
        }
        named_bar_sync(1, kVsSoft);
        if (threadIdx.x == 0) vs_stamp(a, v, 1);
        const int g1 = pl.rank / kVsGroup;
        if (threadIdx.x == 0) {  // barrier, then one gpu-scope fence + atomic (release pattern)
          __threadfence();
          const int gsz = min(kVsGroup, pl.cpu - g1 * kVsGroup);
          flag[0] = atomicAdd(&a.grp_done[u * kVsGroup + g1], 1) == gsz - 1;
        }
        named_bar_sync(1, kVsSoft);
        if (flag[0]) {
          // first-level merge of the group's chunks (fixed order): thread = (row, key half)
          const int row = threadIdx.x & 255, half = threadIdx.x >> 8;
          const int c0 = g1 * kVsGroup, cn = min(pl.cpu, c0 + kVsGroup) - c0;
          float2 vv[kVsGroup];
#pragma unroll
          for (int c = 0; c < kVsGroup; ++c)
            vv[c] = c < cn ? __ldcg(&a.stats[(((size_t)u * kVsMaxCta + c0 + c) * 2 + half) * 256 + row])
                           : make_float2(-INFINITY, 0.f);
          float2 acc = make_float2(-INFINITY, 0.f);
#pragma unroll
          for (int c = 0; c < kVsGroup; ++c) acc = merge_stat(acc, vv[c]);
          if (half) xch[row] = acc;
          named_bar_sync(1, kVsSoft);
          if (!half) a.stats2[((size_t)u * kVsGroup + g1) * 256 + row] = merge_stat(acc, xch[row]);
          named_bar_sync(1, kVsSoft);
          if (threadIdx.x == 0) {
            __threadfence();
            flag[1] = atomicAdd(&a.unit_done[u], 1) == ng - 1;
          }
          named_bar_sync(1, kVsSoft);
          if (flag[1]) {
            if (!half) {
              float2 v2[kVsGroup];
#pragma unroll
              for (int g = 0; g < kVsGroup; ++g)
                v2[g] = g < ng ? __ldcg(&a.stats2[((size_t)u * kVsGroup + g) * 256 + row])
                               : make_float2(-INFINITY, 0.f);
              float2 r = make_float2(-INFINITY, 0.f);
#pragma unroll
              for (int g = 0; g < kVsGroup; ++g) r = merge_stat(r, v2[g]);
              a.lse2[(size_t)u * 256 + row] = r.y > 0.f ? r.x + log2f(r.y) : INFINITY;
            }
            named_bar_sync(1, kVsSoft);
            if (threadIdx.x == 0) {
              __threadfence();
              st_release(&a.ready[u], 1);
              vs_stamp(a, v, 2);
            }
          }
        }
      }
      // ---------------------------------------------------- pass 2 (thread = key, one head's rows)
      {
        const int h = sub ? hb : ha;
        const bool work = on && h >= 0;
        if (work) {
          if (t == 0) {
            while (ld_relaxed(&a.ready[u]) == 0) __nanosleep(64);
            __threadfence();  // acquire: the statistics written before the release
            if (threadIdx.x == 0) vs_stamp(a, v, 3);
          }
          named_bar_sync(2 + grp, 128);
          if (t < 64) nl[t] = -__ldcg(a.lse2 + (size_t)u * 256 + slot * 128 + sub * 64 + t);
          named_bar_sync(2 + grp, 128);
        }
        const float2 sc2 = make_float2(sl2, sl2);
        const int kslot = 4 * (q4 & 1);  // C2 slot of this warp's blocks: m + 4 (q4 & 1)
        // diagonal op of block m, main column lane: 16 m + 96 - 32 q4 + 46 - lane;
        // second column 32 + (lane >> 1): 16 m + 96 - 32 q4 + 14 - (lane >> 1)
        const int op_main = 142 - 32 * q4 - lane;
        const int op_sec = 110 - 32 * q4 - (lane >> 1);
        const bool sec_on = (lane & 1) == 0 && lane < 30;
        for (int kt = pl.t_lo; kt < pl.t_hi; ++kt, ++jt) {
          const int b = jt & 1;
          mbar_wait(&bars[V_SF + slot * 2 + b], (jt >> 1) & 1);
          if (!work) {
            mbar_arrive(&bars[V_SE + slot * 2 + b]);
            continue;
          }
          tc_fence_after();
          const int j = kt * kTile + t;
          const int obase = a.qrow0 - kt * kTile - 127;
          float Pm[4], Ps[4];  // per 16-row block: main / second column sums
          float2 cs = make_float2(0.f, 0.f);
#pragma unroll
          for (int qh = 0; qh < 2; ++qh) {
            uint32_t s[32];
            tmem_ld32(tbase + lane_off + b * 256 + slot * 128 + sub * 64 + qh * 32, s);
            tmem_ld_wait();
            if (qh == 1) {
              tc_fence_before();
              mbar_arrive(&bars[V_SE + slot * 2 + b]);
            }
            // rows of this quarter: frame rows 32 qh + c, global qrow0 + 32 qh + c; causal j <= i
            const int cmin = j - (a.qrow0 + 32 * qh);  // rows c >= cmin see key j
            const bool cut = __any_sync(0xffffffffu, cmin > 0);
#pragma unroll
            for (int c = 0; c < 32; c += 4) {
              const float4 nv = *reinterpret_cast<const float4*>(nl + qh * 32 + c);  // broadcast
              float2 x0 = ffma2(make_float2(__uint_as_float(s[c]), __uint_as_float(s[c + 1])), sc2,
                                make_float2(nv.x, nv.y));
              float2 x1 = ffma2(make_float2(__uint_as_float(s[c + 2]), __uint_as_float(s[c + 3])), sc2,
                                make_float2(nv.z, nv.w));
              float2 e0 = exp2_mix<P2POLY>(x0, c >> 1);
              float2 e1 = exp2_mix<P2POLY>(x1, (c >> 1) + 1);
              if (cut) {
                e0.x = c >= cmin ? e0.x : 0.f;
                e0.y = c + 1 >= cmin ? e0.y : 0.f;
                e1.x = c + 2 >= cmin ? e1.x : 0.f;
                e1.y = c + 3 >= cmin ? e1.y : 0.f;
              }
              cs = fadd2(cs, fadd2(e0, e1));
              s[c] = __float_as_uint(e0.x);
              s[c + 1] = __float_as_uint(e0.y);
              s[c + 2] = __float_as_uint(e1.x);
              s[c + 3] = __float_as_uint(e1.y);
            }
            // two 16-row blocks through this warp's skewed buffer: lane l writes
            // row c at column l - c + 15, so column x holds one diagonal
            // (c + 31 - l = 46 - x) with zeros elsewhere: lane x sums column x,
            // lanes 2k, 2k+1 sum half of column 32 + k each; no selects, and
            // every address is the lane base plus an immediate
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              __syncwarp();
#pragma unroll
              for (int c = 0; c < 16; ++c) Dw[c * kDw - c + 15 + lane] = __uint_as_float(s[16 * e + c]);
              __syncwarp();
              float v1 = 0.f, v2 = 0.f;
#pragma unroll
              for (int c = 0; c < 16; ++c) v1 += Dw[c * kDw + lane];
              const float* col2 = Dw + 8 * (lane & 1) * kDw + 32 + (lane >> 1);  // lanes 30, 31: zero column 47
#pragma unroll
              for (int c = 0; c < 8; ++c) v2 += col2[c * kDw];
              v2 += __shfl_xor_sync(0xffffffffu, v2, 1);
              Pm[2 * qh + e] = v1;
              Ps[2 * qh + e] = v2;
            }
          }
          if (j < a.n) {
            float* dst = a.col_out + (size_t)h * a.n + j;
            const float tot = cs.x + cs.y;
            *dst = a.accumulate ? (*dst + tot) : tot;
          }
          // partials -> C2[op][slot] (one writer per entry), then each thread sums
          // the 8 slots of diagonals t and t + 128 in slot order
          named_bar_sync(2 + grp, 128);  // the previous tile's readers are done
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            C2[(op_main + 16 * m) * 9 + kslot + m] = Pm[m];
            if (sec_on) C2[(op_sec + 16 * m) * 9 + kslot + m] = Ps[m];
          }
          named_bar_sync(2 + grp, 128);
          float* dd = a.diag_dst + (size_t)h * a.n;
#pragma unroll
          for (int k2 = 0; k2 < 2; ++k2) {
            const int op = t + 128 * k2;
            if (op > 190) break;
            const float* cr = C2 + op * 9;
            const float vsum = ((cr[0] + cr[1]) + (cr[2] + cr[3])) + ((cr[4] + cr[5]) + (cr[6] + cr[7]));
            const int o = obase + op;
            if (o >= 0 && o < a.n) red_add(dd + o, vsum);
          }
        }
        if (threadIdx.x == 0) vs_stamp(a, v, 4);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kVsSoftWarps + 1) tmem_dealloc(tbase, 512);
}

// Units from the device-selected families (one CTA, a warp per kv group): up to
// four selected heads of one kv group per unit (slot A = the first two, slot B
// the next two, -1 padded); head_list = every selected head.  Also zeroes the
// estimator's queue / completion counters.
__global__ void build_units_kernel(const int32_t* gate, int gate_val, int hh_total, int heads, int kv_heads,
                                   int4* units, int32_t* unit_count, int32_t* head_list, int32_t* head_count,
                                   int* sched, int sched_ints) {
  __shared__ int n_units, n_heads;
  if (threadIdx.x == 0) n_units = n_heads = 0;
  for (int x = threadIdx.x; x < sched_ints; x += blockDim.x) sched[x] = 0;
  __syncthreads();
  const int g = heads / kv_heads;
  const int groups = hh_total / g;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int grp = w; grp < groups; grp += nw) {
    for (int base = 0; base < g; base += 32) {
      const int h = grp * g + base + lane;
      const bool on = base + lane < g && (gate == nullptr || gate[h] == gate_val);
      const uint32_t bal = __ballot_sync(0xffffffffu, on);
      const int cnt = __popc(bal);
      const int rank = __popc(bal & ((1u << lane) - 1u));
      int hb = 0, ub = 0;
      const int nu = (cnt + 3) / 4;
      if (lane == 0) {
        hb = atomicAdd(&n_heads, cnt);
        ub = atomicAdd(&n_units, nu);
      }
      hb = __shfl_sync(0xffffffffu, hb, 0);
      ub = __shfl_sync(0xffffffffu, ub, 0);
      if (on) head_list[hb + rank] = h;
      if (lane < nu) units[ub + lane] = make_int4(-1, -1, -1, -1);
      __syncwarp();
      if (on) reinterpret_cast<int*>(&units[ub + rank / 4])[rank & 3] = h;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *unit_count = n_units;
    *head_count = n_heads;
  }
}

// diag_out[h] += dtmp[h] for the scored heads (accumulating launches)
__global__ void diag_add_kernel(float* diag_out, const float* dtmp, int n, const int32_t* head_list,
                                const int32_t* head_count) {
  const int rank = blockIdx.y;
  if (rank >= *head_count) return;
  const size_t h = head_list[rank];
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < n; o += gridDim.x * blockDim.x)
    diag_out[h * n + o] += dtmp[h * n + o];
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

static unsigned long long* g_vs_trace = nullptr;  // set by sa_vs_trace_buffer (profiling only)

static int sched_ints(int hh_total) { return hh_total * (kVsGroup + 2); }

// units per wave: W units' K (256 n bytes each) stay L2-resident between the passes
static int tail_wave_units(int n) {
  static const int env = [] {
    const char* e = getenv("SA_VS_WAVE");  // A/B override
    return e ? atoi(e) : 0;
  }();
  if (env > 0) return env;
  return (int)std::max<size_t>(1, kVsWaveBytes / ((size_t)n * 256));
}

// workspace of one estimator call: statistics, completion state, unit lists and
// the scratch diagonal of accumulating launches
size_t tail_workspace_bytes(int hh_total, int n, int r_hi) {
  (void)r_hi;
  const size_t U = hh_total;
  return align256(U * kVsMaxCta * 2 * 256 * sizeof(float2)) + align256(U * kVsGroup * 256 * sizeof(float2)) +
         align256(U * 256 * 4) + align256((size_t)sched_ints(hh_total) * 4) +
         align256((size_t)(hh_total + 2) * 4) + align256(U * sizeof(int4)) + align256((size_t)hh_total * n * 4) +
         256;
}

// One estimator launch over rows [r_lo, r_hi), r_hi - r_lo <= 64.
static int launch_tail64(int batch, int heads, int kv_heads, int n, float scale, const void* q, const void* k,
                         int r_lo, int r_hi, float* col_out, float* diag_out, int accumulate, const int32_t* gate,
                         int gate_val, void* ws, size_t ws_bytes, cudaStream_t st) {
  TailArgs a;
  memset(&a, 0, sizeof(a));
  int rc;
  if ((rc = make_tmap_3d_bf16(&a.tmap_q, q, kHeadDim, n, batch * heads, 64))) return rc;
  if ((rc = make_tmap_3d_bf16(&a.tmap_k, k, kHeadDim, n, batch * kv_heads, kTile))) return rc;
  a.n = n;
  a.heads = heads;
  a.kv_heads = kv_heads;
  a.hh_total = batch * heads;
  a.r_lo = r_lo;
  a.r_hi = r_hi;
  a.qrow0 = r_hi - 64;
  a.nkt = (r_hi + kTile - 1) / kTile;
  a.wave_units = tail_wave_units(n);
  // fewest key tiles per CTA: a unit of a small launch (the auto layer's few
  // VS heads) takes ceil(key tiles / 8) CTAs instead of one per key tile, so
  // its CTAs leave SMs to the block GEMM beside it (32K auto layer 1.100 ->
  // 1.090 ms with the side stream at top priority; all-VS layers, whose units
  // fill the waves, unchanged).  SA_VS_MIN_TILES overrides, for A/B.
  static const int min_tiles = [] {
    const char* e = getenv("SA_VS_MIN_TILES");
    const int v = e ? atoi(e) : 8;
    return v >= 1 ? v : 1;
  }();
  a.min_tiles = min_tiles;
  a.scale_log2 = scale * 1.4426950408889634f;
  if (ws_bytes < tail_workspace_bytes(a.hh_total, n, r_hi))
    return fail(SA_ERR_DIMENSION, "score_tail workspace too small");
  const size_t U = a.hh_total;
  char* w = reinterpret_cast<char*>(ws);
  a.stats = reinterpret_cast<float2*>(w);
  w += align256(U * kVsMaxCta * 2 * 256 * sizeof(float2));
  a.stats2 = reinterpret_cast<float2*>(w);
  w += align256(U * kVsGroup * 256 * sizeof(float2));
  a.lse2 = reinterpret_cast<float*>(w);
  w += align256(U * 256 * 4);
  int* sched = reinterpret_cast<int*>(w);
  w += align256((size_t)sched_ints(a.hh_total) * 4);
  int32_t* list = reinterpret_cast<int32_t*>(w);  // [0] head count, [1] unit count, [2..] heads
  w += align256((size_t)(a.hh_total + 2) * 4);
  int4* units = reinterpret_cast<int4*>(w);
  w += align256(U * sizeof(int4));
  float* dtmp = reinterpret_cast<float*>(w);
  a.grp_done = sched;
  a.unit_done = sched + a.hh_total * kVsGroup;
  a.ready = a.unit_done + a.hh_total;
  a.col_out = col_out;
  a.diag_dst = accumulate ? dtmp : diag_out;
  a.accumulate = accumulate;
  a.units = units;
  a.unit_count = list + 1;
  a.trace = g_vs_trace;
  build_units_kernel<<<1, 1024, 0, st>>>(gate, gate_val, a.hh_total, heads, kv_heads, units, list + 1, list + 2,
                                          list, sched, sched_ints(a.hh_total));
  if ((rc = check_launch("build_units_kernel"))) return rc;
  // exp split between MUFU and the FMA pipe per pass (SA_VS_POLY="p1,p2" for A/B)
  static const int poly = [] {
    const char* e = getenv("SA_VS_POLY");
    int p1 = 3, p2 = 0;
    if (e) sscanf(e, "%d,%d", &p1, &p2);
    return p1 * 10 + p2;
  }();
  void (*kern)(TailArgs);
  switch (poly) {
    case 0: kern = vs_estimator_kernel<0, 0>; break;
    case 20: kern = vs_estimator_kernel<2, 0>; break;
    case 40: kern = vs_estimator_kernel<4, 0>; break;
    case 32: kern = vs_estimator_kernel<3, 2>; break;
    default: kern = vs_estimator_kernel<3, 0>; break;
  }
  static std::atomic<uint64_t> attr_done{0};
  once_per_device(attr_done, [] {
    cudaFuncSetAttribute(vs_estimator_kernel<0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kVsSmemBytes);
    cudaFuncSetAttribute(vs_estimator_kernel<2, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kVsSmemBytes);
    cudaFuncSetAttribute(vs_estimator_kernel<3, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kVsSmemBytes);
    cudaFuncSetAttribute(vs_estimator_kernel<4, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kVsSmemBytes);
    cudaFuncSetAttribute(vs_estimator_kernel<3, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kVsSmemBytes);
  });
  // one CTA per SM: the waiting CTAs of a unit only wait for CTAs that are resident
  const int grid = device_sm_count();
  kern<<<grid, kVsThreads, kVsSmemBytes, st>>>(a);
  if ((rc = check_launch("vs_estimator_kernel"))) return rc;
  if (accumulate) {
    dim3 g2((n + 1023) / 1024, a.hh_total);
    diag_add_kernel<<<g2, 256, 0, st>>>(diag_out, dtmp, n, list + 2, list);
    if ((rc = check_launch("diag_add_kernel"))) return rc;
  }
  return SA_OK;
}

// Score rows [r_lo, r_hi) (R <= 128) of every (gated) head into col/diag (fp32,
// [HH, n]); launches of <= 64 rows, the later ones accumulating.
int launch_score_tail(int batch, int heads, int kv_heads, int n, float scale, const void* q, const void* k,
                      int r_lo, int r_hi, float* col_out, float* diag_out, int accumulate, const int32_t* gate,
                      int gate_val, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (r_hi > n || r_lo < 0 || r_hi - r_lo < 1 || r_hi - r_lo > 128)
    return fail(SA_ERR_PATTERN_PARAM, "tail rows [%d, %d) invalid for n=%d", r_lo, r_hi, n);
  int rc;
  int hi = r_hi;
  int acc = accumulate;
  while (hi > r_lo) {
    const int lo = std::max(r_lo, hi - 64);
    if ((rc = launch_tail64(batch, heads, kv_heads, n, scale, q, k, lo, hi, col_out, diag_out, acc, gate, gate_val,
                            ws, ws_bytes, st)))
      return rc;
    hi = lo;
    acc = 1;
  }
  return SA_OK;
}

}  // namespace sa

// Profiling hook: a device buffer of [grid, 64] u64 globaltimer stamps per
// estimator launch (nullptr disables).  Not part of the reference interface.
extern "C" int sa_vs_trace_buffer(void* p) {
  sa::g_vs_trace = reinterpret_cast<unsigned long long*>(p);
  return 0;
}

extern "C" size_t sa_score_tail_workspace(int batch, int heads, int n, int r_hi) {
  return sa::tail_workspace_bytes(batch * heads, n, r_hi);
}

extern "C" int sa_score_tail(int batch, int heads, int kv_heads, int n, float scale, const void* q,
                             const void* k, int r_lo, int r_hi, float* col_out, float* diag_out,
                             int accumulate, const int32_t* gate, int gate_val, void* ws,
                             size_t ws_bytes, void* stream) {
  using namespace sa;
  if (batch < 1 || heads < 1 || kv_heads < 1 || n < 1 || heads % kv_heads)
    return fail(SA_ERR_DIMENSION, "bad head layout");
  if (!q || !k || !col_out || !diag_out || !ws) return fail(SA_ERR_DIMENSION, "null pointer");
  return launch_score_tail(batch, heads, kv_heads, n, scale, q, k, r_lo, r_hi, col_out, diag_out,
                           accumulate, gate, gate_val, ws, ws_bytes,
                           reinterpret_cast<cudaStream_t>(stream));
}
