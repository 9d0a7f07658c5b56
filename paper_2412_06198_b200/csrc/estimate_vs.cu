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
// Work items (unit, pass, key chunk) come from one atomic queue ordered
//   P1(0) | P1(1) P2(0) | P1(2) P2(1) | ... | P2(U-1)
// so a unit's pass 2 re-reads K that its pass 1 brought into L2 one unit ago
// (K is read from HBM about once), and CTAs that finish pass 1 early have the
// next unit's pass 1 to work on while the statistics are merged.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "api_common.h"
#include "internal.h"
#include "sa_types.h"
#include "sm100_common.cuh"

namespace sa {

constexpr int kVsThreads = 320;  // warps 0-3: slot A, 4-7: slot B, 8: TMA producer, 9: MMA issuer
constexpr int kVsSoft = 256;
constexpr int kVsRing = 2;       // work-item ring: the producer claims one item ahead
constexpr int kVsKSlots = 2;
constexpr int kVsGroup = 16;     // pass-1 chunks merged per first-level group
constexpr int kVsMaxChunks = kVsGroup * kVsGroup;  // chunks per unit (two-level merge)
// shared memory: Q [2 buffers][64 KB] | K [2 slots][32 KB] | D [8 warps][16 x 32] f32 |
// C [2 groups][2 buffers][4 warps][6][32] f32 | misc
constexpr int kVsOffK = 2 * 65536;
constexpr int kVsOffD = kVsOffK + kVsKSlots * 32768;
constexpr int kVsOffC = kVsOffD + 8 * 2048;
constexpr int kVsOffMisc = kVsOffC + 2 * 2 * 768 * 4;
constexpr int kVsOffNl = kVsOffMisc + 256;  // [2 groups][128] -lse2 of the slot's rows
constexpr int kVsSmemBytes = kVsOffMisc + 1536 + 1024;

enum VBar {
  V_QF = 0,              // [2] Q buffer loaded
  V_QE = 2,              // [2] MMAs done with a Q buffer
  V_KF = 4,              // [2] K slot loaded
  V_KE = 6,              // [2] MMAs done with a K slot
  V_SF = 8,              // [slot * 2 + buf] S ready
  V_SE = 12,             // [slot * 2 + buf] S consumed (128 arrivals)
  V_IF = 16,             // [4] ring entry written
  V_IE = 20,             // [4] ring entry read (MMA + 8 softmax warps)
  V_NUM = 24
};

struct TailArgs {
  CUtensorMap tmap_q;  // [HH, n, 128], box {64, 64 rows}
  CUtensorMap tmap_k;  // [HK, n, 128], box {64, 128 rows}
  int n, heads, kv_heads, hh_total;
  int r_lo, r_hi;      // scored rows, r_hi - r_lo <= 64
  int qrow0;           // global row of Q box row 0 (r_hi - 64, may be negative)
  int nkt;             // key tiles with a causal key: ceil(r_hi / 128)
  int t1, c1;          // pass-1 tiles per item, items per unit
  int t2, c2;          // pass-2 tiles per item, items per unit
  int look;            // units between a unit's pass 1 and its pass 2 in the queue
  float scale_log2;
  float2* stats;       // [U, c1, 256] per-(chunk, row) (max2, sum)
  float2* stats2;      // [U, 16, 256] per-(group, row)
  float* lse2;         // [U, 256] log2-sum-exp per row (+inf: no weight)
  int* next;           // work-queue head
  int* grp_done;       // [U, 16]
  int* unit_done;      // [U]
  int* ready;          // [U] pass 2 may start
  float* col_out;      // [HH, n]
  float* diag_dst;     // [HH, n] zeroed by pass 1, red.add by pass 2
  int accumulate;      // col_out += (diag goes to a scratch buffer, added afterwards)
  const int4* units;
  const int32_t* unit_count;
};

struct VsItem {
  int pass, unit, chunk, t_lo, t_hi;
};

// queue position -> (pass, unit, chunk): block b holds P1(b) (b < U) then
// P2(b - L) (L <= b < U + L); the look-ahead L keeps the claimed-but-unfinished
// window of the grid inside the pass-1 items of later units
__device__ __forceinline__ int vs_block_start(int b, int U, const TailArgs& a) {
  return min(b, U) * a.c1 + max(0, min(b, U + a.look) - a.look) * a.c2;
}
__device__ __forceinline__ VsItem vs_item(int i, int U, const TailArgs& a) {
  VsItem w;
  int blk = 0;
  while (vs_block_start(blk + 1, U, a) <= i) ++blk;
  const int r = i - vs_block_start(blk, U, a);
  if (blk < U && r < a.c1) {
    w.pass = 1;
    w.unit = blk;
    w.chunk = r;
  } else {
    w.pass = 2;
    w.unit = blk - a.look;
    w.chunk = blk < U ? r - a.c1 : r;
  }
  const int T = w.pass == 1 ? a.t1 : a.t2;
  w.t_lo = w.chunk * T;
  w.t_hi = min(a.nkt, w.t_lo + T);
  return w;
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

__global__ void __launch_bounds__(kVsThreads, 1) vs_estimator_kernel(const __grid_constant__ TailArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem;
  uint8_t* sK = smem + kVsOffK;
  float* sD = reinterpret_cast<float*>(smem + kVsOffD);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kVsOffMisc);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + V_NUM);
  volatile int* ring = reinterpret_cast<volatile int*>(tmem_holder + 4);
  volatile int* flag = ring + kVsRing;
  const int warp = warp_id();
  const int U = *a.unit_count;
  const int total = U * (a.c1 + a.c2);
  if ((int)blockIdx.x >= total) return;

  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bars[V_QF + s], 1);
      mbar_init(&bars[V_QE + s], 1);
      mbar_init(&bars[V_KF + s], 1);
      mbar_init(&bars[V_KE + s], 1);
    }
    for (int s = 0; s < 4; ++s) {
      mbar_init(&bars[V_SF + s], 1);
      mbar_init(&bars[V_SE + s], 128);
      if (s < kVsRing) {
        mbar_init(&bars[V_IF + s], 1);
        mbar_init(&bars[V_IE + s], 1 + 8);
      }
    }
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_holder;

  if (warp == 8) {
    // ------------------------------------------------------------ producer
    if (elect_one()) {
      int cur_unit = -1, qb = -1, kj = 0;
      int quse0 = 0, quse1 = 0;  // loads into each Q buffer
      for (int it = 0;; ++it) {
        const int rs = it & (kVsRing - 1);
        if (it >= kVsRing) mbar_wait_backoff<32>(&bars[V_IE + rs], ((it / kVsRing) - 1) & 1);
        int item = atomicAdd(a.next, 1);
        if (item >= total) item = -1;
        ring[rs] = item;
        mbar_arrive(&bars[V_IF + rs]);
        if (item < 0) break;
        const VsItem w = vs_item(item, U, a);
        const int4 un = a.units[w.unit];
        if (w.unit != cur_unit) {
          qb = qb < 0 ? 0 : qb ^ 1;
          const int qu = qb ? quse1 : quse0;
          if (qu > 0) mbar_wait_backoff<32>(&bars[V_QE + qb], (qu - 1) & 1);
          if (qb) ++quse1;
          else ++quse0;
          const int nslot = un.z >= 0 ? 2 : 1;
          uint8_t* q = sQ + qb * 65536;
          mbar_arrive_expect_tx(&bars[V_QF + qb], 32768 * nslot);
          for (int s = 0; s < nslot; ++s) {
            const int h0 = s ? un.z : un.x;
            const int h1r = s ? un.w : un.y;
            const int h1 = h1r >= 0 ? h1r : h0;  // a lone head fills both halves (rows inactive)
#pragma unroll
            for (int dh = 0; dh < 2; ++dh) {
              tma_load_3d(q + dh * 32768 + s * 16384, &a.tmap_q, &bars[V_QF + qb], 64 * dh, a.qrow0, h0);
              tma_load_3d(q + dh * 32768 + s * 16384 + 8192, &a.tmap_q, &bars[V_QF + qb], 64 * dh, a.qrow0, h1);
            }
          }
          cur_unit = w.unit;
        }
        const int hkv = (un.x / a.heads) * a.kv_heads + (un.x % a.heads) / (a.heads / a.kv_heads);
        for (int kt = w.t_lo; kt < w.t_hi; ++kt, ++kj) {
          const int ks = kj & 1;
          if (kj >= kVsKSlots) mbar_wait_backoff<32>(&bars[V_KE + ks], ((kj >> 1) - 1) & 1);
          uint8_t* dst = sK + ks * 32768;
          mbar_arrive_expect_tx(&bars[V_KF + ks], 32768);
          tma_load_3d(dst, &a.tmap_k, &bars[V_KF + ks], 0, kt * kTile, hkv);
          tma_load_3d(dst + 16384, &a.tmap_k, &bars[V_KF + ks], 64, kt * kTile, hkv);
        }
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc1 = idesc_bf16_f32(128, 128, 0, 0);
      constexpr uint32_t idesc2a = idesc_bf16_f32(128, 128, 0, 0);
      constexpr uint32_t idesc2b = idesc_bf16_f32(128, 256, 0, 0);
      int cur_unit = -1, qb = -1, kj = 0, jt = 0;
      int qfn0 = 0, qfn1 = 0;  // uses of each Q buffer
      for (int it = 0;; ++it) {
        const int rs = it & (kVsRing - 1);
        mbar_wait(&bars[V_IF + rs], (it / kVsRing) & 1);
        const int item = ring[rs];
        if (item < 0) break;
        const VsItem w = vs_item(item, U, a);
        const bool sb = a.units[w.unit].z >= 0;
        if (w.unit != cur_unit) {
          qb = qb < 0 ? 0 : qb ^ 1;
          mbar_wait(&bars[V_QF + qb], (qb ? qfn1 : qfn0) & 1);
          if (qb) ++qfn1;
          else ++qfn0;
          cur_unit = w.unit;
        }
        const uint32_t q_addr = smem_u32(sQ + qb * 65536);
        tc_fence_after();
        for (int kt = w.t_lo; kt < w.t_hi; ++kt, ++kj, ++jt) {
          const int ks = kj & 1, b = jt & 1;
          mbar_wait(&bars[V_KF + ks], (kj >> 1) & 1);
          if (jt >= 2) {
            mbar_wait(&bars[V_SE + b], ((jt >> 1) - 1) & 1);
            mbar_wait(&bars[V_SE + 2 + b], ((jt >> 1) - 1) & 1);
          }
          tc_fence_after();
          const uint32_t k_addr = smem_u32(sK + ks * 32768);
          const uint32_t d0 = tbase + b * 256;
          if (w.pass == 1) {
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
        // hand the Q buffer back when the next item belongs to another unit
        const int rn = (it + 1) & (kVsRing - 1);
        mbar_wait(&bars[V_IF + rn], ((it + 1) / kVsRing) & 1);
        const int nxt = ring[rn];
        if (nxt >= 0 && vs_item(nxt, U, a).unit != cur_unit) mma_commit(&bars[V_QE + qb]);
        mbar_arrive(&bars[V_IE + rs]);
      }
    }
  } else {
    // ------------------------------------------------------------ softmax warps
    const int grp = warp >> 2;  // slot
    const int t = threadIdx.x & 127;
    const int lane = threadIdx.x & 31;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const float sl2 = a.scale_log2;
    const int pw = warp & 3;                                  // this warp's 32 keys of the tile
    float* Dw = sD + warp * 512;                              // [16 rows][32 keys] per warp
    float* sC = reinterpret_cast<float*>(smem + kVsOffC) + grp * 1536;  // [2][4 warps][6][32]
    int cbuf = 0;
    float* nl = reinterpret_cast<float*>(smem + kVsOffNl) + grp * 128;  // pass 2: -lse2 (-inf: no weight)
    int jt = 0;
    int nl_unit = -1;
    for (int it = 0;; ++it) {
      const int rs = it & (kVsRing - 1);
      mbar_wait(&bars[V_IF + rs], (it / kVsRing) & 1);
      const int item = ring[rs];
      if (item < 0) break;
      const VsItem w = vs_item(item, U, a);
      const int4 un = a.units[w.unit];
      const int ha = grp ? un.z : un.x, hb = grp ? un.w : un.y;
      const bool on = ha >= 0;
      if (w.pass == 1) {
        // ---------------------------------------------------- pass 1 (thread = row)
        const int hrow = (t < 64) ? ha : hb;
        const int i = a.qrow0 + (t & 63);
        const bool active = on && hrow >= 0 && i >= a.r_lo && i < a.r_hi;
        float m = -INFINITY, ssum = 0.f;
        for (int kt = w.t_lo; kt < w.t_hi; ++kt, ++jt) {
          const int b = jt & 1;
          mbar_wait(&bars[V_SF + grp * 2 + b], (jt >> 1) & 1);
          if (on) {
            tc_fence_after();
#pragma unroll
            for (int c2 = 0; c2 < 2; ++c2) {
              uint32_t s[64];
              tmem_ld32(tbase + lane_off + b * 256 + grp * 128 + 64 * c2, *reinterpret_cast<uint32_t(*)[32]>(s));
              tmem_ld32(tbase + lane_off + b * 256 + grp * 128 + 64 * c2 + 32,
                        *reinterpret_cast<uint32_t(*)[32]>(s + 32));
              tmem_ld_wait();
              if (!active) continue;
              const int lim = i - (kt * kTile + 64 * c2);  // keep columns c <= lim
              if (lim < 63) {
#pragma unroll
                for (int u = 0; u < 64; ++u)
                  if (u > lim) s[u] = __float_as_uint(-INFINITY);
              }
              float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
              for (int u = 0; u < 64; u += 8) {
                m4[0] = fmax3(m4[0], __uint_as_float(s[u]), __uint_as_float(s[u + 1]));
                m4[1] = fmax3(m4[1], __uint_as_float(s[u + 2]), __uint_as_float(s[u + 3]));
                m4[2] = fmax3(m4[2], __uint_as_float(s[u + 4]), __uint_as_float(s[u + 5]));
                m4[3] = fmax3(m4[3], __uint_as_float(s[u + 6]), __uint_as_float(s[u + 7]));
              }
              const float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
              if (mx == -INFINITY) continue;
              const float mn = fmaxf(m, mx * sl2);
              const float2 sc2 = make_float2(sl2, sl2), mo2 = make_float2(-mn, -mn);
              float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                               make_float2(0.f, 0.f)};
#pragma unroll
              for (int u = 0; u < 64; u += 2) {
                const float2 x = ffma2(make_float2(__uint_as_float(s[u]), __uint_as_float(s[u + 1])), sc2, mo2);
                acc[(u >> 1) & 3] = fadd2(acc[(u >> 1) & 3], exp2_mix<3>(x, u >> 1));
              }
              const float2 a01 = fadd2(acc[0], acc[1]), a23 = fadd2(acc[2], acc[3]);
              ssum = ssum * fast_exp2(m - mn) + ((a01.x + a01.y) + (a23.x + a23.y));
              m = mn;
            }
          }
          tc_fence_before();
          mbar_arrive(&bars[V_SE + grp * 2 + b]);
        }
        // per-(chunk, row) statistics; both slots always write (unscored rows: (-inf, 0))
        a.stats[((size_t)w.unit * a.c1 + w.chunk) * 256 + grp * 128 + t] = make_float2(m, ssum);
        // zero this chunk's range of the diagonal output (and the column tail
        // beyond the scored keys) for the unit's heads: pass 2 adds into them
        {
          const int o_lo = w.t_lo * kTile;
          int o_hi = min(a.n, w.t_hi * kTile);
          if (w.t_hi == a.nkt) o_hi = a.n;
          const int tid = threadIdx.x;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int h = q == 0 ? un.x : (q == 1 ? un.y : (q == 2 ? un.z : un.w));
            if (h < 0) continue;
            float* dd = a.diag_dst + (size_t)h * a.n;
            for (int o = o_lo + tid; o < o_hi; o += kVsSoft) dd[o] = 0.f;
            if (!a.accumulate && w.t_hi == a.nkt) {
              float* cc = a.col_out + (size_t)h * a.n;
              for (int j = a.nkt * kTile + tid; j < a.n; j += kVsSoft) cc[j] = 0.f;
            }
          }
        }
        named_bar_sync(1, kVsSoft);
        const int g1 = w.chunk / kVsGroup;
        const int ngrp = (a.c1 + kVsGroup - 1) / kVsGroup;
        if (threadIdx.x == 0) {  // barrier, then one gpu-scope fence + atomic (release pattern)
          __threadfence();
          const int gsz = min(kVsGroup, a.c1 - g1 * kVsGroup);
          flag[0] = atomicAdd(&a.grp_done[w.unit * kVsGroup + g1], 1) == gsz - 1;
        }
        named_bar_sync(1, kVsSoft);
        if (flag[0]) {
          // first-level merge of the group's chunks (fixed order), thread = row
          const int tid = threadIdx.x;
          // (all loads in flight at once, then the fixed-order merge)
          const int c0 = g1 * kVsGroup, cn = min(a.c1, c0 + kVsGroup) - c0;
          float2 v[kVsGroup];
#pragma unroll
          for (int c = 0; c < kVsGroup; ++c)
            v[c] = c < cn ? __ldcg(&a.stats[((size_t)w.unit * a.c1 + c0 + c) * 256 + tid])
                          : make_float2(-INFINITY, 0.f);
          float2 acc = make_float2(-INFINITY, 0.f);
#pragma unroll
          for (int c = 0; c < kVsGroup; ++c) acc = merge_stat(acc, v[c]);
          a.stats2[((size_t)w.unit * kVsGroup + g1) * 256 + tid] = acc;
          named_bar_sync(1, kVsSoft);
          if (threadIdx.x == 0) {
            __threadfence();
            flag[1] = atomicAdd(&a.unit_done[w.unit], 1) == ngrp - 1;
          }
          named_bar_sync(1, kVsSoft);
          if (flag[1]) {
            float2 v2[kVsGroup];
#pragma unroll
            for (int g = 0; g < kVsGroup; ++g)
              v2[g] = g < ngrp ? __ldcg(&a.stats2[((size_t)w.unit * kVsGroup + g) * 256 + tid])
                               : make_float2(-INFINITY, 0.f);
            float2 r = make_float2(-INFINITY, 0.f);
#pragma unroll
            for (int g = 0; g < kVsGroup; ++g) r = merge_stat(r, v2[g]);
            a.lse2[(size_t)w.unit * 256 + tid] = r.y > 0.f ? r.x + log2f(r.y) : INFINITY;
            named_bar_sync(1, kVsSoft);
            if (threadIdx.x == 0) {
              __threadfence();
              st_release(&a.ready[w.unit], 1);
            }
          }
        }
      } else {
        // ---------------------------------------------------- pass 2 (thread = key)
        if (on && nl_unit != w.unit) {
          if (t == 0) {
            while (ld_relaxed(&a.ready[w.unit]) == 0) __nanosleep(64);
            __threadfence();  // acquire: the statistics written before the release
          }
          named_bar_sync(2 + grp, 128);
          nl[t] = -__ldcg(a.lse2 + (size_t)w.unit * 256 + grp * 128 + t);
          named_bar_sync(2 + grp, 128);
          nl_unit = w.unit;
        }
        for (int kt = w.t_lo; kt < w.t_hi; ++kt, ++jt) {
          const int b = jt & 1;
          mbar_wait(&bars[V_SF + grp * 2 + b], (jt >> 1) & 1);
          if (on) {
            tc_fence_after();
            const int j = kt * kTile + t;
            const int obase = a.qrow0 - kt * kTile - 127;
            const float2 sc2 = make_float2(sl2, sl2);
#pragma unroll
            for (int hi = 0; hi < 2; ++hi) {
              const int h = hi ? hb : ha;
              if (h < 0) continue;
              // R[jj]: this lane's partial of diagonal op = lane + 16 jj + 96 - 32 p
              float R[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
              float2 cs = make_float2(0.f, 0.f);
#pragma unroll
              for (int qh = 0; qh < 2; ++qh) {
                uint32_t s[32];
                tmem_ld32(tbase + lane_off + b * 256 + grp * 128 + hi * 64 + qh * 32, s);
                float nlq[32];  // broadcast reads of this quarter's -lse2
#pragma unroll
                for (int c = 0; c < 32; c += 4) {
                  const float4 v = *reinterpret_cast<const float4*>(nl + hi * 64 + qh * 32 + c);
                  nlq[c] = v.x;
                  nlq[c + 1] = v.y;
                  nlq[c + 2] = v.z;
                  nlq[c + 3] = v.w;
                }
                tmem_ld_wait();
                // rows of this quarter: frame rows 32 qh + c, global qrow0 + 32 qh + c; causal j <= i
                const int cmin = j - (a.qrow0 + 32 * qh);  // rows c >= cmin see key j
                const bool cut = __any_sync(0xffffffffu, cmin > 0);
                float wv[32];
#pragma unroll
                for (int c = 0; c < 32; c += 2) {
                  const float2 x = ffma2(make_float2(__uint_as_float(s[c]), __uint_as_float(s[c + 1])), sc2,
                                         make_float2(nlq[c], nlq[c + 1]));
                  float2 e = make_float2(fast_exp2(x.x), fast_exp2(x.y));
                  if (cut) {
                    e.x = c >= cmin ? e.x : 0.f;
                    e.y = c + 1 >= cmin ? e.y : 0.f;
                  }
                  cs = fadd2(cs, e);
                  wv[c] = e.x;
                  wv[c + 1] = e.y;
                }
                // two 16-row blocks through this warp's 16 x 32 buffer: lane l
                // writes key l of each row; the rotated read (row s, key
                // (s + 31 - lane) & 31) gives diagonal lane (s <= lane) or
                // lane + 32 (s > lane) of the block, bank-conflict free
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                  __syncwarp();
#pragma unroll
                  for (int c = 0; c < 16; ++c) Dw[c * 32 + lane] = wv[16 * e + c];
                  __syncwarp();
                  float A = 0.f, B = 0.f;
#pragma unroll
                  for (int sr = 0; sr < 16; ++sr) {
                    const float v = Dw[sr * 32 + ((sr + 31 - lane) & 31)];
                    if (sr <= lane) A += v;
                    else B += v;
                  }
                  R[2 * qh + e] += A;
                  R[2 * qh + e + 2] += B;
                }
              }
              if (j < a.n) {
                float* dst = a.col_out + (size_t)h * a.n + j;
                const float tot = cs.x + cs.y;
                *dst = a.accumulate ? (*dst + tot) : tot;
              }
              // the four warps' partials meet in C (double-buffered per head)
              float* Cb = sC + (cbuf & 1) * 768;
              ++cbuf;
#pragma unroll
              for (int jj = 0; jj < 6; ++jj) Cb[(pw * 6 + jj) * 32 + lane] = R[jj];
              named_bar_sync(2 + grp, 128);
              float* dd = a.diag_dst + (size_t)h * a.n;
#pragma unroll
              for (int k2 = 0; k2 < 2; ++k2) {
                const int op = t + 128 * k2;
                if (op > 190) break;
                float v = 0.f;
#pragma unroll
                for (int p2 = 0; p2 < 4; ++p2) {
                  const int x = op - 96 + 32 * p2;  // = lane' + 16 jj'
                  if (x < 0) continue;
                  const int j1 = x >> 4;
                  if (j1 - 1 >= 0 && j1 - 1 < 6) v += Cb[(p2 * 6 + j1 - 1) * 32 + (x - 16 * (j1 - 1))];
                  if (j1 < 6) v += Cb[(p2 * 6 + j1) * 32 + (x - 16 * j1)];
                }
                const int o = obase + op;
                if (o >= 0 && o < a.n) red_add(dd + o, v);
              }
            }
          }
          tc_fence_before();
          mbar_arrive(&bars[V_SE + grp * 2 + b]);
        }
      }
      // ring entry released only now: the producer claims at most one item ahead
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[V_IE + rs]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) tmem_dealloc(tbase, 512);
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

static void tail_chunking(int r_hi, int* nkt, int* t1, int* c1, int* t2, int* c2) {
  *nkt = (r_hi + kTile - 1) / kTile;
  *t1 = std::max(2, (*nkt + kVsMaxChunks - 1) / kVsMaxChunks);
  *c1 = (*nkt + *t1 - 1) / *t1;
  *t2 = 2;
  *c2 = (*nkt + *t2 - 1) / *t2;
}

// pass-1 blocks between a unit's pass 1 and its pass 2: enough that the grid's
// claimed-but-unfinished window (~2 items per CTA) lies inside later units' pass 1
static int tail_lookahead(int c1, int sms) {
  static const int env = [] {
    const char* e = getenv("SA_VS_LOOK");  // A/B override
    return e ? atoi(e) : 0;
  }();
  if (env > 0) return env;
  return std::max(1, std::min(4, (2 * sms + c1 - 1) / c1));
}

static int sched_ints(int hh_total) { return 1 + hh_total * (kVsGroup + 2); }

// workspace of one estimator call: statistics, queue state, unit lists and
// (when rows > 64 or accumulate is possible) the scratch diagonal
size_t tail_workspace_bytes(int hh_total, int n, int r_hi) {
  int nkt, t1, c1, t2, c2;
  tail_chunking(r_hi, &nkt, &t1, &c1, &t2, &c2);
  const size_t U = hh_total;
  return align256(U * c1 * 256 * sizeof(float2)) + align256(U * kVsGroup * 256 * sizeof(float2)) +
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
  tail_chunking(r_hi, &a.nkt, &a.t1, &a.c1, &a.t2, &a.c2);
  a.look = tail_lookahead(a.c1, device_sm_count());
  a.scale_log2 = scale * 1.4426950408889634f;
  if (ws_bytes < tail_workspace_bytes(a.hh_total, n, r_hi))
    return fail(SA_ERR_DIMENSION, "score_tail workspace too small");
  const size_t U = a.hh_total;
  char* w = reinterpret_cast<char*>(ws);
  a.stats = reinterpret_cast<float2*>(w);
  w += align256(U * a.c1 * 256 * sizeof(float2));
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
  a.next = sched;
  a.grp_done = sched + 1;
  a.unit_done = sched + 1 + a.hh_total * kVsGroup;
  a.ready = a.unit_done + a.hh_total;
  a.col_out = col_out;
  a.diag_dst = accumulate ? dtmp : diag_out;
  a.accumulate = accumulate;
  a.units = units;
  a.unit_count = list + 1;
  build_units_kernel<<<1, 1024, 0, st>>>(gate, gate_val, a.hh_total, heads, kv_heads, units, list + 1, list + 2,
                                          list, sched, sched_ints(a.hh_total));
  if ((rc = check_launch("build_units_kernel"))) return rc;
  static std::atomic<uint64_t> attr_done{0};
  once_per_device(attr_done, [] {
    cudaFuncSetAttribute(vs_estimator_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kVsSmemBytes);
  });
  const long long max_items = (long long)a.hh_total * (a.c1 + a.c2);
  const int grid = (int)std::min<long long>(device_sm_count(), max_items);
  vs_estimator_kernel<<<grid, kVsThreads, kVsSmemBytes, st>>>(a);
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
