// estimate_vs.cu — the vertical-slash pattern estimator on tcgen05.
//
// Reference: patterns.py:165-202 (_tail_weights, _column_scores,
// _diagonal_scores) and patterns.py:237-259 (build_vertical_slash_index).
// For each selected head, the last R (<= 128) query rows [r_lo, r_hi) are
// scored against every causal key: w = softmax_row(q_i . k_j * scale) over
// j <= i, then
//     col[j]  = sum_i w[i, j]            (column mass)
//     diag[o] = sum_i w[i, i - o]        (diagonal mass, o >= 0).
// Row statistics need every key before any weight is final, so the estimator
// is two streaming passes over K (the second mostly L2-resident):
//   pass 1: S = Q_tail K_tile^T in TMEM -> per-(row, chunk) online (max, sum)
//   pass 2: merge the chunk stats, recompute S^T (keys on TMEM lanes),
//           w = exp2(s*c - lse2); each key's column sum is a register sum,
//           the weights go to a skewed shared-memory buffer whose columns
//           are the tile's diagonals; a final deterministic pass adds the
//           (<= 3) per-tile partials of each diagonal in key order.
// Work is split over (unit = one head or a GQA pair of heads, key-tile chunk)
// of a device-built list of the heads whose family == gate_val, so one launch
// serves the device-selected VS heads of a layer.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <algorithm>

#include "api_common.h"
#include "internal.h"
#include "sa_types.h"
#include "sm100_common.cuh"

namespace sa {

struct TailArgs {
  CUtensorMap tmap_q;  // [HH, n, 128], box rows 128 (single) or 64 (paired)
  CUtensorMap tmap_k;  // [HK, n, 128]
  int n, heads, kv_heads, hh_total;
  int r_lo, r_hi;      // scored rows (global indices), r_hi - r_lo <= 128
  int s0;              // first row of the Q box (lane 0)
  int nkt;             // key tiles with any causal key: ceil(r_hi / 128)
  int chunk_tiles;     // key tiles per work item
  int nchunks;
  float scale_log2;
  float2* stats;       // [HH, nchunks, 128] (max2, sum) per lane
  float* lse2;         // [HH, 128] merged log2-sum-exp per row (pass 2 input)
  float* col_out;      // [HH, n]
  float* dpart;        // [HH, nkt, 256] per-tile diagonal partials
  int accumulate;      // add into col_out (multi-group exact scoring)
  const int32_t* head_list;   // optional: the scored heads (ascending), else all heads
  const int32_t* head_count;  // device count of head_list
  // work units: paired (R <= 64): two heads sharing a kv head stack their 64
  // tail rows in one M=128 MMA box (rows 0-63 head A, 64-127 head B, B may be
  // -1); single: one head, rows in the last R lanes of the 128-row box
  int paired;
  const int2* units;          // optional unit list (device), else unit u = head u
  const int32_t* unit_count;  // device count of units
};

// warps 0-7: two per TMEM lane quarter (pass 1: warp / 4 = half of each row's
// 128 keys; pass 2: warp / 4 = which half of the box's rows, keys on lanes);
// warp 8: TMA producer; warp 9: MMA issuer
constexpr int kTailThreads = 320;
constexpr int kTailSoft = 256;
constexpr int kTailSmemQ = 0;
constexpr int kTailKSlots = 4;  // barrier slots; pass 1 streams K through 4 x 32 KB, pass 2 through 2
constexpr int kTailSmemK = 32768;
// pass 1: K ring (4 slots) + a 1 KB statistics exchange; pass 2: K ring
// (2 slots) + the skewed diagonal buffer D[128 rows][256 offsets] fp32 +
// a 512 B column-sum exchange
__host__ __device__ constexpr int tail_slots(int pass) { return pass == 1 ? 4 : 2; }
__host__ __device__ constexpr int tail_smem_x(int pass) { return kTailSmemK + tail_slots(pass) * 32768; }
constexpr int kDStride = 256;
__host__ __device__ constexpr int tail_smem_bar(int pass) {
  return tail_smem_x(pass) + (pass == 1 ? 1024 : 128 * kDStride * 4 + 512);
}
__host__ __device__ constexpr int tail_smem_bytes(int pass) { return tail_smem_bar(pass) + 256 + 1024; }

enum TBar { T_Q = 0, T_QE, T_KF0, T_KE0 = T_KF0 + kTailKSlots, T_SF0 = T_KE0 + kTailKSlots, T_SF1,
            T_SE0, T_SE1, T_NUM };

__device__ __forceinline__ int tail_count(const TailArgs& a) {
  return a.head_count ? *a.head_count : a.hh_total;
}
__device__ __forceinline__ int unit_count(const TailArgs& a) {
  return a.unit_count ? *a.unit_count : a.hh_total;
}
__device__ __forceinline__ int2 unit_at(const TailArgs& a, int u) {
  return a.units ? a.units[u] : make_int2(u, -1);
}
__device__ __forceinline__ int tail_head(const TailArgs& a, int rank) {
  return a.head_list ? a.head_list[rank] : rank;
}

// Persistent: one CTA per SM walks the work items (unit, chunk of chunk_tiles
// key tiles) with a grid stride; barrier phases run on across items (jg counts
// every key tile this CTA has processed).  A paired unit reads each K tile once
// for two heads of the same kv head and keeps all four softmax warps busy.
template <int PASS>
__global__ void __launch_bounds__(kTailThreads, 1) tail_kernel(const __grid_constant__ TailArgs a) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-aligned offset into the dynamic shared array (pointer arithmetic on
  // smem_raw keeps the shared address space, so accesses compile to LDS/STS)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int n_items = unit_count(a) * a.nchunks;
  if ((int)blockIdx.x >= n_items) return;

  uint8_t* sQ = smem + kTailSmemQ;
  uint8_t* sK = smem + kTailSmemK;
  constexpr int kSlots = tail_slots(PASS);
  float* sX = reinterpret_cast<float*>(smem + tail_smem_x(PASS));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + tail_smem_bar(PASS));
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + T_NUM);
  const int warp = warp_id();

  if (threadIdx.x == 0) {
    mbar_init(&bars[T_Q], 1);
    mbar_init(&bars[T_QE], 1);
    for (int s = 0; s < kTailKSlots; ++s) {
      mbar_init(&bars[T_KF0 + s], 1);
      mbar_init(&bars[T_KE0 + s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bars[T_SF0 + s], 1);
      mbar_init(&bars[T_SE0 + s], kTailSoft);
    }
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc(tmem_holder, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_holder;

  // Consecutive items of a CTA usually belong to the same unit (head pair):
  // its Q box is loaded once and reused (qn counts Q loads; the MMA warp
  // releases Q after the last item of the unit).
  if (warp == 8) {
    if (elect_one()) {
      int jg = 0, qn = 0, prev_unit = -1;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int unit = item / a.nchunks;
        const int2 un = unit_at(a, unit);
        const int chunk = item % a.nchunks;
        const int kt_lo = chunk * a.chunk_tiles;
        const int kt_hi = min(a.nkt, kt_lo + a.chunk_tiles);
        const int hh = un.x;
        const int hkv = (hh / a.heads) * a.kv_heads + (hh % a.heads) / (a.heads / a.kv_heads);
        if (unit != prev_unit) {
          if (qn > 0) mbar_wait_backoff<64>(&bars[T_QE], (qn - 1) & 1);  // MMAs of the last unit have read Q
          mbar_arrive_expect_tx(&bars[T_Q], 32768);
          if (a.paired) {
            const int hb = un.y >= 0 ? un.y : un.x;  // a lone head fills the B half (rows inactive)
            tma_load_3d(sQ, &a.tmap_q, &bars[T_Q], 0, a.r_hi - 64, hh);
            tma_load_3d(sQ + 8192, &a.tmap_q, &bars[T_Q], 0, a.r_hi - 64, hb);
            tma_load_3d(sQ + 16384, &a.tmap_q, &bars[T_Q], 64, a.r_hi - 64, hh);
            tma_load_3d(sQ + 24576, &a.tmap_q, &bars[T_Q], 64, a.r_hi - 64, hb);
          } else {
            tma_load_3d(sQ, &a.tmap_q, &bars[T_Q], 0, a.s0, hh);
            tma_load_3d(sQ + 16384, &a.tmap_q, &bars[T_Q], 64, a.s0, hh);
          }
          ++qn;
          prev_unit = unit;
        }
        for (int kt = kt_lo; kt < kt_hi; ++kt, ++jg) {
          const int slot = jg % kSlots;
          if (jg >= kSlots) mbar_wait_backoff<64>(&bars[T_KE0 + slot], ((jg / kSlots) - 1) & 1);
          uint8_t* dst = sK + slot * 32768;
          mbar_arrive_expect_tx(&bars[T_KF0 + slot], 32768);
          tma_load_3d(dst, &a.tmap_k, &bars[T_KF0 + slot], 0, kt * kTile, hkv);
          tma_load_3d(dst + 16384, &a.tmap_k, &bars[T_KF0 + slot], 64, kt * kTile, hkv);
        }
      }
    }
  } else if (warp == 9) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16_f32(128, 128, 0, 0);
      const uint32_t q_addr = smem_u32(sQ);
      int jg = 0, qn = 0, prev_unit = -1;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int unit = item / a.nchunks;
        const int chunk = item % a.nchunks;
        const int kt_lo = chunk * a.chunk_tiles;
        const int kt_hi = min(a.nkt, kt_lo + a.chunk_tiles);
        if (unit != prev_unit) {
          mbar_wait_backoff<16>(&bars[T_Q], qn & 1);
          ++qn;
          prev_unit = unit;
        }
        tc_fence_after();
        for (int kt = kt_lo; kt < kt_hi; ++kt, ++jg) {
          const int slot = jg % kSlots, sbuf = jg & 1;
          mbar_wait_backoff<16>(&bars[T_KF0 + slot], (jg / kSlots) & 1);
          if (jg >= 2) mbar_wait_backoff<16>(&bars[T_SE0 + sbuf], ((jg >> 1) - 1) & 1);
          tc_fence_after();
          const uint32_t k_addr = smem_u32(sK + slot * 32768);
          // pass 1: S (rows on TMEM lanes); pass 2: S^T (keys on lanes, rows on columns)
          const uint32_t a_addr = PASS == 1 ? q_addr : k_addr, b_addr = PASS == 1 ? k_addr : q_addr;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
            mma_ss(tbase + sbuf * 128, sdesc_sw128(a_addr + off, 16, 1024),
                   sdesc_sw128(b_addr + off, 16, 1024), idesc, kk > 0 ? 1u : 0u);
          }
          mma_commit(&bars[T_KE0 + slot]);
          mma_commit(&bars[T_SF0 + sbuf]);
        }
        const int nxt = item + (int)gridDim.x;
        if (nxt >= n_items || nxt / a.nchunks != unit) mma_commit(&bars[T_QE]);  // last item of the unit
      }
    }
  } else if (PASS == 1) {
    // ---------------------------------------------------------- pass 1
    const int t = threadIdx.x & 127;  // TMEM lane = row of the MMA box
    const int cpart = warp >> 2;      // this thread's half of the row's 128 keys
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const float sl2 = a.scale_log2;
    // rows of this thread: paired -> head half t >> 6, row r_hi - 64 + (t & 63),
    // stats lane 64 + (t & 63); single -> row s0 + t, stats lane t
    const int i = a.paired ? a.r_hi - 64 + (t & 63) : a.s0 + t;
    const int slane = a.paired ? 64 + (t & 63) : t;
    int jg = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int2 un = unit_at(a, item / a.nchunks);
      const int hh = (a.paired && t >= 64) ? un.y : un.x;
      const bool active = hh >= 0 && i >= a.r_lo && i < a.r_hi;
      const int chunk = item % a.nchunks;
      const int kt_lo = chunk * a.chunk_tiles;
      const int kt_hi = min(a.nkt, kt_lo + a.chunk_tiles);
      float m = -INFINITY, ssum = 0.f;
      for (int kt = kt_lo; kt < kt_hi; ++kt, ++jg) {
        const int slot = jg & 1;
        const int j0 = kt * kTile + 64 * cpart;  // first key of this thread's half
        mbar_wait(&bars[T_SF0 + slot], (jg >> 1) & 1);
        tc_fence_after();
        uint32_t s[2][32];
#pragma unroll
        for (int c = 0; c < 2; ++c) tmem_ld32(tbase + lane_off + slot * 128 + 64 * cpart + 32 * c, s[c]);
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&bars[T_SE0 + slot]);
        if (!active) continue;
        const int lim = i - j0;  // keep columns c <= lim
        if (lim < 63) {  // causal cut (the diagonal tile only)
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int u = 0; u < 32; ++u)
              if (32 * c + u > lim) s[c][u] = __float_as_uint(-INFINITY);
        }
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int u = 0; u < 32; u += 4) {
            m4[2 * c] = fmax3(m4[2 * c], __uint_as_float(s[c][u]), __uint_as_float(s[c][u + 1]));
            m4[2 * c + 1] = fmax3(m4[2 * c + 1], __uint_as_float(s[c][u + 2]), __uint_as_float(s[c][u + 3]));
          }
        const float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
        if (mx == -INFINITY) continue;  // no causal key of this row in the half tile
        const float mn = fmaxf(m, mx * sl2);
        const float2 sc2 = make_float2(sl2, sl2), mo2 = make_float2(-mn, -mn);
        float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int u = 0; u < 32; u += 2) {
            // (MUFU only: the scores feed a bit-exact top-k, keep them at ex2.approx accuracy)
            float2 x = ffma2(make_float2(__uint_as_float(s[c][u]), __uint_as_float(s[c][u + 1])), sc2, mo2);
            x.x = fast_exp2(x.x);
            x.y = fast_exp2(x.y);
            acc[(u >> 1) & 1] = fadd2(acc[(u >> 1) & 1], x);
          }
        ssum = ssum * fast_exp2(m - mn) + (acc[0].x + acc[0].y + acc[1].x + acc[1].y);
        m = mn;
      }
      // statistics per (row, chunk): the key half 1 thread hands its (max, sum)
      // to the half 0 thread
      float2* xch = reinterpret_cast<float2*>(sX);
      if (cpart) xch[t] = make_float2(m, ssum);
      named_bar_sync(1, kTailSoft);
      if (!cpart && hh >= 0) {
        const float2 o = xch[t];
        const float mn = fmaxf(m, o.x);
        float sum = 0.f;
        if (mn > -INFINITY) sum = ssum * fast_exp2(m - mn) + o.y * fast_exp2(o.x - mn);
        a.stats[((size_t)hh * a.nchunks + chunk) * 128 + slane] = make_float2(mn, sum);
      }
      named_bar_sync(1, kTailSoft);
    }
  } else {
    // ---------------------------------------------------------- pass 2
    // S^T in TMEM: lane = key j0 + t of the tile, column = row of the Q box.
    // Thread (t, half hf = warp / 4) owns key t against the box rows
    // [64 hf, 64 hf + 64).  w = exp2(s * c - lse2[row]) with lse2 = +inf on rows
    // that are not scored (w = 0); the column sum of key t is a register sum;
    // the diagonal partials go through D[row][op] (skewed so a diagonal is a
    // column of D, op = (row - w_lo) + 127 - t) and are summed per column.
    const int t = threadIdx.x & 127;
    const int hf = warp >> 2;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const float sl2 = a.scale_log2;
    const int R = a.r_hi - a.r_lo;
    // the box rows of this half: row r = 64 hf + rl (rl < 64), global row i(r)
    const int ibase = a.paired ? a.r_hi - 64 : a.s0 + 64 * hf;  // global row of rl = 0
    const int w_hi = a.paired ? 64 * hf + 64 : a.r_hi - a.s0;  // box rows of the scored window
    const int w_lo = w_hi - R;
    const int rl_lo = max(0, w_lo - 64 * hf);  // scored rl of this half: [rl_lo, rl_hi)
    const int rl_hi = min(64, w_hi - 64 * hf);
    float* sD = sX;
    float* sC = sX + 128 * kDStride;  // [128] column-sum exchange (single-head units)
    int jg = 0, cur_unit = -1;
    float nl[64];
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int2 un = unit_at(a, item / a.nchunks);
      const int hx = a.paired ? (hf ? un.y : un.x) : un.x;
      const int chunk = item % a.nchunks;
      const int kt_lo = chunk * a.chunk_tiles;
      const int kt_hi = min(a.nkt, kt_lo + a.chunk_tiles);
      // -lse2 per row of this half (registers, reloaded when the unit
      // changes), -inf -> w = 0 for unscored rows
      if (item / a.nchunks != cur_unit) {
        cur_unit = item / a.nchunks;
        const int sl0 = a.paired ? 64 : 64 * hf;  // stats lane of rl = 0
        const float* src = a.lse2 + (size_t)max(hx, 0) * 128 + sl0;
        // rows outside [rl_lo, rl_hi) were never written by pass 1: not read
#pragma unroll
        for (int rl = 0; rl < 64; ++rl)
          nl[rl] = (hx >= 0 && rl >= rl_lo && rl < rl_hi) ? -src[rl] : -INFINITY;
      }
      for (int kt = kt_lo; kt < kt_hi; ++kt, ++jg) {
        const int slot = jg & 1;
        const int j = kt * kTile + t;  // this thread's key
        mbar_wait(&bars[T_SF0 + slot], (jg >> 1) & 1);
        tc_fence_after();
        uint32_t s[2][32];
#pragma unroll
        for (int c = 0; c < 2; ++c) tmem_ld32(tbase + lane_off + slot * 128 + 64 * hf + 32 * c, s[c]);
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&bars[T_SE0 + slot]);
        // causal: row rl sees key j iff ibase + rl >= j, i.e. rl >= j - ibase
        const int rl_causal = j - ibase;
        const float2 sc2 = make_float2(sl2, sl2);
        float2 cs = make_float2(0.f, 0.f);
        float w[64];
        const bool cut = __any_sync(0xffffffffu, rl_causal > 0);  // only tiles at the scored rows
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int u = 0; u < 32; u += 2) {
            const int rl = 32 * c + u;
            float2 x = ffma2(make_float2(__uint_as_float(s[c][u]), __uint_as_float(s[c][u + 1])), sc2,
                             make_float2(nl[rl], nl[rl + 1]));
            x.x = fast_exp2(x.x);
            x.y = fast_exp2(x.y);
            if (cut) {
              x.x = rl >= rl_causal ? x.x : 0.f;
              x.y = rl + 1 >= rl_causal ? x.y : 0.f;
            }
            cs = fadd2(cs, x);
            w[rl] = x.x;
            w[rl + 1] = x.y;
          }
        named_bar_sync(1, kTailSoft);  // the previous tile's D readers are done
        // D[r][op], op = (r - w_lo) + 127 - t for the scored rows r of this half
#pragma unroll
        for (int rl = 0; rl < 64; ++rl) {
          const int r = 64 * hf + rl;
          if (rl >= rl_lo && rl < rl_hi) sD[r * kDStride + (r - w_lo) + 127 - t] = w[rl];
        }
        const float csum = cs.x + cs.y;
        if (!a.paired && hf) sC[t] = csum;
        named_bar_sync(1, kTailSoft);
        const int kt0 = kt * kTile;
        if (a.paired) {
          if (hx >= 0 && j < a.n) {
            float* dst = a.col_out + (size_t)hx * a.n + j;
            *dst = a.accumulate ? (*dst + csum) : csum;
          }
        } else if (!hf && hx >= 0 && j < a.n) {
          const float tot = csum + sC[t];
          float* dst = a.col_out + (size_t)hx * a.n + j;
          *dst = a.accumulate ? (*dst + tot) : tot;
        }
        // diagonal partials: (unit half, op) tasks, op < R + 127, over the D rows
        // [r_a, r_b) holding them; 32 independent predicated loads per block
        const int nh = a.paired ? 2 : 1;
        const int nop = R + 127;
#pragma unroll 1
        for (int task = threadIdx.x; task < nh * nop; task += kTailSoft) {
          const int uh = task / nop, op = task % nop;
          const int ux = a.paired ? (uh ? un.y : un.x) : un.x;
          if (ux < 0) continue;
          const int wl = a.paired ? 64 * uh + 64 - R : w_lo;  // w_lo of that half's frame
          const int r_a = wl + max(0, op - 127), r_b = wl + min(R, op + 1);
          float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
          for (int rb = r_a; rb < r_b; rb += 32) {
#pragma unroll
            for (int u = 0; u < 32; ++u)
              if (rb + u < r_b) acc[u & 7] += sD[(rb + u) * kDStride + op];
          }
          a.dpart[((size_t)ux * a.nkt + kt) * 256 + op] =
              ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) tmem_dealloc(tbase, 256);
}

// Merge the per-chunk (max2, sum) row statistics into log2-sum-exp: one warp per
// (scored head, row), lanes stride over the chunks, then a shuffle merge.
__global__ void tail_merge_kernel(TailArgs a) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= tail_count(a) * 128) return;
  const int hh = tail_head(a, gw / 128), t = gw % 128;
  // only the lanes holding scored rows carry statistics
  if (t < (a.paired ? 128 - (a.r_hi - a.r_lo) : a.r_lo - a.s0)) return;
  const float2* st = a.stats + (size_t)hh * a.nchunks * 128 + t;
  float m = -INFINITY, s = 0.f;
  for (int c = lane; c < a.nchunks; c += 32) {
    const float2 v = st[(size_t)c * 128];
    if (v.y > 0.f) {
      const float mn = fmaxf(m, v.x);
      s = s * fast_exp2(m - mn) + v.y * fast_exp2(v.x - mn);
      m = mn;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
    const float s2 = __shfl_xor_sync(0xffffffffu, s, o);
    const float mn = fmaxf(m, m2);
    if (mn > -INFINITY) {
      s = s * fast_exp2(m - mn) + s2 * fast_exp2(m2 - mn);
      m = mn;
    }
  }
  if (lane == 0) a.lse2[(size_t)hh * 128 + t] = m + log2f(s);
}

// diag[hh][o] = sum over key tiles kt (ascending) of dpart[hh][kt][o - r_lo + 127 + 128 kt]
__global__ void diag_combine_kernel(const float* dpart, float* diag_out, int n, int nkt, int r_lo,
                                    int R, int accumulate, const int32_t* head_list,
                                    const int32_t* head_count) {
  const int rank = blockIdx.y;
  if (head_count && rank >= *head_count) return;
  const int hh = head_list ? head_list[rank] : rank;
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= n) return;
  // op = o - r_lo + 127 + 128 kt in [0, R + 127)
  int kt_a = r_lo - 127 - o;            // 128 kt >= kt_a
  int kt_b = r_lo + R - o;              // 128 kt <  kt_b
  int lo = kt_a <= 0 ? 0 : (kt_a + 127) / 128;
  int hi = kt_b <= 0 ? -1 : (kt_b - 1) / 128;
  if (hi > nkt - 1) hi = nkt - 1;
  float acc = 0.f;
  for (int kt = lo; kt <= hi; ++kt) {
    const int op = o - r_lo + 127 + 128 * kt;
    if (op >= 0 && op < 256) acc += dpart[((size_t)hh * nkt + kt) * 256 + op];
  }
  float* dst = diag_out + (size_t)hh * n + o;
  *dst = accumulate ? (*dst + acc) : acc;
}

// Scored heads and work units from the device-selected families (one CTA, a
// warp per kv group): head_list = every head whose gate equals gate_val (or
// all heads), units = consecutive pairs of those heads inside a kv group (a
// lone head pairs with -1), or one unit per head when pairing is off.
__global__ void build_units_kernel(const int32_t* gate, int gate_val, int hh_total, int heads,
                                   int kv_heads, int pair, int2* units, int32_t* unit_count,
                                   int32_t* head_list, int32_t* head_count) {
  __shared__ int n_units, n_heads;
  if (threadIdx.x == 0) n_units = n_heads = 0;
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
      const int nu = pair ? (cnt + 1) / 2 : cnt;
      if (lane == 0) {
        hb = atomicAdd(&n_heads, cnt);
        ub = atomicAdd(&n_units, nu);
      }
      hb = __shfl_sync(0xffffffffu, hb, 0);
      ub = __shfl_sync(0xffffffffu, ub, 0);
      if (on) head_list[hb + rank] = h;
      // the partner of selected rank 2p is the next selected lane
      const uint32_t above = bal & ~((2u << lane) - 1u);
      const int nxt = above ? __ffs(above) - 1 : -1;
      const int hn = __shfl_sync(0xffffffffu, h, nxt >= 0 ? nxt : lane);
      if (on && pair && (rank & 1) == 0) units[ub + rank / 2] = make_int2(h, nxt >= 0 ? hn : -1);
      else if (on && !pair) units[ub + rank] = make_int2(h, -1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *unit_count = n_units;
    *head_count = n_heads;
  }
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

size_t tail_workspace_bytes(int hh_total, int n, int r_hi, int nchunks) {
  const int nkt = (r_hi + kTile - 1) / kTile;
  return align256((size_t)hh_total * nchunks * 128 * sizeof(float2)) +
         align256((size_t)hh_total * nkt * 256 * 4) + align256((size_t)hh_total * 128 * 4) +
         align256((size_t)(hh_total + 2) * 4) + align256((size_t)hh_total * 8) + 256;
}

// two key tiles per work item: enough items to fill every SM for one VS head
int tail_pick_chunks(int r_hi) {
  const int nkt = (r_hi + kTile - 1) / kTile;
  const int nch = (nkt + 1) / 2;
  return nch < 1 ? 1 : nch;
}

// Score rows [r_lo, r_hi) (R <= 128) of every (gated) head into col/diag (fp32, [HH, n]).
int launch_score_tail(int batch, int heads, int kv_heads, int n, float scale, const void* q,
                      const void* k, int r_lo, int r_hi, float* col_out, float* diag_out,
                      int accumulate, const int32_t* gate, int gate_val, void* ws, size_t ws_bytes,
                      cudaStream_t st) {
  if (r_hi > n || r_lo < 0 || r_hi - r_lo < 1 || r_hi - r_lo > 128)
    return fail(SA_ERR_PATTERN_PARAM, "tail rows [%d, %d) invalid for n=%d", r_lo, r_hi, n);
  TailArgs a;
  memset(&a, 0, sizeof(a));
  int rc;
  if ((rc = make_tmap_3d_bf16(&a.tmap_q, q, kHeadDim, n, batch * heads, kTile))) return rc;
  if ((rc = make_tmap_3d_bf16(&a.tmap_k, k, kHeadDim, n, batch * kv_heads, kTile))) return rc;
  a.n = n;
  a.heads = heads;
  a.kv_heads = kv_heads;
  a.hh_total = batch * heads;
  a.r_lo = r_lo;
  a.r_hi = r_hi;
  a.s0 = r_hi >= kTile ? r_hi - kTile : 0;
  a.nkt = (r_hi + kTile - 1) / kTile;
  a.nchunks = tail_pick_chunks(r_hi);
  a.chunk_tiles = (a.nkt + a.nchunks - 1) / a.nchunks;
  a.scale_log2 = scale * 1.4426950408889634f;
  if (ws_bytes < tail_workspace_bytes(a.hh_total, n, r_hi, a.nchunks))
    return fail(SA_ERR_DIMENSION, "score_tail workspace too small");
  char* w = reinterpret_cast<char*>(ws);
  a.stats = reinterpret_cast<float2*>(w);
  w += align256((size_t)a.hh_total * a.nchunks * 128 * sizeof(float2));
  a.dpart = reinterpret_cast<float*>(w);
  w += align256((size_t)a.hh_total * a.nkt * 256 * 4);
  a.lse2 = reinterpret_cast<float*>(w);
  w += align256((size_t)a.hh_total * 128 * 4);
  int32_t* list = reinterpret_cast<int32_t*>(w);  // [0] head count, [1] unit count, [2..] heads
  w += align256((size_t)(a.hh_total + 2) * 4);
  int2* units = reinterpret_cast<int2*>(w);
  a.col_out = col_out;
  a.accumulate = accumulate;
  // two heads of one kv head share an M=128 box when the tail fits 64 rows
  a.paired = (r_hi - r_lo <= 64 && heads / kv_heads >= 2) ? 1 : 0;
  if (a.paired && (rc = make_tmap_3d_bf16(&a.tmap_q, q, kHeadDim, n, batch * heads, 64))) return rc;
  build_units_kernel<<<1, 1024, 0, st>>>(gate, gate_val, a.hh_total, heads, kv_heads, a.paired, units, list + 1,
                                          list + 2, list);
  if ((rc = check_launch("build_units_kernel"))) return rc;
  a.head_list = list + 2;
  a.head_count = list;
  a.units = units;
  a.unit_count = list + 1;
  if (!accumulate) {
    // columns past the last scored row never receive mass
    cudaMemsetAsync(col_out, 0, (size_t)a.hh_total * n * sizeof(float), st);
  }
  static std::atomic<uint64_t> attr_done{0};
  once_per_device(attr_done, [] {
    cudaFuncSetAttribute(tail_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, tail_smem_bytes(1));
    cudaFuncSetAttribute(tail_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, tail_smem_bytes(2));
  });
  const int num_sms = device_sm_count();
  const int grid = std::min(num_sms, a.hh_total * a.nchunks);
  tail_kernel<1><<<grid, kTailThreads, tail_smem_bytes(1), st>>>(a);
  if ((rc = check_launch("tail_kernel<1>"))) return rc;
  tail_merge_kernel<<<(a.hh_total * 128 * 32 + 255) / 256, 256, 0, st>>>(a);
  if ((rc = check_launch("tail_merge_kernel"))) return rc;
  tail_kernel<2><<<grid, kTailThreads, tail_smem_bytes(2), st>>>(a);
  if ((rc = check_launch("tail_kernel<2>"))) return rc;
  dim3 g2((n + 255) / 256, a.hh_total);
  diag_combine_kernel<<<g2, 256, 0, st>>>(a.dpart, diag_out, n, a.nkt, r_lo, r_hi - r_lo,
                                          accumulate, a.head_list, a.head_count);
  return check_launch("diag_combine_kernel");
}

}  // namespace sa

extern "C" size_t sa_score_tail_workspace(int batch, int heads, int n, int r_hi) {
  return sa::tail_workspace_bytes(batch * heads, n, r_hi, sa::tail_pick_chunks(r_hi));
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
