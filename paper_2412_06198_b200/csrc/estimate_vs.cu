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
//   pass 2: merge the chunk stats, recompute S, w = exp2(s*c - lse2), then a
//           skewed shared-memory transpose turns rows into column sums and
//           per-tile diagonal partials; a final deterministic pass adds the
//           (<= 3) per-tile partials of each diagonal in key order.
// Work is split over (key-tile chunk, head); heads whose family != gate_val
// exit at once, so one launch serves the device-selected VS heads of a layer.
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
  CUtensorMap tmap_q;  // [HH, n, 128]
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
};

constexpr int kTailThreads = 192;
constexpr int kWStride = 129;  // padded row stride of the W transpose buffer
constexpr int kTailSmemQ = 0;
constexpr int kTailSmemK = 32768;       // two 32 KB K slots
constexpr int kTailSmemW = 98304;       // 128 x 129 floats
constexpr int kTailSmemBar = kTailSmemW + 128 * kWStride * 4;
constexpr int kTailSmemBytes = kTailSmemBar + 256 + 1024;

enum TBar { T_Q = 0, T_QE, T_KF0, T_KF1, T_KE0, T_KE1, T_SF0, T_SF1, T_SE0, T_SE1, T_NUM };

__device__ __forceinline__ int tail_count(const TailArgs& a) {
  return a.head_count ? *a.head_count : a.hh_total;
}
__device__ __forceinline__ int tail_head(const TailArgs& a, int rank) {
  return a.head_list ? a.head_list[rank] : rank;
}

// Persistent: one CTA per SM walks the work items (scored head, chunk of
// chunk_tiles key tiles) with a grid stride; barrier phases run on across
// items (jg counts every key tile this CTA has processed).
template <int PASS>
__global__ void __launch_bounds__(kTailThreads, 1) tail_kernel(const __grid_constant__ TailArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int n_items = tail_count(a) * a.nchunks;
  if ((int)blockIdx.x >= n_items) return;

  uint8_t* sQ = smem + kTailSmemQ;
  uint8_t* sK = smem + kTailSmemK;
  float* sW = reinterpret_cast<float*>(smem + kTailSmemW);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kTailSmemBar);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + T_NUM);
  const int warp = warp_id();

  if (threadIdx.x == 0) {
    mbar_init(&bars[T_Q], 1);
    mbar_init(&bars[T_QE], 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bars[T_KF0 + s], 1);
      mbar_init(&bars[T_KE0 + s], 1);
      mbar_init(&bars[T_SF0 + s], 1);
      mbar_init(&bars[T_SE0 + s], 128);
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
      int jg = 0, it = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
        const int hh = tail_head(a, item / a.nchunks);
        const int chunk = item % a.nchunks;
        const int kt_lo = chunk * a.chunk_tiles;
        const int kt_hi = min(a.nkt, kt_lo + a.chunk_tiles);
        const int hkv = (hh / a.heads) * a.kv_heads + (hh % a.heads) / (a.heads / a.kv_heads);
        if (it > 0) mbar_wait(&bars[T_QE], (it - 1) & 1);  // previous item's MMAs have read Q
        mbar_arrive_expect_tx(&bars[T_Q], 32768);
        tma_load_3d(sQ, &a.tmap_q, &bars[T_Q], 0, a.s0, hh);
        tma_load_3d(sQ + 16384, &a.tmap_q, &bars[T_Q], 64, a.s0, hh);
        for (int kt = kt_lo; kt < kt_hi; ++kt, ++jg) {
          const int slot = jg & 1;
          if (jg >= 2) mbar_wait(&bars[T_KE0 + slot], ((jg >> 1) - 1) & 1);
          uint8_t* dst = sK + slot * 32768;
          mbar_arrive_expect_tx(&bars[T_KF0 + slot], 32768);
          tma_load_3d(dst, &a.tmap_k, &bars[T_KF0 + slot], 0, kt * kTile, hkv);
          tma_load_3d(dst + 16384, &a.tmap_k, &bars[T_KF0 + slot], 64, kt * kTile, hkv);
        }
      }
    }
  } else if (warp == 5) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16_f32(128, 128, 0, 0);
      const uint32_t q_addr = smem_u32(sQ);
      int jg = 0, it = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
        const int chunk = item % a.nchunks;
        const int kt_lo = chunk * a.chunk_tiles;
        const int kt_hi = min(a.nkt, kt_lo + a.chunk_tiles);
        mbar_wait(&bars[T_Q], it & 1);
        tc_fence_after();
        for (int kt = kt_lo; kt < kt_hi; ++kt, ++jg) {
          const int slot = jg & 1;
          mbar_wait(&bars[T_KF0 + slot], (jg >> 1) & 1);
          if (jg >= 2) mbar_wait(&bars[T_SE0 + slot], ((jg >> 1) - 1) & 1);
          tc_fence_after();
          const uint32_t k_addr = smem_u32(sK + slot * 32768);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
            mma_ss(tbase + slot * 128, sdesc_sw128(q_addr + off, 16, 1024),
                   sdesc_sw128(k_addr + off, 16, 1024), idesc, kk > 0 ? 1u : 0u);
          }
          mma_commit(&bars[T_KE0 + slot]);
          mma_commit(&bars[T_SF0 + slot]);
        }
        mma_commit(&bars[T_QE]);
      }
    }
  } else {
    const int t = threadIdx.x;  // lane / Q-box row
    const int i = a.s0 + t;     // global query row
    const bool active = (i >= a.r_lo) && (i < a.r_hi);
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    const float sl2 = a.scale_log2;
    const int t_lo = a.r_lo - a.s0, t_hi = a.r_hi - a.s0;
    int jg = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int hh = tail_head(a, item / a.nchunks);
      const int chunk = item % a.nchunks;
      const int kt_lo = chunk * a.chunk_tiles;
      const int kt_hi = min(a.nkt, kt_lo + a.chunk_tiles);
      float m = -INFINITY, ssum = 0.f, lse2 = 0.f;
      if (PASS == 2 && active) lse2 = a.lse2[(size_t)hh * 128 + t];
      for (int kt = kt_lo; kt < kt_hi; ++kt, ++jg) {
        const int slot = jg & 1;
        const int j0 = kt * kTile;
        mbar_wait(&bars[T_SF0 + slot], (jg >> 1) & 1);
        tc_fence_after();
        uint32_t s[4][32];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32(tbase + lane_off + slot * 128 + 32 * c, s[c]);
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&bars[T_SE0 + slot]);
        const int lim = i - j0;  // keep columns c <= lim
        if (PASS == 1) {
          if (active) {
            float mx = -INFINITY;
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
              for (int u = 0; u < 32; ++u)
                if (32 * c + u <= lim) mx = fmaxf(mx, __uint_as_float(s[c][u]));
            if (mx > -INFINITY) {
              const float mn = fmaxf(m, mx * sl2);
              float acc = 0.f;
#pragma unroll
              for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int u = 0; u < 32; ++u)
                  if (32 * c + u <= lim) acc += fast_exp2(fmaf(__uint_as_float(s[c][u]), sl2, -mn));
              ssum = ssum * fast_exp2(m - mn) + acc;
              m = mn;
            }
          }
        } else {
          float* wrow = sW + t * kWStride;
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int u = 0; u < 32; ++u) {
              const int cc = 32 * c + u;
              float w = 0.f;
              if (active && cc <= lim) w = fast_exp2(fmaf(__uint_as_float(s[c][u]), sl2, -lse2));
              wrow[cc] = w;
            }
          named_bar_sync(1, 128);
          // column sums: thread t owns column j0 + t
          {
            float acc = 0.f;
            for (int r = t_lo; r < t_hi; ++r) acc += sW[r * kWStride + t];
            float* dst = a.col_out + (size_t)hh * a.n + j0 + t;
            if (j0 + t < a.n) *dst = a.accumulate ? (*dst + acc) : acc;
          }
          // diagonal partials: local offset op in [0, 256): c = (r - t_lo) + 127 - op
          float* dp = a.dpart + ((size_t)hh * a.nkt + kt) * 256;
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            const int op = t + 128 * half;
            float acc = 0.f;
            for (int r = t_lo; r < t_hi; ++r) {
              const int c = (r - t_lo) + 127 - op;
              if (c >= 0 && c < 128) acc += sW[r * kWStride + c];
            }
            dp[op] = acc;
          }
          named_bar_sync(1, 128);
        }
      }
      if (PASS == 1) {
        a.stats[((size_t)hh * a.nchunks + chunk) * 128 + t] = make_float2(m, ssum);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) tmem_dealloc(tbase, 256);
}

// Merge the per-chunk (max2, sum) row statistics into log2-sum-exp: one warp per
// (scored head, row), lanes stride over the chunks, then a shuffle merge.
__global__ void tail_merge_kernel(TailArgs a) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= tail_count(a) * 128) return;
  const int hh = tail_head(a, gw / 128), t = gw % 128;
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

// Ascending list of the heads whose gate equals gate_val (one CTA, ballot compaction).
__global__ void gate_list_kernel(const int32_t* gate, int gate_val, int hh_total, int32_t* list,
                                 int32_t* count) {
  __shared__ int base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  for (int h0 = 0; h0 < hh_total; h0 += blockDim.x) {
    const int h = h0 + threadIdx.x;
    const bool on = h < hh_total && gate[h] == gate_val;
    const uint32_t bal = __ballot_sync(0xffffffffu, on);
    __shared__ int wsum[32];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) wsum[w] = __popc(bal);
    __syncthreads();
    int before = base;
    for (int x = 0; x < w; ++x) before += wsum[x];
    if (on) list[before + __popc(bal & ((1u << lane) - 1u))] = h;
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int x = 0; x < (int)(blockDim.x >> 5); ++x) tot += wsum[x];
      base += tot;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = base;
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

size_t tail_workspace_bytes(int hh_total, int n, int r_hi, int nchunks) {
  const int nkt = (r_hi + kTile - 1) / kTile;
  return align256((size_t)hh_total * nchunks * 128 * sizeof(float2)) +
         align256((size_t)hh_total * nkt * 256 * 4) + align256((size_t)hh_total * 128 * 4) +
         align256((size_t)(hh_total + 1) * 4) + 256;
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
  int32_t* list = reinterpret_cast<int32_t*>(w);
  a.col_out = col_out;
  a.accumulate = accumulate;
  a.head_list = nullptr;
  a.head_count = nullptr;
  if (gate) {
    gate_list_kernel<<<1, 1024, 0, st>>>(gate, gate_val, a.hh_total, list + 1, list);
    if ((rc = check_launch("gate_list_kernel"))) return rc;
    a.head_list = list + 1;
    a.head_count = list;
  }
  if (!accumulate) {
    // columns past the last scored row never receive mass
    cudaMemsetAsync(col_out, 0, (size_t)a.hh_total * n * sizeof(float), st);
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tail_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTailSmemBytes);
    cudaFuncSetAttribute(tail_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTailSmemBytes);
    attr = true;
  }
  static int num_sms = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  const int grid = std::min(num_sms, a.hh_total * a.nchunks);
  tail_kernel<1><<<grid, kTailThreads, kTailSmemBytes, st>>>(a);
  if ((rc = check_launch("tail_kernel<1>"))) return rc;
  tail_merge_kernel<<<(a.hh_total * 128 * 32 + 255) / 256, 256, 0, st>>>(a);
  if ((rc = check_launch("tail_merge_kernel"))) return rc;
  tail_kernel<2><<<grid, kTailThreads, kTailSmemBytes, st>>>(a);
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
