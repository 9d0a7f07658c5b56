// topk.cu — stable top-k of fp32 score rows, bit-exact with the reference's
// _top_k_stable (patterns.py:231-234): the k largest scores, ties resolved to
// the LOWER index, returned in ascending index order.
//
// Per row (one CTA): map each score to a 32-bit preference key (larger key =
// preferred; -0.0 == +0.0; NaN least preferred, matching numpy's argsort which
// sorts NaN last), radix-select the k-th largest key T with four 8-bit MSB
// passes, then one ordered compaction keeps every key > T plus the first
// (k - #{key > T}) keys == T in index order.  The result is the exact set the
// stable sort would return, independent of thread scheduling.
#include <cuda_runtime.h>

#include <cstdint>

#include "api_common.h"
#include "internal.h"
#include "sa_types.h"

namespace sa {

constexpr int kTopkThreads = 1024;
constexpr int kTopkSmemKeys = 53248;  // 208 KB of cached keys per row

__device__ __forceinline__ uint32_t pref_key(float f) {
  uint32_t b = __float_as_uint(f);
  if ((b & 0x7fffffffu) > 0x7f800000u) return 0u;  // NaN
  if ((b & 0x7fffffffu) == 0u) b = 0u;               // -0.0 -> +0.0
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// Exclusive block-wide scan of one int per thread (1024 threads).
__device__ __forceinline__ int block_excl_scan(int v, int* warp_tot, int& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = warp_tot[lane];
    int s = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    warp_tot[lane] = s - t;  // exclusive warp offsets
    if (lane == 31) warp_tot[32] = s;
  }
  __syncthreads();
  const int r = warp_tot[w] + x - v;
  total = warp_tot[32];
  __syncthreads();
  return r;
}



__global__ void __launch_bounds__(kTopkThreads) topk_rows_kernel(TopkArgs a) {
  int r = blockIdx.x;
  const float* scores = a.scores;
  int kk = a.k;
  int32_t* idx_out = a.idx_out;
  long long out_ld = a.out_ld;
  uint32_t* bits = a.bits;
  int bit_base = a.bit_base, bit_neg = a.bit_neg;
  if (a.split > 0 && r >= a.split) {
    r -= a.split;
    scores = a.scores2;
    kk = a.k2;
    idx_out = a.idx_out2;
    out_ld = a.out_ld2;
    bits = a.bits2;
    bit_base = a.bit_base2;
    bit_neg = a.bit_neg2;
  }
  if (a.gate && a.gate[r / a.gate_div] != a.gate_val) return;
  const int len = a.lens ? a.lens[r] : a.n;
  int k = a.ks ? a.ks[r] : kk;
  k = k < len ? k : len;
  const float* s = scores + (long long)r * a.ld;
  // Rows that fit are staged once into shared memory as preference keys
  // (coalesced, many loads in flight); every radix pass and the compaction
  // then read shared memory instead of re-walking global memory.
  extern __shared__ uint32_t kcache[];
  const bool cached = len <= a.smem_keys;
  if (cached) {
    for (int j0 = threadIdx.x; j0 < len; j0 += 4 * blockDim.x) {
      float v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = j0 + u * blockDim.x;
        v[u] = j < len ? s[j] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = j0 + u * blockDim.x;
        if (j < len) kcache[j] = pref_key(v[u]);
      }
    }
    __syncthreads();
  }
  auto key_at = [&](int j) -> uint32_t { return cached ? kcache[j] : pref_key(__ldg(s + j)); };
  __shared__ int hist[256];
  __shared__ int warp_tot[33];
  __shared__ uint32_t sh_digit;
  __shared__ int sh_remaining;

  uint32_t prefix = 0u, mask = 0u;
  int remaining = k;
  bool take_all = (k >= len);
  if (!take_all && k > 0) {
    for (int pass = 0; pass < 4; ++pass) {
      const int shift = 24 - 8 * pass;
      for (int t = threadIdx.x; t < 256; t += blockDim.x) hist[t] = 0;
      __syncthreads();
      // warp-aggregated histogram: scores of similar magnitude share their top
      // bits, so lanes are matched on the bin and one leader adds the count
      const int len_pad = (len + 31) & ~31;
      for (int j = threadIdx.x; j < len_pad; j += blockDim.x) {
        const bool in = j < len;
        const uint32_t key = in ? key_at(j) : 0u;
        const bool hit = in && ((key & mask) == prefix);
        const uint32_t bin = hit ? ((key >> shift) & 255u) : 256u;
        const uint32_t peers = __match_any_sync(0xffffffffu, bin);
        if (hit && (threadIdx.x & 31) == (__ffs(peers) - 1)) atomicAdd(&hist[bin], __popc(peers));
      }
      __syncthreads();
      if (threadIdx.x < 32) {
        // lane l owns digits [255 - 8l - 7, 255 - 8l]; find the digit where the
        // running count from the top reaches `remaining`.
        const int lane = threadIdx.x;
        int c[8];
        int tot = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          c[q] = hist[255 - 8 * lane - q];
          tot += c[q];
        }
        int incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        const int excl = incl - tot;  // count strictly above this lane's digits
        if (excl < remaining && incl >= remaining) {
          int run = excl;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            if (run + c[q] >= remaining) {
              sh_digit = 255u - 8u * lane - q;
              sh_remaining = remaining - run;
              break;
            }
            run += c[q];
          }
        }
      }
      __syncthreads();
      prefix |= sh_digit << shift;
      mask |= 255u << shift;
      remaining = sh_remaining;
      __syncthreads();
    }
  }
  const uint32_t T = prefix;
  const int need_eq = remaining;  // keys == T to keep, lowest indices first

  // Ordered compaction: thread t owns the contiguous segment [b0, b1).
  const int per = (len + blockDim.x - 1) / blockDim.x;
  const int b0 = min(len, (int)threadIdx.x * per), b1 = min(len, b0 + per);
  int n_eq = 0, n_gt = 0;
  if (!take_all && k > 0) {
    for (int j = b0; j < b1; ++j) {
      const uint32_t key = key_at(j);
      n_gt += key > T;
      n_eq += key == T;
    }
  }
  int tot_eq;
  const int eq_before = block_excl_scan(n_eq, warp_tot, tot_eq);
  int keep_eq = need_eq - eq_before;
  keep_eq = keep_eq < 0 ? 0 : (keep_eq > n_eq ? n_eq : keep_eq);
  const int mine = take_all ? (b1 - b0) : (k > 0 ? n_gt + keep_eq : 0);
  int total;
  int pos = block_excl_scan(mine, warp_tot, total);
  if (mine > 0) {
    int eq_seen = 0;
    for (int j = b0; j < b1; ++j) {
      bool keep;
      if (take_all) {
        keep = true;
      } else {
        const uint32_t key = key_at(j);
        keep = key > T;
        if (key == T) {
          keep = eq_seen < keep_eq;
          ++eq_seen;
        }
      }
      if (keep) {
        if (idx_out) idx_out[(long long)r * out_ld + pos] = j;
        if (bits) {
          const int bp = bit_neg ? bit_base - j : bit_base + j;
          atomicOr(bits + (long long)r * a.bits_ld + (bp >> 5), 1u << (bp & 31));
        }
        ++pos;
      }
    }
  }
  if (threadIdx.x == 0 && a.count_out) a.count_out[blockIdx.x] = total;
}

int launch_topk(const TopkArgs& a, cudaStream_t st) {
  const int rows = a.split > 0 ? 2 * a.split : a.rows;
  if (rows <= 0) return SA_OK;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(topk_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTopkSmemKeys * 4);
    attr = true;
  }
  TopkArgs b = a;
  b.smem_keys = kTopkSmemKeys;
  topk_rows_kernel<<<rows, kTopkThreads, kTopkSmemKeys * 4, st>>>(b);
  return check_launch("topk_rows_kernel");
}

}  // namespace sa

extern "C" int sa_topk_stable_f32(const float* scores, int rows, int n, long long ld, int k,
                                  int32_t* idx_out, long long out_ld, void* stream) {
  using namespace sa;
  if (rows < 0 || n < 1 || ld < n) return fail(SA_ERR_DIMENSION, "bad topk shape");
  if (k < 1 || k > n) return fail(SA_ERR_PATTERN_PARAM, "k must be in [1, %d], got %d", n, k);
  if (!scores || !idx_out || out_ld < k) return fail(SA_ERR_DIMENSION, "bad topk output");
  TopkArgs a{};
  a.scores = scores;
  a.ld = ld;
  a.rows = rows;
  a.n = n;
  a.k = k;
  a.idx_out = idx_out;
  a.out_ld = out_ld;
  return launch_topk(a, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int sa_topk_stable_rows_f32(const float* scores, int rows, long long ld,
                                       const int32_t* lens, const int32_t* ks, int32_t* idx_out,
                                       long long out_ld, int32_t* count_out, void* stream) {
  using namespace sa;
  if (rows < 0 || !scores || !lens || !ks || !idx_out)
    return fail(SA_ERR_DIMENSION, "bad segmented topk arguments");
  TopkArgs a{};
  a.scores = scores;
  a.ld = ld;
  a.rows = rows;
  a.lens = lens;
  a.ks = ks;
  a.idx_out = idx_out;
  a.out_ld = out_ld;
  a.count_out = count_out;
  return launch_topk(a, reinterpret_cast<cudaStream_t>(stream));
}
