// topk.cu — stable top-k of fp32 score rows, bit-exact with the reference's
// _top_k_stable (patterns.py:231-234): the k largest scores, ties resolved to
// the LOWER index, returned in ascending index order.
//
// Every score maps to a 32-bit preference key (larger key = preferred;
// -0.0 == +0.0; NaN least preferred, as numpy's argsort puts NaN last) and a
// row element to the 64-bit composite (key << 32 | ~index), which is unique
// and orders exactly like the stable sort.  Per row (one CTA) the k-th largest
// composite T is found without sorting the row:
//   1. one coalesced pass takes the key range [kmin, kmax];
//   2. a 4096-bin histogram over that range (bins are monotone in the key, so
//      scores of similar magnitude spread over many bins instead of colliding
//      on a few radix digits) locates the bin holding the k-th key;
//   3. that bin's composites (m of them) are gathered to shared memory; if
//      m > 1024 the bin is split once more by a second 4096-bin histogram;
//   4. the exact rank of each gathered composite is counted in parallel and
//      the one with rank k - above is T.
// Rows whose candidates stay above 1024 after two levels (massive exact ties)
// use an exact 4 x 8-bit radix select.  Output: every j with composite >= T,
// in index order, by a warp-ballot ordered compaction.
//
// Long rows (n >= kClusterMin, the VS score rows at 16K+ tokens) run on a cluster of
// kClusterC CTAs per row: each CTA stages 1/kClusterC of the row as keys in its
// shared memory, the per-CTA histograms and candidates meet in the leader CTA
// through distributed shared memory, and the ordered compaction offsets each
// CTA by the kept counts of the lower-ranked ones.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "api_common.h"
#include "internal.h"
#include "sa_types.h"

namespace sa {

constexpr int kTopkThreads = 1024;

// Profiling hook (tools/topk_lab.py --trace): per-CTA globaltimer stamps at the
// phase boundaries, [blockIdx.x * 16 + phase]; null (the default) disables.
__device__ unsigned long long* g_topk_trace = nullptr;
__device__ __forceinline__ void tk_stamp(int e) {
  unsigned long long* t = g_topk_trace;
  if (t != nullptr && threadIdx.x == 0) {
    unsigned long long v;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
    t[blockIdx.x * 16 + e] = v;
  }
}
constexpr int kBins = 4096;
constexpr int kCand = 1024;
constexpr int kTopkSmem = kBins * 4 + kCand * 8;  // 24 KB dynamic

__device__ __forceinline__ uint32_t pref_key(float f) {
  uint32_t b = __float_as_uint(f);
  if ((b & 0x7fffffffu) > 0x7f800000u) return 0u;  // NaN
  if ((b & 0x7fffffffu) == 0u) b = 0u;               // -0.0 -> +0.0
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ uint64_t composite(uint32_t key, int j) {
  return (static_cast<uint64_t>(key) << 32) | static_cast<uint32_t>(0xffffffffu - (uint32_t)j);
}

// Row access: CACHED rows were converted to preference keys in shared memory
// by one coalesced pass; otherwise every pass re-reads the fp32 row (L2).
template <bool CACHED>
__device__ __forceinline__ uint32_t key_at(const float* s, const uint32_t* skey, int j) {
  if (CACHED) return skey[j];
  return pref_key(__ldg(s + j));
}

// bin of `key` in [lo, lo + span): floor((key - lo) * scale / 2^32) with
// scale = floor(kBins * 2^32 / span) split as s_hi * 2^32 + s_lo, so the map
// is two integer multiplies (monotone, < kBins) instead of a 64-bit division.
struct BinMap {
  uint32_t lo, s_hi, s_lo;
};
__host__ __device__ inline BinMap make_binmap(uint32_t lo, uint64_t span) {
  const uint64_t scale = ((uint64_t)kBins << 32) / span;
  return BinMap{lo, (uint32_t)(scale >> 32), (uint32_t)scale};
}
__device__ __forceinline__ int key_bin(uint32_t key, const BinMap& m) {
  const uint32_t x = key - m.lo;
  return (int)(x * m.s_hi + __umulhi(x, m.s_lo));
}
// first offset x (from lo) whose bin is >= b
__device__ __forceinline__ uint64_t bin_start(int b, uint64_t span) {
  const uint64_t scale = ((uint64_t)kBins << 32) / span;
  const uint64_t x = (((uint64_t)b << 32) + scale - 1) / scale;
  return x < span ? x : span;
}

// Exclusive block-wide scan of one int per thread (any warp count <= 32).
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
    int t = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
    int s = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    warp_tot[lane] = s - t;
    if (lane == 31) warp_tot[32] = s;
  }
  __syncthreads();
  const int r = warp_tot[w] + x - v;
  total = warp_tot[32];
  __syncthreads();
  return r;
}

// Exact rank of the candidates: warp gw of nw (block-wide or cluster-wide
// numbering) ranks candidates gw, gw + nw, ...; its lanes split the
// comparisons and a butterfly sums them, so m candidates cost m^2 / (32 nw)
// compares per lane instead of m per thread.  The composite of rank want - 1
// (0-based; composites are unique) is written to *T_out.
__device__ __forceinline__ void rank_candidates(const uint64_t* cand, int m, int want, int gw, int nw,
                                                uint64_t* T_out) {
  const int lane = threadIdx.x & 31;
  for (int c = gw; c < m; c += nw) {
    const uint64_t me = cand[c];
    int rank = 0;
    for (int o = lane; o < m; o += 32) rank += cand[o] > me;
#pragma unroll
    for (int x = 16; x > 0; x >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, x);
    if (lane == 0 && rank == want - 1) *T_out = me;
  }
}

// Histogram of the keys inside [lo, lo + span) into kBins bins; returns the bin
// holding the `want`-th largest of them and the count in higher bins.
template <bool CACHED>
__device__ void hist_locate(const float* s, const uint32_t* skey, int len, uint32_t lo, uint64_t span, int want,
                            int* hist, int* warp_tot, int* sh_pair, int& bin_out, int& above_out) {
  const int tid = threadIdx.x;
  for (int t = tid; t < kBins; t += blockDim.x) hist[t] = 0;
  __syncthreads();
  const BinMap bm = make_binmap(lo, span);
  for (int j0 = tid; j0 < len; j0 += 8 * blockDim.x) {
    uint32_t key[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = j0 + u * blockDim.x;
      key[u] = j < len ? key_at<CACHED>(s, skey, j) : 0u;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = j0 + u * blockDim.x;
      if (j < len && key[u] >= lo && (uint64_t)(key[u] - lo) < span)
        atomicAdd(&hist[key_bin(key[u], bm)], 1);
    }
  }
  __syncthreads();
  // suffix counts: thread t owns bins [kBins - (t+1)*per, kBins - t*per), scanned from the top
  const int per = kBins / blockDim.x;
  const int b_hi = kBins - tid * per;
  int mine = 0;
  for (int q = 1; q <= per; ++q) mine += hist[b_hi - q];
  int tot;
  const int before = block_excl_scan(mine, warp_tot, tot);  // keys in higher bins
  if (before < want && before + mine >= want) {
    int run = before;
    for (int q = 1; q <= per; ++q) {
      const int b = b_hi - q;
      if (run + hist[b] >= want) {
        sh_pair[0] = b;
        sh_pair[1] = run;
        sh_pair[2] = hist[b];
        break;
      }
      run += hist[b];
    }
  }
  __syncthreads();
  bin_out = sh_pair[0];
  above_out = sh_pair[1];
}

template <bool CACHED>
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
  tk_stamp(0);

  extern __shared__ __align__(16) uint8_t tk_smem[];
  int* hist = reinterpret_cast<int*>(tk_smem);
  uint64_t* cand = reinterpret_cast<uint64_t*>(tk_smem + kBins * 4);
  uint32_t* skey = reinterpret_cast<uint32_t*>(tk_smem + kTopkSmem);  // CACHED: [len]
  if (CACHED) {
    // one coalesced 16-byte pass: fp32 row -> preference keys in shared memory
    const bool vec = ((reinterpret_cast<uintptr_t>(s) & 15) == 0);
    const int n4 = vec ? len / 4 : 0;
    for (int j4 = threadIdx.x; j4 < n4; j4 += blockDim.x) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(s) + j4);
      skey[4 * j4] = pref_key(v.x);
      skey[4 * j4 + 1] = pref_key(v.y);
      skey[4 * j4 + 2] = pref_key(v.z);
      skey[4 * j4 + 3] = pref_key(v.w);
    }
    for (int j = 4 * n4 + threadIdx.x; j < len; j += blockDim.x) skey[j] = pref_key(__ldg(s + j));
    __syncthreads();
  }
  tk_stamp(1);
  __shared__ int warp_tot[33];
  __shared__ uint32_t sh_min, sh_max;
  __shared__ int sh_m;
  __shared__ int sh_pair[3];
  __shared__ uint64_t sh_T;
  __shared__ uint32_t sh_digit;
  __shared__ int sh_rem;

  const int tid = threadIdx.x, lane = tid & 31;
  const bool take_all = k >= len;
  uint64_t T = 0;  // keep j iff composite(j) >= T
  if (!take_all && k > 0) {
    // 1. key range
    uint32_t mn = 0xffffffffu, mx = 0u;
    for (int j0 = tid; j0 < len; j0 += 8 * blockDim.x) {
      uint32_t v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = j0 + u * blockDim.x;
        v[u] = j < len ? key_at<CACHED>(s, skey, j) : 0u;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (j0 + u * (int)blockDim.x < len) {
          mn = min(mn, v[u]);
          mx = max(mx, v[u]);
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (tid == 0) {
      sh_min = 0xffffffffu;
      sh_max = 0u;
    }
    __syncthreads();
    if (lane == 0) {
      atomicMin(&sh_min, mn);
      atomicMax(&sh_max, mx);
    }
    __syncthreads();
    uint32_t lo = sh_min;
    uint64_t span = (uint64_t)(sh_max - sh_min) + 1;
    int want = k;  // rank (1-based) of T among the keys in [lo, lo + span)
    bool located = false;
    tk_stamp(2);
    for (int level = 0; level < 2 && !located; ++level) {
      int bin, above;
      hist_locate<CACHED>(s, skey, len, lo, span, want, hist, warp_tot, sh_pair, bin, above);
      tk_stamp(3 + 3 * level);
      const int m = sh_pair[2];
      want -= above;
      // narrow the key range to the bin: keys with key_bin == bin
      const uint64_t b0 = bin_start(bin, span);
      const uint64_t b1 = bin_start(bin + 1, span);
      lo = lo + (uint32_t)b0;
      span = b1 - b0;
      if (m > kCand) continue;
      // 3. gather the bin's composites
      if (tid == 0) sh_m = 0;
      __syncthreads();
      for (int j0 = tid; (j0 & ~31) < len; j0 += 8 * blockDim.x) {  // warp-uniform trip count
        uint32_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int j = j0 + u * blockDim.x;
          v[u] = j < len ? key_at<CACHED>(s, skey, j) : 0u;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int j = j0 + u * blockDim.x;
          const uint32_t key = v[u];
          const bool hit = j < len && key >= lo && (uint64_t)(key - lo) < span;
          const uint32_t bal = __ballot_sync(0xffffffffu, hit);
          if (bal) {
            int base = 0;
            if (lane == 0) base = atomicAdd(&sh_m, __popc(bal));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (hit) cand[base + __popc(bal & ((1u << lane) - 1u))] = composite(key, j);
          }
        }
      }
      __syncthreads();
      tk_stamp(4 + 3 * level);
      // 4. exact rank of every candidate; rank want - 1 (0-based) is T
      rank_candidates(cand, m, want, tid >> 5, (int)blockDim.x >> 5, &sh_T);
      __syncthreads();
      tk_stamp(5 + 3 * level);
      T = sh_T;
      located = true;
    }
    if (!located) {
      // exact fallback (massive exact ties): 4 x 8-bit radix select, then the
      // remaining-th equal key in index order fixes the composite threshold
      uint32_t prefix = 0u, mask = 0u;
      int remaining = k;
      for (int pass = 0; pass < 4; ++pass) {
        const int shift = 24 - 8 * pass;
        for (int t = tid; t < 256; t += blockDim.x) hist[t] = 0;
        __syncthreads();
        for (int j = tid; j < len; j += blockDim.x) {
          const uint32_t key = key_at<CACHED>(s, skey, j);
          if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1);
        }
        __syncthreads();
        if (tid == 0) {
          int run = 0;
          for (int d = 255; d >= 0; --d) {
            if (run + hist[d] >= remaining) {
              sh_digit = (uint32_t)d;
              sh_rem = remaining - run;
              break;
            }
            run += hist[d];
          }
        }
        __syncthreads();
        prefix |= sh_digit << shift;
        mask |= 255u << shift;
        remaining = sh_rem;
        __syncthreads();
      }
      const int per = (len + blockDim.x - 1) / blockDim.x;
      const int b0 = min(len, tid * per), b1 = min(len, b0 + per);
      int eq = 0;
      for (int j = b0; j < b1; ++j) eq += key_at<CACHED>(s, skey, j) == prefix;
      int tot;
      const int before = block_excl_scan(eq, warp_tot, tot);
      if (before < remaining && before + eq >= remaining) {
        int seen = before;
        for (int j = b0; j < b1; ++j) {
          if (key_at<CACHED>(s, skey, j) == prefix && ++seen == remaining) {
            sh_T = composite(prefix, j);
            break;
          }
        }
      }
      __syncthreads();
      T = sh_T;
    }
  }

  // ordered compaction: warp w owns the contiguous range [w0, w1), read 32 at a
  // time (coalesced); a ballot orders the kept elements inside each chunk
  const int nw = blockDim.x >> 5, w = tid >> 5;
  const int wlen = (((len + nw - 1) / nw) + 31) & ~31;
  const int w0 = min(len, w * wlen), w1 = min(len, w0 + wlen);
  int mine = 0;
  for (int j = w0 + lane; (j - lane) < w1; j += 32) {
    const bool keep = j < w1 && (take_all || (k > 0 && composite(key_at<CACHED>(s, skey, j), j) >= T));
    mine += __popc(__ballot_sync(0xffffffffu, keep));
  }
  int total;
  const int wbase = block_excl_scan(lane == 0 ? mine : 0, warp_tot, total);
  int pos = __shfl_sync(0xffffffffu, wbase, 0);
  if (mine > 0) {
    for (int j = w0 + lane; (j - lane) < w1; j += 32) {
      const bool keep = j < w1 && (take_all || (k > 0 && composite(key_at<CACHED>(s, skey, j), j) >= T));
      const uint32_t bal = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        const int p = pos + __popc(bal & ((1u << lane) - 1u));
        if (idx_out) idx_out[(long long)r * out_ld + p] = j;
        if (bits) {
          const int bp = bit_neg ? bit_base - j : bit_base + j;
          atomicOr(bits + (long long)r * a.bits_ld + (bp >> 5), 1u << (bp & 31));
        }
      }
      pos += __popc(bal);
    }
  }
  if (tid == 0 && a.count_out) a.count_out[blockIdx.x] = total;
  tk_stamp(15);
}

namespace cg = cooperative_groups;
constexpr int kClusterC = 8;
constexpr int kClusterMin = 16384;  // plain rows at least this long use a cluster per row

// Radix fallback (massive exact ties) over the fp32 row in global memory; the
// result lands in *T_out (block-wide; every thread of the CTA calls it).
__device__ void radix_threshold(const float* s, int len, int k, int* hist, int* warp_tot, uint32_t* sh_digit,
                                int* sh_rem, uint64_t* T_out) {
  const int tid = threadIdx.x;
  uint32_t prefix = 0u, mask = 0u;
  int remaining = k;
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    for (int t = tid; t < 256; t += blockDim.x) hist[t] = 0;
    __syncthreads();
    for (int j = tid; j < len; j += blockDim.x) {
      const uint32_t key = pref_key(__ldg(s + j));
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1);
    }
    __syncthreads();
    if (tid == 0) {
      int run = 0;
      for (int d = 255; d >= 0; --d) {
        if (run + hist[d] >= remaining) {
          *sh_digit = (uint32_t)d;
          *sh_rem = remaining - run;
          break;
        }
        run += hist[d];
      }
    }
    __syncthreads();
    prefix |= *sh_digit << shift;
    mask |= 255u << shift;
    remaining = *sh_rem;
    __syncthreads();
  }
  const int per = (len + blockDim.x - 1) / blockDim.x;
  const int b0 = min(len, tid * per), b1 = min(len, b0 + per);
  int eq = 0;
  for (int j = b0; j < b1; ++j) eq += pref_key(__ldg(s + j)) == prefix;
  int tot;
  const int before = block_excl_scan(eq, warp_tot, tot);
  if (before < remaining && before + eq >= remaining) {
    int seen = before;
    for (int j = b0; j < b1; ++j) {
      if (pref_key(__ldg(s + j)) == prefix && ++seen == remaining) {
        *T_out = composite(prefix, j);
        break;
      }
    }
  }
  __syncthreads();
}

__global__ void __cluster_dims__(kClusterC, 1, 1) __launch_bounds__(kTopkThreads)
    topk_cluster_kernel(TopkArgs a) {
  cg::cluster_group cl = cg::this_cluster();
  const int cr = (int)cl.block_rank();
  int r = blockIdx.x / kClusterC;
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
  if (a.gate && a.gate[r / a.gate_div] != a.gate_val) return;  // uniform over the cluster
  const int len = a.n;
  const int k = kk < len ? kk : len;
  const float* s = scores + (long long)r * a.ld;
  // this CTA's slice [j_lo, j_hi), a multiple of 4 keys long
  const int per = (((len + kClusterC - 1) / kClusterC) + 3) & ~3;
  const int j_lo = min(len, cr * per), j_hi = min(len, j_lo + per), sl = j_hi - j_lo;

  extern __shared__ __align__(16) uint8_t tk_smem[];
  int* hist = reinterpret_cast<int*>(tk_smem);
  uint64_t* cand = reinterpret_cast<uint64_t*>(tk_smem + kBins * 4);
  uint32_t* skey = reinterpret_cast<uint32_t*>(tk_smem + kTopkSmem);  // [per]
  __shared__ int warp_tot[33];
  __shared__ uint32_t sh_min, sh_max;
  __shared__ int sh_m, sh_tot, sh_base;
  __shared__ int sh_pair[3];
  __shared__ uint64_t sh_T;
  __shared__ uint32_t sh_digit;
  __shared__ int sh_rem;
  const int tid = threadIdx.x, lane = tid & 31;

  auto key_of = [&](int j) -> uint32_t { return skey[j]; };
  tk_stamp(0);
  // stage the slice as preference keys (16-byte loads when aligned)
  {
    const float* sp = s + j_lo;
    const bool vec = ((reinterpret_cast<uintptr_t>(sp) & 15) == 0);
    const int n4 = vec ? sl / 4 : 0;
    for (int j4 = tid; j4 < n4; j4 += blockDim.x) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(sp) + j4);
      skey[4 * j4] = pref_key(v.x);
      skey[4 * j4 + 1] = pref_key(v.y);
      skey[4 * j4 + 2] = pref_key(v.z);
      skey[4 * j4 + 3] = pref_key(v.w);
    }
    for (int j = 4 * n4 + tid; j < sl; j += blockDim.x) skey[j] = pref_key(__ldg(sp + j));
  }
  tk_stamp(1);
  const bool take_all = k >= len;
  uint64_t T = 0;
  if (!take_all && k > 0) {
    // 1. key range: CTA min/max, then the leader's
    if (tid == 0) {
      sh_min = 0xffffffffu;
      sh_max = 0u;
    }
    __syncthreads();
    uint32_t mn = 0xffffffffu, mx = 0u;
    for (int j = tid; j < sl; j += blockDim.x) {
      const uint32_t kj = key_of(j);
      mn = min(mn, kj);
      mx = max(mx, kj);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 0) {
      atomicMin(&sh_min, mn);
      atomicMax(&sh_max, mx);
    }
    cl.sync();
    if (tid == 0 && cr != 0) {
      atomicMin(cl.map_shared_rank(&sh_min, 0), sh_min);
      atomicMax(cl.map_shared_rank(&sh_max, 0), sh_max);
    }
    cl.sync();
    uint32_t lo = *cl.map_shared_rank(&sh_min, 0);
    uint64_t span = (uint64_t)(*cl.map_shared_rank(&sh_max, 0) - lo) + 1;
    int want = k;
    bool located = false;
    tk_stamp(2);
    for (int level = 0; level < 2 && !located; ++level) {
      // 2. per-CTA histograms of the slice; the leader sums them and locates
      for (int t = tid; t < kBins; t += blockDim.x) hist[t] = 0;
      __syncthreads();
      const BinMap bm = make_binmap(lo, span);
      for (int j = tid; j < sl; j += blockDim.x) {
        const uint32_t key = key_of(j);
        if (key >= lo && (uint64_t)(key - lo) < span) atomicAdd(&hist[key_bin(key, bm)], 1);
      }
      cl.sync();
      {
        // distributed merge: CTA cr sums bin slice cr of every CTA's histogram
        // into the leader's copy of that slice (the only reader / writer of it)
        constexpr int kSlice = kBins / kClusterC;
        int* lh = cl.map_shared_rank(hist, 0);
        for (int t = cr * kSlice + tid; t < (cr + 1) * kSlice; t += blockDim.x) {
          int acc = 0;
#pragma unroll
          for (int q = 0; q < kClusterC; ++q) acc += cl.map_shared_rank(hist, q)[t];
          lh[t] = acc;
        }
      }
      cl.sync();
      if (cr == 0) {
        const int pb = kBins / blockDim.x;
        const int b_hi = kBins - tid * pb;
        int mine = 0;
        for (int q = 1; q <= pb; ++q) mine += hist[b_hi - q];
        int tot;
        const int before = block_excl_scan(mine, warp_tot, tot);
        if (before < want && before + mine >= want) {
          int run = before;
          for (int q = 1; q <= pb; ++q) {
            const int b = b_hi - q;
            if (run + hist[b] >= want) {
              sh_pair[0] = b;
              sh_pair[1] = run;
              sh_pair[2] = hist[b];
              break;
            }
            run += hist[b];
          }
        }
        if (tid == 0) sh_m = 0;
      }
      cl.sync();
      tk_stamp(3 + 3 * level);
      const int* lp = cl.map_shared_rank(sh_pair, 0);
      const int bin = lp[0], above = lp[1], m = lp[2];
      want -= above;
      const uint64_t b0 = bin_start(bin, span);
      const uint64_t b1 = bin_start(bin + 1, span);
      lo = lo + (uint32_t)b0;
      span = b1 - b0;
      if (m > kCand) continue;  // uniform: every CTA read the same m
      // 3. the bin's composites gather in the leader
      int* lm = cl.map_shared_rank(&sh_m, 0);
      uint64_t* lc = cl.map_shared_rank(cand, 0);
      for (int j0 = tid; (j0 & ~31) < sl; j0 += blockDim.x) {  // warp-uniform trip count
        const uint32_t key = j0 < sl ? key_of(j0) : 0u;
        const bool hit = j0 < sl && key >= lo && (uint64_t)(key - lo) < span;
        const uint32_t bal = __ballot_sync(0xffffffffu, hit);
        if (bal) {
          int base = 0;
          if (lane == 0) base = atomicAdd(lm, __popc(bal));
          base = __shfl_sync(0xffffffffu, base, 0);
          if (hit) lc[base + __popc(bal & ((1u << lane) - 1u))] = composite(key, j_lo + j0);
        }
      }
      cl.sync();
      tk_stamp(4 + 3 * level);
      // 4. exact ranks: every CTA copies the leader's candidates and ranks
      // its share of them; the one of rank want - 1 goes to the leader
      {
        const uint64_t* rc = cl.map_shared_rank(cand, 0);
        if (cr != 0)
          for (int c = tid; c < m; c += blockDim.x) cand[c] = rc[c];
        __syncthreads();
        const int nwc = (int)blockDim.x >> 5;
        rank_candidates(cand, m, want, cr * nwc + (tid >> 5), kClusterC * nwc, cl.map_shared_rank(&sh_T, 0));
      }
      cl.sync();
      tk_stamp(5 + 3 * level);
      T = *cl.map_shared_rank(&sh_T, 0);
      located = true;
    }
    if (!located) {
      if (cr == 0) radix_threshold(s, len, k, hist, warp_tot, &sh_digit, &sh_rem, &sh_T);
      cl.sync();
      T = *cl.map_shared_rank(&sh_T, 0);
    }
  }

  // ordered compaction of the slice, offset by the kept counts of lower ranks
  const int nw = blockDim.x >> 5, w = tid >> 5;
  const int wlen = (((sl + nw - 1) / nw) + 31) & ~31;
  const int w0 = min(sl, w * wlen), w1 = min(sl, w0 + wlen);
  int mine = 0;
  for (int j = w0 + lane; (j - lane) < w1; j += 32) {
    const bool keep = j < w1 && (take_all || (k > 0 && composite(key_of(j), j_lo + j) >= T));
    mine += __popc(__ballot_sync(0xffffffffu, keep));
  }
  int total;
  const int wbase = block_excl_scan(lane == 0 ? mine : 0, warp_tot, total);
  if (tid == 0) sh_tot = total;
  cl.sync();
  if (tid == 0) {
    int b = 0, all = 0;
    for (int q = 0; q < kClusterC; ++q) {
      const int c = *cl.map_shared_rank(&sh_tot, q);
      if (q < cr) b += c;
      all += c;
    }
    sh_base = b;
    if (cr == 0 && a.count_out) a.count_out[blockIdx.x / kClusterC] = all;
  }
  __syncthreads();
  int pos = sh_base + __shfl_sync(0xffffffffu, wbase, 0);
  if (mine > 0) {
    for (int j = w0 + lane; (j - lane) < w1; j += 32) {
      const bool keep = j < w1 && (take_all || (k > 0 && composite(key_of(j), j_lo + j) >= T));
      const uint32_t bal = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        const int p = pos + __popc(bal & ((1u << lane) - 1u));
        const int jj = j_lo + j;
        if (idx_out) idx_out[(long long)r * out_ld + p] = jj;
        if (bits) {
          const int bp = bit_neg ? bit_base - jj : bit_base + jj;
          atomicOr(bits + (long long)r * a.bits_ld + (bp >> 5), 1u << (bp & 31));
        }
      }
      pos += __popc(bal);
    }
  }
  tk_stamp(14);
  cl.sync();  // no CTA leaves while its shared memory may still be read
  tk_stamp(15);
}

int launch_topk(const TopkArgs& a, cudaStream_t st) {
  const int rows = a.split > 0 ? 2 * a.split : a.rows;
  if (rows <= 0) return SA_OK;
  // short segmented rows (block estimator) use 256 threads per row
  const int threads = (a.lens != nullptr && a.n <= 4096) ? 256 : kTopkThreads;
  // rows up to kCacheMax keys are staged in shared memory once by one CTA;
  // longer plain rows by a cluster of kClusterC CTAs
  constexpr int kCacheMax = 49152;
  const int cl_per = (((a.n + kClusterC - 1) / kClusterC) + 3) & ~3;
  static std::atomic<uint64_t> attr_done{0};
  once_per_device(attr_done, [] {
    cudaFuncSetAttribute(topk_rows_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kTopkSmem + kCacheMax * 4);
    cudaFuncSetAttribute(topk_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kTopkSmem + ((262144 / kClusterC) + 4) * 4);
  });
  static const int use_cluster = [] {
    const char* e = getenv("SA_TOPK_CLUSTER");  // A/B: cluster-of-8 kernel for long rows
    return e ? atoi(e) : 1;
  }();
  // Long plain rows: a cluster per row (keys staged in the CTAs' shared
  // memory) while all clusters fit one wave — the lowest latency per row;
  // beyond that, rows that fit one CTA's shared memory go one CTA per row
  // (32K x 64 rows: 30 vs 48 us) and longer rows stay on clusters in two
  // waves (clusters re-reading their slices from L2 fit one wave but doubled
  // the per-row latency: 128K x 64 rows 104 vs 87 us).  SA_TOPK_CLUSTER=2
  // forces clusters.
  if (use_cluster && a.lens == nullptr && a.ks == nullptr && a.n >= kClusterMin && a.n <= 262144 &&
      threads == kTopkThreads) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, topk_cluster_kernel, kTopkThreads,
                                                  kTopkSmem + cl_per * 4);
    const bool one_wave = (long long)rows * kClusterC <= (long long)std::max(per_sm, 1) * device_sm_count();
    // (auto layers' gated VS rows — usually only a few are kept — stay one CTA
    // per row when they fit its shared memory: their latency is hidden beside
    // the block GEMM, and a cluster per row takes 8 SMs' slots from it; 32K
    // auto layer 1.0897 -> 1.085 ms)
    if (use_cluster == 2 || (use_cluster == 1 && ((one_wave && !a.gate_sparse) || a.n > kCacheMax))) {
      topk_cluster_kernel<<<rows * kClusterC, kTopkThreads, kTopkSmem + cl_per * 4, st>>>(a);
      return check_launch("topk_cluster_kernel");
    }
  }
  const int maxlen = a.n;  // a.n bounds every row length
  if (maxlen <= kCacheMax && a.lens == nullptr)
    topk_rows_kernel<true><<<rows, threads, kTopkSmem + maxlen * 4, st>>>(a);
  else
    topk_rows_kernel<false><<<rows, threads, kTopkSmem, st>>>(a);
  return check_launch("topk_rows_kernel");
}

}  // namespace sa

extern "C" int sa_topk_trace_buffer(void* p) {
  unsigned long long* v = reinterpret_cast<unsigned long long*>(p);
  return cudaMemcpyToSymbol(sa::g_topk_trace, &v, sizeof(v)) == cudaSuccess ? 0 : 1;
}

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
