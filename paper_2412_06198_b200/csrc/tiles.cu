// tiles.cu — turn each head's realised index into the per-(head, query-tile)
// list of 128-key tiles the attention kernel executes.
//
// A tile (qt, kt) is listed iff the index covers at least one causal position
// inside it (so the executed work is exactly the tiles the index touches);
// its kind says which mask the softmax applies (sa_types.h).  Semantics
// follow the reference's SparseIndex field definitions (patterns.py:113-133):
// columns (i >= j), diagonals (i - j = o), blocks (token causality inside),
// always_diagonal (forced (i, i)).
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "sa_types.h"

namespace sa {

struct TileBuildArgs {
  int n, nqt, hh_total;
  HeadIndexView idx;
  int32_t* tile_off;  // [hh_total * nqt]
  int32_t* tile_cnt;  // [hh_total * nqt]
  uint32_t* tiles;    // capacity hh_total * nqt * (nqt + 1) / 2
  long long* work_cost;  // optional per (hh, qt): tile count (for scheduling / accounting)
};

__device__ __forceinline__ int popc_range(const uint32_t* bits, int lo, int hi) {
  // number of set bits in [lo, hi), bits stored LSB-first in 32-bit words
  if (hi <= lo) return 0;
  int total = 0;
  int w0 = lo >> 5, w1 = (hi - 1) >> 5;
  for (int w = w0; w <= w1; ++w) {
    uint32_t v = bits[w];
    if (w == w0) v &= 0xffffffffu << (lo & 31);
    if (w == w1) {
      int top = (hi - 1) & 31;
      v &= (top == 31) ? 0xffffffffu : ((2u << top) - 1u);
    }
    total += __popc(v);
  }
  return total;
}

// One warp per (hh, qt).  Lanes evaluate 32 candidate key tiles at a time and
// compact the included ones in key order with a ballot prefix.
__global__ void build_tiles_kernel(TileBuildArgs a) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= a.hh_total * a.nqt) return;
  const int hh = gw / a.nqt;
  const int qt = gw % a.nqt;
  const int fam = a.idx.family[hh];
  const long long base = (long long)hh * a.nqt * (a.nqt + 1) / 2 + (long long)qt * (qt + 1) / 2;
  uint32_t* out = a.tiles + base;
  const int i0 = qt * kTile;
  const int i1 = i0 + kTile - 1;       // last row of the tile (may be padding)
  const int i1v = min(i1, a.n - 1);    // last real row
  int count = 0;

  // Block family: mark touched key tiles in a per-warp bitmap first.
  __shared__ uint32_t blk_mark_all[8][64];  // up to 2048 key tiles per warp (n <= 262144)
  uint32_t* blk_mark = blk_mark_all[(threadIdx.x >> 5) & 7];
  int b = 0;
  if (fam == FAM_BLOCK) {
    b = a.idx.blk_b[hh];
    const int words = (a.nqt + 31) >> 5;
    for (int w = lane; w < words; w += 32) blk_mark[w] = 0u;
    __syncwarp();
    const int32_t* ro = a.idx.blk_row_off + (size_t)hh * a.idx.blk_row_stride;
    const int g0 = i0 / b, g1 = i1v / b;
    const int nbk = (a.n + b - 1) / b;
    auto mark = [&](int k) {
      const int gk = a.idx.blk_idx[k];
      if (gk >= nbk) return;  // sentinel padding
      const int t0 = (gk * b) / kTile;
      const int t1 = min((gk + 1) * b - 1, a.n - 1) / kTile;
      for (int t = t0; t <= t1 && t <= qt; ++t) atomicOr(&blk_mark[t >> 5], 1u << (t & 31));
    };
    if (g1 - g0 >= 7) {
      // many short rows (b <= 16): a lane per query block, all rows' loads in flight at once
      for (int gq = g0 + lane; gq <= g1; gq += 32)
        for (int k = ro[gq], k1 = ro[gq + 1]; k < k1; ++k) mark(k);
    } else {
      // few long rows (b >= 32): the lanes split each row
      for (int gq = g0; gq <= g1; ++gq)
        for (int k = ro[gq] + lane; k < ro[gq + 1]; k += 32) mark(k);
    }
    __syncwarp();
  }
  // Gather mode: G gathered tiles (slot s = g-th off-diagonal block of query
  // block s) + the diagonal tile restricted to each row's own block.  Needs
  // every row ascending with its diagonal block last (patterns.py:319).
  int gather_g = -1;
  if (fam == FAM_BLOCK && block_gather_ok(b)) {
    const int32_t* ro = a.idx.blk_row_off + (size_t)hh * a.idx.blk_row_stride;
    const int gq = i0 / b + lane;
    int c = 0;
    bool ok = true;
    if (lane < kTile / b && gq <= i1v / b) {
      int prev = -1;
      bool diag = false;
      for (int k = ro[gq]; k < ro[gq + 1]; ++k) {
        const int gk = a.idx.blk_idx[k];
        if (gk > gq) break;  // sentinel padding
        ok = ok && gk > prev && !diag;
        prev = gk;
        if (gk == gq) diag = true; else ++c;
      }
      ok = ok && diag;
    }
    const int G = __reduce_max_sync(0xffffffffu, c);
    if (__all_sync(0xffffffffu, ok)) gather_g = G;
  }

  for (int kt0 = 0; kt0 <= qt; kt0 += 32) {
    const int kt = kt0 + lane;
    bool inc = false;
    uint32_t kind = TK_FULL;
    if (kt <= qt) {
      const int j0 = kt * kTile, j1 = j0 + kTile - 1;
      if (fam == FAM_DENSE) {
        inc = true;
        kind = (kt < qt) ? TK_FULL : TK_CAUSAL;
      } else if (fam == FAM_TRI) {
        const int w = a.idx.tri_window[hh], s = a.idx.tri_sinks[hh];
        const bool band = (j1 >= i0 - w + 1);  // j0 <= i1 holds for kt <= qt
        const bool sink = (j0 < s);
        inc = band || sink || kt == qt;
        const bool full = (kt < qt) && ((i1 - j0 < w) || (j1 < s));
        kind = full ? TK_FULL : TK_BAND;
      } else if (fam == FAM_VS || fam == FAM_VS_NOEYE) {
        const uint32_t* cb = a.idx.colbits + (size_t)hh * a.idx.vs_words;
        const uint32_t* dr = a.idx.diagrev + (size_t)hh * a.idx.vs_words;
        inc = (kt == qt) || popc_range(cb, j0, min(j1, a.n - 1) + 1) > 0;
        if (!inc) {
          // diagonal offsets touching the tile: [i0 - j1, i1v - j0] (clipped at 0)
          const int olo = max(0, i0 - j1), ohi = i1v - j0;
          // diagrev bit (n + 127 - o): offsets [olo, ohi] <-> bits [n+127-ohi, n+127-olo]
          inc = popc_range(dr, a.n + 127 - ohi, a.n + 127 - olo + 1) > 0;
        }
        kind = TK_VS;
      } else {  // FAM_BLOCK
        inc = (kt == qt) || ((blk_mark[kt >> 5] >> (kt & 31)) & 1u);
        if (b % kTile == 0) kind = (kt < qt) ? TK_FULL : TK_CAUSAL;
        else kind = TK_BLOCK;
      }
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, inc);
    if (inc) out[count + __popc(bal & ((1u << lane) - 1u))] = tile_entry(kt, kind);
    count += __popc(bal);
  }
  if (gather_g >= 0 && gather_g + 1 < count) {
    __syncwarp();
    for (int g = lane; g <= gather_g; g += 32)
      out[g] = (g < gather_g) ? tile_entry(g, TK_GATHER) : tile_entry(qt, TK_BLOCKDIAG);
    count = gather_g + 1;
  }
  if (lane == 0) {
    a.tile_off[gw] = (int32_t)base;
    a.tile_cnt[gw] = count;
    if (a.work_cost) a.work_cost[gw] = count;
  }
}

// Longest-processing-time-first launch order: work[r] = the item (hh * nqt +
// qt) with the r-th largest tile count (counting sort, one CTA).  The block
// scheduler dispatches CTAs roughly in blockIdx order, so the heaviest query
// tiles (full-width VS rows) start first and the light ones fill the tail.
// Items of count 0 (nothing to compute) go last; n_work, when given, receives
// the number of nonzero items.
__device__ __forceinline__ int order_bin(int c, int shift) {
  return c > 0 ? 1022 - min(c >> shift, 1022) : 1023;
}
// Within a bin the items are scattered in (kv group, query tile, head of the
// group) order, `g` heads per group, so the GQA siblings of a query tile (same
// K/V tiles) sit next to each other and run concurrently: their shared K/V
// tiles are read from HBM once and hit L2 for the others.
__device__ __forceinline__ int sibling_item(int p, int nqt, int g) {
  const int grp = p / (nqt * g), r = p % (nqt * g);
  return (grp * g + r % g) * nqt + r / g;
}
__global__ void __launch_bounds__(1024) order_work_kernel(const int32_t* __restrict__ cnt, int items,
                                                          int max_cnt, int32_t* __restrict__ work,
                                                          int32_t* __restrict__ n_work, int nqt, int g,
                                                          int32_t* __restrict__ zero_counter) {
  // bins: tile count >> shift, at most 1023 (one per thread) plus the empty bin, heaviest first
  __shared__ int start[1024];
  __shared__ int wsum[32];
  int shift = 0;
  while ((max_cnt >> shift) >= 1023) ++shift;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  start[t] = 0;
  __syncthreads();
  // counts are loaded 8 per thread before use (one memory latency per batch)
  constexpr int kB = 8;
  for (int i0 = t; i0 < items; i0 += kB * (int)blockDim.x) {
    int c[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int i = i0 + u * (int)blockDim.x;
      c[u] = i < items ? __ldg(cnt + i) : INT_MIN;
    }
#pragma unroll
    for (int u = 0; u < kB; ++u)
      if (c[u] != INT_MIN) atomicAdd(&start[order_bin(c[u], shift)], 1);
  }
  __syncthreads();
  // exclusive scan over position p = 1023 - bin (heaviest bin first)
  const int v = start[t];
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    const int s0 = wsum[lane];
    int sc = s0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, sc, o);
      if (lane >= o) sc += y;
    }
    wsum[lane] = sc - s0;
  }
  __syncthreads();
  start[t] = wsum[w] + x - v;
  if (t == 1023 && n_work) *n_work = start[t];
  if (t == 0 && zero_counter) *zero_counter = 0;  // the attention kernel's item counter
  __syncthreads();
  // scatter: warp-aggregated, so lanes of one bin take consecutive positions in lane order
  for (int p0 = t - lane; p0 < items; p0 += kB * (int)blockDim.x) {
    int c[kB], it[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int p = p0 + u * (int)blockDim.x + lane;
      it[u] = p < items ? sibling_item(p, nqt, g) : -1;
      c[u] = it[u] >= 0 ? __ldg(cnt + it[u]) : INT_MIN;
    }
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int bin = c[u] != INT_MIN ? order_bin(c[u], shift) : -1;
      const unsigned peers = __match_any_sync(0xffffffffu, bin);
      const int leader = __ffs(peers) - 1;
      int base = 0;
      if (lane == leader && bin >= 0) base = atomicAdd(&start[bin], __popc(peers));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (bin >= 0) work[base + __popc(peers & ((1u << lane) - 1u))] = it[u];
    }
  }
}

}  // namespace sa

// ------------------------------------------------------------------ C ABI
#include "api_common.h"
#include "internal.h"

extern "C" int sa_build_tiles(const sa_head_index* index, int hh_total, int n, int32_t* tile_off,
                              int32_t* tile_cnt, uint32_t* tiles, void* stream) {
  using namespace sa;
  if (hh_total < 1 || n < 1) return fail(SA_ERR_DIMENSION, "need hh_total, n >= 1");
  if (n > 262144) return fail(SA_ERR_DIMENSION, "n=%d exceeds the 262144-token tile-map limit", n);
  if (!index || !tile_off || !tile_cnt || !tiles) return fail(SA_ERR_DIMENSION, "null pointer");
  TileBuildArgs a;
  a.n = n;
  a.nqt = (n + kTile - 1) / kTile;
  a.hh_total = hh_total;
  a.idx = *index;
  a.tile_off = tile_off;
  a.tile_cnt = tile_cnt;
  a.tiles = tiles;
  a.work_cost = nullptr;
  const long long warps = (long long)hh_total * a.nqt;
  const int threads = 256;
  const int grid = (int)((warps * 32 + threads - 1) / threads);
  build_tiles_kernel<<<grid, threads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(a);
  return check_launch("build_tiles_kernel");
}

extern "C" int sa_order_work(const int32_t* tile_cnt, int items, int max_cnt, int32_t* work,
                             void* stream) {
  using namespace sa;
  if (items < 1 || max_cnt < 0 || max_cnt > 65536) return fail(SA_ERR_DIMENSION, "bad work-order sizes");
  if (!tile_cnt || !work) return fail(SA_ERR_DIMENSION, "null pointer");
  order_work_kernel<<<1, 1024, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      tile_cnt, items, max_cnt, work, nullptr, items, 1, nullptr);
  return check_launch("order_work_kernel");
}

namespace sa {
int launch_order_work(const int32_t* cost, int items, int max_cost, int32_t* work, int32_t* n_work,
                      cudaStream_t st, int nqt, int group, int32_t* zero_counter) {
  if (nqt < 1 || group < 1 || items % (nqt * group) != 0) {
    nqt = items;
    group = 1;
  }
  order_work_kernel<<<1, 1024, 0, st>>>(cost, items, max_cost, work, n_work, nqt, group, zero_counter);
  return check_launch("order_work_kernel");
}
}  // namespace sa
