// attn_mask.cuh — per-row masks of a listed 128-key tile, shared by the
// attention kernels (attn_fwd.cu, attn_pair.cu).  `Args` needs `n` (tokens)
// and `idx` (the device index, sa_types.h).  See attn_fwd.cu for the tile
// kinds and the reference semantics (patterns.py:113-133, 262-321, 353-484).
#pragma once
#include <cstdint>

#include "sa_types.h"
#include "sm100_common.cuh"

namespace sa {

// Per-row constants of the mask builders, loaded once per CTA.
struct RowConst {
  int b;             // Block-Cluster block side
  int ro_lo, ro_hi;  // the row's query-block entries in blk_idx
  int w, s;          // Triangular window / sinks
  bool eye;          // VS forced diagonal (patterns.py:378)
};

template <class Args>
__device__ __forceinline__ RowConst row_const(const Args& a, int hh, int i) {
  RowConst c;
  const int fam = a.idx.family[hh];
  c.b = a.idx.blk_b[hh];
  c.ro_lo = c.ro_hi = 0;
  if (fam == FAM_BLOCK && i < a.n) {
    const int32_t* ro = a.idx.blk_row_off + (size_t)hh * a.idx.blk_row_stride;
    c.ro_lo = ro[i / c.b];
    c.ro_hi = ro[i / c.b + 1];
  }
  c.w = a.idx.tri_window[hh];
  c.s = a.idx.tri_sinks[hh];
  c.eye = fam != FAM_VS_NOEYE;
  return c;
}

// Global words a tile's row mask needs, fetched one tile ahead so the load
// latency hides under the previous tile's softmax.
template <class Args>
__device__ __forceinline__ void mask_fetch(const Args& a, const RowConst& c, int hh, int i,
                                           uint32_t e, uint32_t (&raw)[9]) {
  const uint32_t kind = tile_kind(e);
  const int kt = (int)tile_ktile(e);
  if (i >= a.n) return;
  if (kind == TK_VS) {
    const int j0 = kt * kTile;
    const uint32_t* cb = a.idx.colbits + (size_t)hh * a.idx.vs_words + (j0 >> 5);
    const uint32_t* dr = a.idx.diagrev + (size_t)hh * a.idx.vs_words + ((a.n + 127 - i + j0) >> 5);
#pragma unroll
    for (int k = 0; k < 4; ++k) raw[k] = __ldg(cb + k);
#pragma unroll
    for (int k = 0; k < 5; ++k) raw[4 + k] = __ldg(dr + k);
  } else if (kind == TK_GATHER) {
    const int k = c.ro_lo + kt;
    raw[0] = k < c.ro_hi ? (uint32_t)__ldg(a.idx.blk_idx + k) : 0x7fffffffu;
  }
}

// The 128-bit row mask of tile entry e for query row i (registers only,
// except the rare union-mode Block tiles).
template <class Args>
__device__ __forceinline__ void mask_make(const Args& a, const RowConst& c, int i, int qt,
                                          uint32_t e, const uint32_t (&raw)[9], uint32_t (&m)[4]) {
  const uint32_t kind = tile_kind(e);
  const int kt = (int)tile_ktile(e);
  if (i >= a.n) {  // padding rows past n: any non-empty mask (finite logits), never stored
    m[0] = m[1] = m[2] = m[3] = 0xffffffffu;
    return;
  }
  m[0] = m[1] = m[2] = m[3] = 0u;
  const int j0 = kt * kTile;
  const int diag_c = i - j0;  // column (within tile) of the main diagonal
  if (kind == TK_CAUSAL) {
    mask_set_range(m, 0, diag_c + 1);
  } else if (kind == TK_GATHER) {
    // kt is the rank g; the row's query block owns slot s = gq - qt * 128 / b,
    // filled iff the block row has a g-th off-diagonal entry (all causal)
    const int gq = i / c.b;
    if ((int)raw[0] < gq) {
      const int s = gq - qt * (kTile / c.b);
      mask_set_range(m, s * c.b, s * c.b + c.b);
    }
  } else if (kind == TK_LIMIT) {
    mask_set_range(m, 0, a.n - j0);
  } else if (kind == TK_BLOCKDIAG) {
    mask_set_range(m, (i / c.b) * c.b - j0, diag_c + 1);
  } else if (kind == TK_BAND) {
    mask_set_range(m, diag_c - c.w + 1, diag_c + 1);
    mask_set_range(m, 0, min(c.s - j0, diag_c + 1));
  } else if (kind == TK_VS) {
    // window bit c <=> diag[i - j0 - c] <=> diagrev bit (n + 127 - i + j0 + c)
    const int sh = (a.n + 127 - i + j0) & 31;
#pragma unroll
    for (int k = 0; k < 4; ++k) m[k] = raw[k] | __funnelshift_r(raw[4 + k], raw[5 + k], sh);
    if (diag_c >= 0 && diag_c < 128 && c.eye) {
#pragma unroll
      for (int k = 0; k < 4; ++k) m[k] |= ((diag_c >> 5) == k) ? 1u << (diag_c & 31) : 0u;
    }
    if (kt == qt) {  // causal cut on the diagonal tile
      uint32_t c4[4] = {0u, 0u, 0u, 0u};
      mask_set_range(c4, 0, diag_c + 1);
#pragma unroll
      for (int k = 0; k < 4; ++k) m[k] &= c4[k];
    }
  } else if (kind == TK_BLOCK) {
    const int b = c.b;
    // rows are ascending key-block ids, possibly padded with INT32_MAX sentinels
    const int gfirst = j0 / b;                // first block ending after j0
    const int kend = (j0 + 128 + b - 1) / b;  // first block starting at/after j0 + 128
    int L = c.ro_lo, R = c.ro_hi;
    while (L < R) {
      int mid = (L + R) >> 1;
      if (a.idx.blk_idx[mid] >= gfirst) R = mid; else L = mid + 1;
    }
    for (int k = L; k < c.ro_hi; ++k) {
      const int gk = a.idx.blk_idx[k];
      if (gk >= kend) break;
      mask_set_range(m, gk * b - j0, (gk + 1) * b - j0);
    }
    uint32_t c4[4] = {0u, 0u, 0u, 0u};
    mask_set_range(c4, 0, diag_c + 1);
#pragma unroll
    for (int k = 0; k < 4; ++k) m[k] &= c4[k];
  } else {
    m[0] = m[1] = m[2] = m[3] = 0xffffffffu;
  }
}

}  // namespace sa
