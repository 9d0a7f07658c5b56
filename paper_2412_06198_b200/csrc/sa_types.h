// sa_types.h — device-side data layout shared by the kernels of the prefill
// sparse-attention path.
#pragma once
#include <cstdint>

#include "sparseattn_b200.h"

namespace sa {

// Pattern families, in the reference's DEFAULT_FAMILIES order
// (search.py:322): the selector's argmin index is the family id.
enum Family : int32_t { FAM_TRI = 0, FAM_VS = 1, FAM_BLOCK = 2, FAM_DENSE = 3,
                        FAM_VS_NOEYE = 5 /* VS index with always_diagonal=False */,
                        FAM_DENSE_NC = 6 /* non-causal dense (core.py:138-154, causal=False) */ };

// Per-tile mask kinds (bits 28..31 of a tile-list entry).
enum TileKind : uint32_t {
  TK_FULL = 0,    // every (i, j) of the 128x128 tile is included
  TK_CAUSAL = 1,  // j <= i
  TK_BAND = 2,    // Triangular: (i - j < window || j < sinks) && j <= i
  TK_VS = 3,      // column bitmap | diagonal bitmap | i == j, && j <= i
  TK_BLOCK = 4,   // (i/b, j/b) in the block list of the row's query block, && j <= i
  // Block-Cluster gather mode (b in {8,16,32,64}): the query tile's 128/b query
  // blocks each contribute one b-key slot to a gathered 128-key tile.
  TK_GATHER = 5,     // ktile field = rank g: slot s holds the g-th off-diagonal block of query block s
  TK_BLOCKDIAG = 6,  // kt == qt: only the row's own (diagonal) block, j <= i
  TK_LIMIT = 7,      // non-causal dense, last key tile: every key j < n
};

// Gather mode applies to block sides whose blocks are whole 8-row swizzle atoms
// and tile the 128-row query tile exactly.
__host__ __device__ inline bool block_gather_ok(int b) { return b >= 8 && b < 128 && 128 % b == 0; }

constexpr int kTile = 128;   // query rows and key rows per tile
constexpr int kHeadDim = 128;

__host__ __device__ inline uint32_t tile_entry(uint32_t ktile, uint32_t kind) {
  return ktile | (kind << 28);
}
__host__ __device__ inline uint32_t tile_ktile(uint32_t e) { return e & 0x0FFFFFFFu; }
__host__ __device__ inline uint32_t tile_kind(uint32_t e) { return e >> 28; }

// The device-resident realised index (C ABI struct, include/sparseattn_b200.h).
using HeadIndexView = sa_head_index;


}  // namespace sa
