/*
 * sparseattn_b200.h — C ABI of the B200-native prefill sparse-attention path
 * (SparseAccelerate, arXiv 2412.06198).  Drop-in boundary for the reference's
 * Python package `sparseattn` (/root/reference/pkg/src/sparseattn).
 *
 * Conventions:
 *   - every pointer argument is a DEVICE pointer unless its name ends in _host;
 *   - `stream` is a cudaStream_t passed as void*; all calls are stream-ordered
 *     and asynchronous unless documented otherwise; no call frees caller memory;
 *   - tensors are row-major; q is [B, H, n, 128] bf16, k and v are [B, HK, n, 128]
 *     bf16 (HK divides H: the GQA extension of runtime.py:119-131), head_dim is
 *     fixed at 128 (the host mirror zero-pads smaller head dims and passes the
 *     original 1/sqrt(d) as `scale`);
 *   - outputs use the reference layout (B, n, H * 128) (runtime.py:194);
 *   - every entry point returns an sa_status; a non-zero status maps 1:1 to the
 *     reference exception class named below and sa_last_error() returns the
 *     message of the last failure on the calling thread.
 */
#ifndef SPARSEATTN_B200_H_
#define SPARSEATTN_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SA_OK = 0,
  SA_ERR_DIMENSION = 1,       /* core.DimensionError        (core.py:36)     */
  SA_ERR_NONFINITE = 2,       /* core.NonFiniteError        (core.py:40)     */
  SA_ERR_EMPTY_ROW = 3,       /* core.EmptyRowError         (core.py:44)     */
  SA_ERR_PATTERN_PARAM = 4,   /* patterns.PatternParamError (patterns.py:55) */
  SA_ERR_SEARCH = 5,          /* search.SearchError         (search.py:47)   */
  SA_ERR_CACHE_OVERFLOW = 6,  /* runtime.CacheOverflowError (runtime.py:35)  */
  SA_ERR_GENERIC = 7,         /* core.SparseAttnError       (core.py:32)     */
  SA_ERR_CUDA = 100,          /* launch / driver failure                     */
} sa_status;

/* Family ids = index into the reference's DEFAULT_FAMILIES (search.py:322). */
typedef enum { SA_TRIANGULAR = 0, SA_VERTICAL_SLASH = 1, SA_BLOCK_SPARSE = 2, SA_DENSE = 3 } sa_family;

/* Device-resident realised index for HH = B * H heads (patterns.py:113-158
 * SparseIndex, one per head).  See sa_types.h / DESIGN.md for the encodings. */
typedef struct {
  const int32_t* family;      /* [HH] sa_family                                   */
  const int32_t* tri_window;  /* [HH] Triangular band width                       */
  const int32_t* tri_sinks;   /* [HH] Triangular sink columns                     */
  const uint32_t* colbits;    /* [HH, vs_words] column bitmap (bit j: column j)   */
  const uint32_t* diagrev;    /* [HH, vs_words] bit (n+127-o): diagonal offset o  */
  int32_t vs_words;           /* >= (n + 256) / 32 + 2                            */
  const int32_t* blk_b;       /* [HH] block side b                                */
  const int32_t* blk_row_off; /* [HH, blk_row_stride] CSR row offsets per q-block */
  const int32_t* blk_idx;     /* key blocks, ascending within a row, incl. gq     */
  int32_t blk_row_stride;     /* >= ceil(n / b) + 1 for every block head          */
} sa_head_index;

const char* sa_last_error(void);
int sa_version(void);

/* ---- index -> executed tiles (patterns.py:113-158 field semantics) ------- */
/* Replaces the per-head structural iteration of vertical_slash_attention /
 * block_sparse_attention (patterns.py:353-484).  tile_off/tile_cnt: [HH*nqt],
 * tiles: capacity HH*nqt*(nqt+1)/2 entries (entry = key_tile | kind << 28). */
int sa_build_tiles(const sa_head_index* index, int hh_total, int n, int32_t* tile_off,
                   int32_t* tile_cnt, uint32_t* tiles, void* stream);

/* ---- sparse attention (patterns.py:487-497 sparse_attention, need_weights=False;
 *      core.py:138-154 dense_attention when family == SA_DENSE) ------------- */
int sa_attn_sparse(int batch, int heads, int kv_heads, int n, float scale, const void* q,
                   const void* k, const void* v, void* out, const sa_head_index* index,
                   const int32_t* tile_off, const int32_t* tile_cnt, const uint32_t* tiles,
                   float* lse, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SPARSEATTN_B200_H_ */
