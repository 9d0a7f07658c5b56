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

/* A pattern: Triangular(window=p1, sinks=p2) | VerticalSlash(k_v=p1, k_s=p2) |
 * BlockSparse(b=p1, k_b=p2) | dense (patterns.py:59-94). */
typedef struct {
  int32_t family; /* sa_family */
  int32_t p1, p2;
} sa_pattern;

/* Most candidates one auto-mode selection holds (cand / full below, the
 * [HH, SA_MAX_CAND] error rows of sa_prefill_view).  The reference's default
 * search space has 3 (search.py:322-357). */
#define SA_MAX_CAND 16

typedef enum { SA_MODE_DENSE = 0, SA_MODE_FIXED = 1, SA_MODE_AUTO = 2 } sa_prefill_mode;

/* One layer of runtime.prefill (runtime.py:134-206).  `cand` are the
 * refined candidates at window scale (search.py:236-241), `full` the same
 * candidates rescaled to n (search.py:261-273); the host computes both (pure
 * integer math) and the device picks one per head. */
typedef struct {
  int32_t batch, heads, kv_heads, n;
  float scale;           /* 1/sqrt(d_head) of the caller's head dim         */
  int32_t mode;          /* sa_prefill_mode                                  */
  sa_pattern fixed;      /* SA_MODE_FIXED                                    */
  int32_t q_est;         /* estimated-scoring rows (runtime.py:170)          */
  int32_t cal;           /* SA_MODE_AUTO: calibration window (<= 64)         */
  int32_t ncand;         /* SA_MODE_AUTO: 1..SA_MAX_CAND                     */
  sa_pattern cand[SA_MAX_CAND];
  sa_pattern full[SA_MAX_CAND];
  int32_t preselected;   /* SA_MODE_AUTO: 0 = run the selector inside
                            sa_prefill; 1 = the caller already wrote the per-head
                            choice into view.choice; 2 = sa_prefill_select already
                            selected and applied it (same workspace) */
  void* stage_events[6]; /* optional cudaEvent_t, recorded on `stream` after:
                            [0] selection, [1] VS estimator + top-k, [2] block
                            estimator, [3] tile lists, [4] attention, [5] unused */
  int64_t out_ld;        /* elements between output rows; 0 = heads * 128 (the
                            (B, L, H*d) layout of runtime.py:194).  A larger
                            value writes a head group into a wider layer output;
                            must be a multiple of 8 (16-byte output rows). */
  int32_t stop_after_tiles; /* 1 = selection, estimators and tile lists only (no
                               attention): the realised index of these heads,
                               e.g. for exchange between ranks (multigpu.py) */
  int32_t* check_flag;      /* optional device int: cleared, then set to 1 when q, k
                               or v holds a NaN / Inf (AttnMatrices, core.py:72-74).
                               The scan runs on a side stream beside the layer and
                               is joined before sa_prefill's work completes; the
                               caller reads the flag before using the outputs. */
  void* cache_k;            /* optional bf16 KvCache storage [B, HK, cache_capacity, 128]: */
  void* cache_v;            /* k / v rows 0..n-1 are copied in (runtime.py:197 cache.append) */
  int32_t cache_capacity;   /* on the same side stream as the scan (0 = no cache fill)    */
} sa_prefill_desc;

/* Device views into a prefill workspace (valid after sa_prefill). */
typedef struct {
  int32_t* choice;      /* [HH] chosen candidate (auto)                      */
  int32_t* family;      /* [HH]                                              */
  double* errors;       /* [HH, SA_MAX_CAND] window Frobenius errors (auto)  */
  float* col_scores;    /* [HH, n] estimated column mass (VS heads)          */
  float* diag_scores;   /* [HH, n] estimated diagonal mass (VS heads)        */
  int32_t* col_idx;     /* [HH, col_ld] selected columns, ascending          */
  int32_t* diag_idx;    /* [HH, diag_ld] selected diagonals, ascending       */
  int32_t col_ld, diag_ld;
  sa_head_index index;  /* the realised index of every head                  */
  int64_t blk_head_stride;
  int32_t* tile_off;
  int32_t* tile_cnt;
  uint32_t* tiles;
  int32_t nqt;
} sa_prefill_view;

const char* sa_last_error(void);
int sa_version(void);

/* ---- the whole path: runtime.prefill (runtime.py:134-206) --------------- */
size_t sa_prefill_workspace_size(const sa_prefill_desc* desc);
int sa_prefill_views(const sa_prefill_desc* desc, void* ws, sa_prefill_view* view);
/* The per-head selection of an SA_MODE_AUTO layer alone (search.py:276-319):
 * the windowed selector writes view.choice / view.errors and the chosen
 * patterns' per-head parameters; a following sa_prefill with preselected = 2
 * on the same workspace skips its own selection. */
int sa_prefill_select(const sa_prefill_desc* desc, const void* q, const void* k, void* ws, size_t ws_bytes,
                      void* stream);
int sa_prefill(const sa_prefill_desc* desc, const void* q, const void* k, const void* v,
               void* out, void* ws, size_t ws_bytes, void* stream);

/* AttnMatrices' finiteness check (core.py:72-74) on device: sets *flag to 1
 * if any of `count` bf16 values is NaN or Inf (flag is not cleared). */
int sa_check_finite_bf16(const void* x, long long count, int32_t* flag, void* stream);
/* cudaMemcpy2DAsync passthrough (kind = cudaMemcpyDefault) so host code can
 * move a head group's output columns without torch strided copies. */
/* fp32 <-> bf16 staging of host-API (numpy float32) layers: count elements,
 * round to nearest even; sa_f32_to_bf16 also sets *flag (nullable) to 1 if any
 * input is NaN/Inf (AttnMatrices' check, core.py:72-74, on the rows as given). */
int sa_f32_to_bf16(const float* x, void* y, long long count, int32_t* flag, void* stream);
int sa_bf16_to_f32(const void* x, float* y, long long count, void* stream);
int sa_memcpy2d_async(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                      size_t height, void* stream);

/* ---- selector: search.select_pattern_windowed (search.py:276-319) -------- */
/* Candidate arrays are HOST arrays of length ncand (refined at window scale).
 * choice_out / family_out: [HH]; err_out: [HH, SA_MAX_CAND] float64 (nullable). */
int sa_select_windowed(int batch, int heads, int kv_heads, int n, int cal, float scale,
                       const void* q, const void* k, int ncand, const int32_t* cand_fam_host,
                       const int32_t* cand_p1_host, const int32_t* cand_p2_host,
                       int32_t* choice_out, int32_t* family_out, double* err_out, void* stream);

/* ---- VS estimator: patterns.score_columns / score_diagonals
 *      (patterns.py:165-228), rows [r_lo, r_hi) with r_hi - r_lo <= 128 ----- */
size_t sa_score_tail_workspace(int batch, int heads, int n, int r_hi);
int sa_score_tail(int batch, int heads, int kv_heads, int n, float scale, const void* q,
                  const void* k, int r_lo, int r_hi, float* col_out, float* diag_out,
                  int accumulate, const int32_t* gate, int gate_val, void* ws, size_t ws_bytes,
                  void* stream);

/* ---- stable top-k: patterns._top_k_stable (patterns.py:231-234) ---------- */
/* Bit-exact given identical fp32 scores: k largest, ties to the lower index,
 * output ascending.  Rows are independent. */
int sa_topk_stable_f32(const float* scores, int rows, int n, long long ld, int k, int32_t* idx_out,
                       long long out_ld, void* stream);
/* Segmented variant: row r uses lens[r] scores and keeps ks[r]. */
int sa_topk_stable_rows_f32(const float* scores, int rows, long long ld, const int32_t* lens,
                            const int32_t* ks, int32_t* idx_out, long long out_ld,
                            int32_t* count_out, void* stream);

/* ---- pattern choice on given errors: search.py:245-250 ------------------- */
/* err [rows, ld] float64 (device): choice_out[r] = strict-< argmin over the
 * first ncand columns (earlier candidate wins ties, NaN never wins). */
int sa_select_family(const double* err, long long ld, int rows, int ncand, int32_t* choice_out, void* stream);

/* ---- block index from given fp32 block weights (patterns.py:309-321) ------ */
/* w [nb, ld] fp32 (device, row gq valid on columns 0..gq): blk_out [nb, k_b + 1]
 * = stable top-min(k_b, gq + 1) of row gq plus gq, ascending, INT32_MAX padded.
 * Bit-exact given identical fp32 weights. */
size_t sa_block_topk_workspace(int nb, int k_b);
int sa_block_topk_f32(const float* w, int nb, long long ld, int k_b, int32_t* blk_out, void* ws, size_t ws_bytes,
                      void* stream);

/* ---- Block estimator: patterns.block_mean / build_block_index
 *      (patterns.py:279-321) ------------------------------------------------ */
/* side 0 = query operand [hi|lo|hi] ([groups, nb, 384] bf16), side 1 = key
 * operand [hi|lo] ([groups, nb, 256] bf16); mean_out (nullable) [groups, nb, 128] fp32. */
int sa_block_pool(int groups, int n, int b, int side, const void* x, void* split_out,
                  float* mean_out, void* stream);
size_t sa_block_select_workspace(int n, int b, int k_b);
/* blk_idx: [HH, nb, k_b + 1] ascending rows padded with INT32_MAX;
 * blk_row_off: [HH, nb + 1] absolute offsets. */
int sa_block_select(int batch, int heads, int kv_heads, int n, int b, int k_b, float scale,
                    const void* qp, const void* kp, int32_t* blk_idx, int32_t* blk_row_off,
                    void* ws, size_t ws_bytes, void* stream);

/* Block-Cluster index for k_b <= 8 straight from bf16 q [B*H, n, 128] and k
 * [B*HK, n, 128] (replaces block_mean + build_block_index,
 * patterns.py:279-321; sa_prefill takes it under SA_BLOCK_SCREEN=1, its
 * default is the split-bf16 GEMM of sa_block_select): fp32 pooling, fp16
 * tcgen05 passes with a rigorous error bound (k_b = 1: a row-max pass, then a
 * pass collecting every logit within the bound of it; 2..8: one pass tracking
 * chunk maxima), exact fp64 re-scoring of every near-cut candidate.  Same row
 * layout as sa_block_select (scale-free: the positive 1/sqrt(d) does not
 * change a row's order). */
size_t sa_block_index_workspace(int batch, int heads, int kv_heads, int n, int b, int k_b);
int sa_block_index_bf16(int batch, int heads, int kv_heads, int n, int b, int k_b, const void* q, const void* k,
                        int32_t* blk_idx, int32_t* blk_row_off, void* ws, size_t ws_bytes, void* stream);

/* Dense [n, n] fp32 weights of head hh under `index` (need_weights=True of
 * patterns.py:422-434, 466-467; core.py:152), rows normalised by the lse that
 * sa_attn_sparse returned.  n <= 1048560 (the caller owns the n * n * 4 bytes). */
int sa_attn_weights(int heads, int kv_heads, int n, int hh, float scale, const void* q,
                    const void* k, const float* lse, const sa_head_index* index, float* w,
                    void* stream);
/* fp32 block_mean of an [n, d] matrix (patterns.py:279-287). */
int sa_block_mean_f32(const float* x, int n, int d, int b, float* out, void* stream);

/* ---- index -> executed tiles (patterns.py:113-158 field semantics) ------- */
/* Replaces the per-head structural iteration of vertical_slash_attention /
 * block_sparse_attention (patterns.py:353-484).  tile_off/tile_cnt: [HH*nqt],
 * tiles: capacity HH*nqt*(nqt+1)/2 entries (entry = key_tile | kind << 28). */
int sa_build_tiles(const sa_head_index* index, int hh_total, int n, int32_t* tile_off,
                   int32_t* tile_cnt, uint32_t* tiles, void* stream);

/* ---- sparse attention (patterns.py:487-497 sparse_attention, need_weights=False;
 *      core.py:138-154 dense_attention when family == SA_DENSE) ------------- */
/* lse (nullable): [HH, n] natural-log row log-sum-exp of the realised logits. */
/* Launch order for sa_attn_sparse's CTAs: work[r] = index (into tile_cnt) of
 * the item with the r-th largest tile count (longest-processing-time first).
 * No reference counterpart: the reference runs heads serially (runtime.py:174). */
int sa_order_work(const int32_t* tile_cnt, int items, int max_cnt, int32_t* work, void* stream);
/* One decode step (reference runtime.py:209-242 decode_step): the new token's
 * queries q [batch * heads, d] fp32 attend densely over the first n rows of a
 * KV cache laid out [batch, kv_heads, capacity, d] (kv_dtype 0 = fp32,
 * 1 = bf16), out [batch * heads, d] fp32.  Split-K over 256-1024-key chunks, K/V
 * read in place once per kv head; n <= 8388608; ws >= sa_decode_workspace(...). */
size_t sa_decode_workspace(int batch, int heads, int kv_heads, int n, int d);
int sa_decode_attn(int batch, int heads, int kv_heads, int n, int d, int capacity, float scale, const float* q,
                   const void* k_cache, const void* v_cache, int kv_dtype, float* out, void* ws, size_t ws_bytes,
                   void* stream);

int sa_attn_sparse(int batch, int heads, int kv_heads, int n, float scale, const void* q,
                   const void* k, const void* v, void* out, const sa_head_index* index,
                   const int32_t* tile_off, const int32_t* tile_cnt, const uint32_t* tiles,
                   float* lse, void* stream);
/* sa_attn_sparse over an explicit work list: items work[0 .. *n_work) (device
 * int32, item = (b * heads + h) * nqt + query tile) in that order; other query
 * tiles are not written.  `counter` is one device int32 of scratch per
 * concurrent call.  Used by the balanced head-parallel path (multigpu.py). */
int sa_attn_sparse_work(int batch, int heads, int kv_heads, int n, float scale, const void* q, const void* k,
                        const void* v, void* out, const sa_head_index* index, const int32_t* tile_off,
                        const int32_t* tile_cnt, const uint32_t* tiles, const int32_t* work,
                        const int32_t* n_work, int32_t* counter, long long out_ld, void* stream);

/* Fused output all-gather for the head-parallel layer (the
 * reference has no multi-GPU path, runtime.py:174-195 runs heads serially; the
 * north star names an NVLink all-gather of per-head outputs).  Same as
 * sa_attn_sparse_work, plus: every output row the kernel produces is also
 * stored, from the epilogue, at the same offset into each of the `n_peers`
 * (<= 7) buffers in `peer_out` — other ranks' output buffers mapped with
 * sa_ipc_open — so no separate all-gather follows.  The caller orders the
 * peers' reads after this kernel with sa_peer_barrier on the same stream. */
int sa_attn_sparse_work_peers(int batch, int heads, int kv_heads, int n, float scale, const void* q,
                              const void* k, const void* v, void* out, void* const* peer_out, int n_peers,
                              const sa_head_index* index, const int32_t* tile_off, const int32_t* tile_cnt,
                              const uint32_t* tiles, const int32_t* work, const int32_t* n_work,
                              int32_t* counter, long long out_ld, void* stream);

/* CUDA IPC helpers for the peer buffers: sa_ipc_alloc allocates `bytes` of
 * device memory and writes its SA_IPC_HANDLE_BYTES-byte handle; another
 * process maps it with sa_ipc_open (same or peer GPU) and unmaps it with
 * sa_ipc_close; the owner frees it with sa_ipc_free. */
#define SA_IPC_HANDLE_BYTES 64
int sa_ipc_alloc(size_t bytes, void** ptr, void* handle);
int sa_ipc_free(void* ptr);
int sa_ipc_open(const void* handle, void** ptr);
int sa_ipc_close(void* ptr);

/* Device-side barrier of `world` ranks over IPC-mapped flag buffers (no host
 * synchronisation; capturable in a CUDA graph).  `flags` is this rank's
 * buffer of world + 1 zero-initialised int32 (slot r = rank r's last epoch,
 * slot world = this rank's epoch counter); `peer_flags` are the other
 * world - 1 ranks' buffers mapped with sa_ipc_open.  One thread bumps the
 * epoch, fences (system scope: every earlier write on the stream, including
 * sa_attn_sparse_work_peers' stores into peer outputs, is visible before the
 * flag), writes the epoch into slot `rank` of every peer with a system-scope
 * release and waits (acquire) until every other rank's slot of `flags` holds
 * it.  Work queued after it on `stream` sees every rank's writes issued
 * before their barrier.  A rank that does not arrive within `timeout_ms`
 * traps the kernel (a CUDA error, not a hang). */
int sa_peer_barrier(int32_t* flags, void* const* peer_flags, int rank, int world, int timeout_ms, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SPARSEATTN_B200_H_ */
