// internal.h — launch structs and helpers shared between translation units.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "sparseattn_b200.h"

namespace sa {

// Kernel attributes (cudaFuncSetAttribute) and the SM count belong to a device
// context, so one-time setup is remembered per device: `once_per_device(done,
// f)` runs f the first time the calling thread's current device is seen (two
// threads racing both run f, which is idempotent).
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}
template <class F>
inline void once_per_device(std::atomic<uint64_t>& done, F&& f) {
  const uint64_t bit = 1ull << (current_device() & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  f();
  done.fetch_or(bit, std::memory_order_acq_rel);
}
inline int device_sm_count() {
  static std::atomic<int> sms[64];
  const int dev = current_device();
  int v = sms[dev & 63].load(std::memory_order_relaxed);
  if (v == 0) {
    v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    sms[dev & 63].store(v, std::memory_order_relaxed);
  }
  return v;
}

struct TopkArgs {
  const float* scores;
  long long ld;          // row stride (elements)
  int rows;
  int n;                 // default row length
  const int32_t* lens;   // optional per-row length
  int k;                 // default k
  const int32_t* ks;     // optional per-row k
  int32_t* idx_out;      // optional [rows, out_ld]
  long long out_ld;
  int32_t* count_out;    // optional [rows]: number written
  uint32_t* bits;        // optional bitmap per row: bit (base + sign*j) set for kept j
  long long bits_ld;     // words per row
  int bit_base;
  int bit_neg;
  const int32_t* gate;   // optional: process row r only if gate[r / gate_div] == gate_val
  int gate_div;
  int gate_val;
  int gate_sparse;       // the gate is expected to keep few rows (auto layers): size the launch for that
  // optional second row set: rows r >= split use (scores2, k2, idx_out2, bits2,
  // bit_base2, bit_neg2) with local row r - split (same ld / out_ld / bits_ld)
  int split;
  const float* scores2;
  int k2;
  int32_t* idx_out2;
  long long out_ld2;
  uint32_t* bits2;
  int bit_base2;
  int bit_neg2;
  int smem_keys;  // set by launch_topk: rows up to this length are cached in shared memory
};

int launch_topk(const TopkArgs& a, cudaStream_t st);

// util.cu: *flag |= any non-finite bf16 among count values at x (flag not cleared)
int launch_check_finite(const void* x, long long count, int32_t* flag, cudaStream_t st);
// util.cu: finiteness scan of q (nq values), k and v (nkv values each, rows of
// `row` values) fused with the copy of k / v into cache rows of `cap` values
// per head (cache_k / cache_v may be null); flag as above
int launch_scan_fill(const void* q, long long nq, const void* k, const void* v, long long nkv, long long row,
                     void* cache_k, void* cache_v, long long cap, int32_t* flag, cudaStream_t st, bool chunked = false);

int launch_score_tail(int batch, int heads, int kv_heads, int n, float scale, const void* q,
                      const void* k, int r_lo, int r_hi, float* col_out, float* diag_out,
                      int accumulate, const int32_t* gate, int gate_val, void* ws, size_t ws_bytes,
                      cudaStream_t st);
size_t tail_workspace_bytes(int hh_total, int n, int r_hi);

int launch_block_pool(int groups, int n, int b, int side, const void* x, void* split_out,
                      float* mean_out, const int32_t* gate, int gate_val, cudaStream_t st);
size_t block_select_ws(int n, int b, int k_b, int hh_total);
int launch_fixed_row_off(int32_t* row_off, int hh_total, int nb, int stride, int row_stride, long long head_stride,
                         const int32_t* gate, int gate_val, cudaStream_t st);
// block_screen.cu: Block-Cluster index for k_b <= 8 (fp16 screen + exact refine)
size_t pool16_bytes(int groups, int nb);
size_t block_screen_ws(int nb, int k_b, int hh_total);
int launch_block_pool16(int groups, int n, int b, const void* x, void* pooled, bool key_side, const int32_t* gate,
                        int gate_val, cudaStream_t st);
int launch_block_screen(int batch, int heads, int kv_heads, int n, int b, int k_b, const void* qpool,
                        const void* kpool, int32_t* blk_idx, long long head_stride, int32_t* blk_row_off,
                        int row_stride, const int32_t* gate, int gate_val, void* ws, size_t ws_bytes,
                        cudaStream_t st);
int launch_block_select(int batch, int heads, int kv_heads, int n, int b, int k_b, float scale,
                        const void* qp, const void* kp, int32_t* blk_idx, long long head_stride,
                        int32_t* blk_row_off, int row_stride, const int32_t* gate, int gate_val,
                        void* ws, size_t ws_bytes, cudaStream_t st);
// sa_prefill's use of the selector: the last CTA of each head takes the
// argmin and writes the chosen full-length pattern's per-head parameters (no
// separate argmin / apply kernels); counter: [HH] ints, zeroed by launch_select
struct SelectApply {
  sa_pattern full[SA_MAX_CAND];
  int32_t* family;
  int32_t* tri_w;
  int32_t* tri_s;
  int32_t* blk_b;
  int* counter;
};
int launch_select(int batch, int heads, int kv_heads, int n, int cal, float scale, const void* q,
                  const void* k, int ncand, const int32_t* cand_fam, const int32_t* cand_p1,
                  const int32_t* cand_p2, int32_t* choice_out, int32_t* family_out,
                  double* err_out, cudaStream_t stream, const SelectApply* apply = nullptr);

int launch_attn(int batch, int heads, int kv_heads, int n, float scale, const void* q, const void* k,
                const void* v, void* out, const sa_head_index* index, const int32_t* tile_off,
                const int32_t* tile_cnt, const uint32_t* tiles, const int32_t* work, float* lse,
                cudaStream_t st, long long out_ld = 0, int* counter = nullptr,
                const int32_t* n_work = nullptr, void* const* peer_out = nullptr, int n_peers = 0,
                bool counter_zeroed = false);

// tiles.cu: heaviest-first order of the items with a nonzero cost; *n_work = their number
int launch_order_work(const int32_t* cost, int items, int max_cost, int32_t* work, int32_t* n_work,
                      cudaStream_t st, int nqt = 0, int group = 0, int32_t* zero_counter = nullptr);

}  // namespace sa
