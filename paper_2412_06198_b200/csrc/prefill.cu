// prefill.cu — the whole prefill sparse-attention path of one layer on device.
//
// Reference: runtime.py:134-206 (prefill).  The reference loops over
// (batch, head): select (auto) -> build_index(estimated, q_est) -> kernel.
// Here every stage runs for all heads at once, stream-ordered, with no host
// synchronisation: the per-head choice lives in device memory and gates the
// estimator launches.
//
//   [auto]  select_kernel            -> choice[HH], family[HH], errors[HH, SA_MAX_CAND]
//   apply_choice_kernel              -> family / Triangular params / block side per head
//   [VS]    score_tail (gated)       -> col[HH, n], diag[HH, n]
//           topk (gated per cand)    -> column bitmap, reversed diagonal bitmap, id lists
//   [Block] pool Q (gated), pool K   -> split-bf16 operands
//           block_select (gated)     -> fixed-stride block rows
//   build_tiles                      -> executed (q-tile, k-tile) lists
//   attn_fwd                         -> out (B, n, H * 128)
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <cstdlib>

#include "api_common.h"
#include "internal.h"
#include "sa_types.h"

namespace sa {

static size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// Per-thread, per-device side stream and fork / join events (created on the
// first call that needs them; the warm-up run before a graph capture does).
struct SideStream {
  cudaStream_t s = nullptr, s2 = nullptr;
  cudaEvent_t fork0 = nullptr, kdone = nullptr, fork = nullptr, join = nullptr, fork2 = nullptr, join2 = nullptr;
};
static SideStream* side_stream() {
  static thread_local SideStream tab[16];
  int dev = 0;
  cudaGetDevice(&dev);
  SideStream& x = tab[dev & 15];
  if (!x.s) {
    // the estimator side stream runs at the device's top priority, so the VS
    // chain's CTAs claim SMs ahead of the block chain's and its latency-bound
    // kernels finish early (32K auto layer: VS chain done 101 vs 202 us after
    // selection, layer 1.115 vs 1.119 ms; SA_SIDE_PRIO=0: default priority)
    static const bool hi = [] {
      const char* e = getenv("SA_SIDE_PRIO");
      return !(e && e[0] == '0');
    }();
    int lo_p = 0, hi_p = 0;
    cudaDeviceGetStreamPriorityRange(&lo_p, &hi_p);
    cudaStreamCreateWithPriority(&x.s, cudaStreamNonBlocking, hi ? hi_p : 0);
    cudaStreamCreateWithFlags(&x.s2, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&x.fork2, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&x.join2, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&x.fork0, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&x.kdone, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming);
  }
  return &x;
}

struct Layout {
  size_t off[32];
  size_t total;
};

enum WsSlot {
  W_CHOICE = 0, W_FAMILY, W_ERR, W_TRIW, W_TRIS, W_COLBITS, W_DIAGREV, W_COLSC, W_DIAGSC,
  W_COLIDX, W_DIAGIDX, W_TAIL, W_BLKB, W_ROWOFF, W_BLKIDX, W_QP, W_KP, W_BLKWS,
  W_TOFF, W_TCNT, W_TILES, W_WORK, W_SELCNT, W_NUM
};

struct Plan {
  int hh, hk, n, nqt;
  int ncand;
  sa_pattern cand[SA_MAX_CAND];  // patterns at full n (clamped like build_index)
  int q_est;
  int vs_words;
  int any_vs, any_block;
  int max_kv, max_ks;
  int max_nb, blk_row_stride;
  long long blk_head_stride;
  size_t tail_ws, blk_ws, qp_elems, kp_elems;
  int tail_groups;
};

static int clamp_pattern(const sa_pattern& in, int n, sa_pattern* out) {
  // build_index clamps to n (patterns.py:324-343) and the index builders
  // validate the clamped values (patterns.py:237-321)
  *out = in;
  if (in.family == SA_TRIANGULAR) {
    out->p1 = std::min(in.p1, n);
    out->p2 = std::min(in.p2, n);
    if (out->p1 < 1 || out->p2 < 0)
      return fail(SA_ERR_PATTERN_PARAM, "window must be >= 1 and sinks >= 0");
  } else if (in.family == SA_VERTICAL_SLASH) {
    out->p1 = std::min(in.p1, n);
    out->p2 = std::min(in.p2, n);
    if (out->p1 < 1 || out->p2 < 1) return fail(SA_ERR_PATTERN_PARAM, "k_v and k_s must be >= 1");
  } else if (in.family == SA_BLOCK_SPARSE) {
    if (in.p1 < 1 || in.p2 < 1) return fail(SA_ERR_PATTERN_PARAM, "b and k_b must be >= 1");
    out->p1 = std::min(in.p1, n);
    const int nb = (n + out->p1 - 1) / out->p1;
    out->p2 = std::min(in.p2, nb);
  } else if (in.family != SA_DENSE) {
    return fail(SA_ERR_PATTERN_PARAM, "unknown pattern family %d", in.family);
  }
  return SA_OK;
}

// SA_BLOCK_SCREEN=1: Block-Cluster candidates with k_b <= 8 take the fp16
// paths of block_screen.cu (k_b = 1, the auto search's Block(8, 1): two fp16
// passes + exact refine; 2..8: one fp16 pass tracking chunk maxima + exact
// refine) instead of the split-bf16 GEMM of estimate_block.cu.  Opt-in: both
// measured slower than the split GEMM at 32K ("Block estimator:
// fp16 screen"); kept for A/B and as the sa_block_index_bf16 path.
static bool use_block_screen(int k_b) {
  static const bool on = [] {
    const char* e = getenv("SA_BLOCK_SCREEN");
    return e && e[0] == '1';
  }();
  return on && k_b <= 8;
}

static int make_plan(const sa_prefill_desc* d, Plan* p, Layout* L) {
  if (!d) return fail(SA_ERR_DIMENSION, "null descriptor");
  if (d->batch < 1 || d->heads < 1 || d->kv_heads < 1 || d->n < 1)
    return fail(SA_ERR_DIMENSION, "need batch, heads, kv_heads, n >= 1");
  if (d->heads % d->kv_heads)
    return fail(SA_ERR_DIMENSION, "heads=%d not a multiple of kv_heads=%d", d->heads, d->kv_heads);
  if (d->n > 262144) return fail(SA_ERR_DIMENSION, "n=%d exceeds 262144", d->n);
  if (!(d->scale > 0.f) || !std::isfinite(d->scale)) return fail(SA_ERR_DIMENSION, "bad scale");
  if (d->out_ld != 0 && d->out_ld < (int64_t)d->heads * kHeadDim)
    return fail(SA_ERR_DIMENSION, "out_ld=%lld is below heads * 128", (long long)d->out_ld);
  if (d->out_ld % 8 != 0)
    return fail(SA_ERR_DIMENSION, "out_ld=%lld must be a multiple of 8 (16-byte rows)", (long long)d->out_ld);
  memset(p, 0, sizeof(*p));
  const int n = d->n;
  p->hh = d->batch * d->heads;
  p->hk = d->batch * d->kv_heads;
  p->n = n;
  p->nqt = (n + kTile - 1) / kTile;
  p->vs_words = (n + 256) / 32 + 2;
  int rc;
  if (d->mode == SA_MODE_DENSE) {
    p->ncand = 1;
    p->cand[0] = sa_pattern{SA_DENSE, 0, 0};
  } else if (d->mode == SA_MODE_FIXED) {
    p->ncand = 1;
    if ((rc = clamp_pattern(d->fixed, n, &p->cand[0]))) return rc;
  } else if (d->mode == SA_MODE_AUTO) {
    if (d->ncand < 1 || d->ncand > SA_MAX_CAND)
      return fail(SA_ERR_SEARCH, "candidate list must hold 1..%d patterns", SA_MAX_CAND);
    if (d->cal < 1 || d->cal > n) return fail(SA_ERR_SEARCH, "cal_window must be in [1, %d]", n);
    p->ncand = d->ncand;
    for (int c = 0; c < d->ncand; ++c) {
      if (d->cand[c].family != d->full[c].family) return fail(SA_ERR_SEARCH, "cand/full family mismatch");
      if ((rc = clamp_pattern(d->full[c], n, &p->cand[c]))) return rc;
    }
  } else {
    return fail(SA_ERR_GENERIC, "unknown prefill mode %d", d->mode);
  }
  p->q_est = std::min(std::max(d->q_est, 1), n);
  p->max_kv = p->max_ks = 1;
  p->max_nb = 1;
  long long head_stride = 1;
  size_t blk_ws = 256;
  for (int c = 0; c < p->ncand; ++c) {
    const sa_pattern& pt = p->cand[c];
    if (pt.family == SA_VERTICAL_SLASH) {
      p->any_vs = 1;
      p->max_kv = std::max(p->max_kv, pt.p1);
      p->max_ks = std::max(p->max_ks, pt.p2);
    } else if (pt.family == SA_BLOCK_SPARSE) {
      p->any_block = 1;
      const int nb = (n + pt.p1 - 1) / pt.p1;
      p->max_nb = std::max(p->max_nb, nb);
      head_stride = std::max(head_stride, (long long)nb * (pt.p2 + 1));
      blk_ws = std::max(blk_ws, block_select_ws(n, pt.p1, pt.p2, p->hh));
      if (use_block_screen(pt.p2)) blk_ws = std::max(blk_ws, block_screen_ws(nb, pt.p2, p->hh));
    }
  }
  // block rows are addressed with int32 offsets (hh * head_stride + row * stride)
  if ((long long)p->hh * head_stride > INT32_MAX)
    return fail(SA_ERR_DIMENSION, "block index of %d heads x %lld entries exceeds the int32 row offsets",
                p->hh, head_stride);
  p->blk_row_stride = p->max_nb + 1;
  p->blk_head_stride = head_stride;
  p->blk_ws = blk_ws;
  p->tail_groups = (p->q_est + 127) / 128;
  const int r_hi_max = n;
  p->tail_ws = p->any_vs ? tail_workspace_bytes(p->hh, n, r_hi_max) : 256;
  // pooled blocks: split-bf16 operands (k_b > 8) or the fp16-screen layout (k_b <= 8), whichever is larger
  p->qp_elems = p->any_block ? std::max((size_t)p->hh * p->max_nb * 384, pool16_bytes(p->hh, p->max_nb) / 2) : 128;
  p->kp_elems = p->any_block ? std::max((size_t)p->hk * p->max_nb * 256, pool16_bytes(p->hk, p->max_nb) / 2) : 128;

  size_t sz[W_NUM];
  const size_t hh = p->hh;
  sz[W_CHOICE] = hh * 4;
  sz[W_FAMILY] = hh * 4;
  sz[W_ERR] = hh * SA_MAX_CAND * 8;
  sz[W_TRIW] = hh * 4;
  sz[W_TRIS] = hh * 4;
  sz[W_COLBITS] = hh * p->vs_words * 4;
  sz[W_DIAGREV] = hh * p->vs_words * 4;
  sz[W_COLSC] = p->any_vs ? hh * n * 4 : 4;
  sz[W_DIAGSC] = p->any_vs ? hh * n * 4 : 4;
  sz[W_COLIDX] = p->any_vs ? hh * p->max_kv * 4 : 4;
  sz[W_DIAGIDX] = p->any_vs ? hh * p->max_ks * 4 : 4;
  sz[W_TAIL] = p->tail_ws;
  sz[W_BLKB] = hh * 4;
  sz[W_ROWOFF] = hh * p->blk_row_stride * 4;
  sz[W_BLKIDX] = p->any_block ? hh * (size_t)p->blk_head_stride * 4 : 4;
  sz[W_QP] = p->qp_elems * 2;
  sz[W_KP] = p->kp_elems * 2;
  sz[W_BLKWS] = p->blk_ws;
  sz[W_TOFF] = hh * p->nqt * 4;
  sz[W_TCNT] = hh * p->nqt * 4;
  sz[W_TILES] = hh * (size_t)p->nqt * (p->nqt + 1) / 2 * 4;
  sz[W_WORK] = (64 + hh * p->nqt) * 4;  // [counter, item count], then the work order
  sz[W_SELCNT] = hh * 4;                // selector: candidate CTAs finished per head
  size_t o = 0;
  for (int i = 0; i < W_NUM; ++i) {
    L->off[i] = o;
    o += align_up(sz[i]);
  }
  L->total = o;
  return SA_OK;
}

struct ApplyArgs {
  int hh;
  int ncand;
  sa_pattern cand[SA_MAX_CAND];
  const int32_t* choice;  // null -> candidate 0 for every head
  int32_t* family;
  int32_t* tri_w;
  int32_t* tri_s;
  int32_t* blk_b;
};

__global__ void apply_choice_kernel(ApplyArgs a) {
  const int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= a.hh) return;
  const int c = a.choice ? a.choice[h] : 0;
  const sa_pattern p = a.cand[c];
  a.family[h] = p.family;
  a.tri_w[h] = p.family == SA_TRIANGULAR ? p.p1 : 1;
  a.tri_s[h] = p.family == SA_TRIANGULAR ? p.p2 : 0;
  a.blk_b[h] = p.family == SA_BLOCK_SPARSE ? p.p1 : 1;
}

}  // namespace sa

using namespace sa;

extern "C" size_t sa_prefill_workspace_size(const sa_prefill_desc* desc) {
  Plan p;
  Layout L;
  if (make_plan(desc, &p, &L)) return 0;
  return L.total;
}

extern "C" int sa_prefill_views(const sa_prefill_desc* desc, void* ws, sa_prefill_view* v) {
  Plan p;
  Layout L;
  int rc;
  if ((rc = make_plan(desc, &p, &L))) return rc;
  if (!v) return fail(SA_ERR_DIMENSION, "null view");
  char* b = reinterpret_cast<char*>(ws);
  v->choice = reinterpret_cast<int32_t*>(b + L.off[W_CHOICE]);
  v->family = reinterpret_cast<int32_t*>(b + L.off[W_FAMILY]);
  v->errors = reinterpret_cast<double*>(b + L.off[W_ERR]);
  v->col_scores = reinterpret_cast<float*>(b + L.off[W_COLSC]);
  v->diag_scores = reinterpret_cast<float*>(b + L.off[W_DIAGSC]);
  v->col_idx = reinterpret_cast<int32_t*>(b + L.off[W_COLIDX]);
  v->diag_idx = reinterpret_cast<int32_t*>(b + L.off[W_DIAGIDX]);
  v->col_ld = p.max_kv;
  v->diag_ld = p.max_ks;
  v->index.family = v->family;
  v->index.tri_window = reinterpret_cast<int32_t*>(b + L.off[W_TRIW]);
  v->index.tri_sinks = reinterpret_cast<int32_t*>(b + L.off[W_TRIS]);
  v->index.colbits = reinterpret_cast<uint32_t*>(b + L.off[W_COLBITS]);
  v->index.diagrev = reinterpret_cast<uint32_t*>(b + L.off[W_DIAGREV]);
  v->index.vs_words = p.vs_words;
  v->index.blk_b = reinterpret_cast<int32_t*>(b + L.off[W_BLKB]);
  v->index.blk_row_off = reinterpret_cast<int32_t*>(b + L.off[W_ROWOFF]);
  v->index.blk_idx = reinterpret_cast<int32_t*>(b + L.off[W_BLKIDX]);
  v->index.blk_row_stride = p.blk_row_stride;
  v->blk_head_stride = p.blk_head_stride;
  v->tile_off = reinterpret_cast<int32_t*>(b + L.off[W_TOFF]);
  v->tile_cnt = reinterpret_cast<int32_t*>(b + L.off[W_TCNT]);
  v->tiles = reinterpret_cast<uint32_t*>(b + L.off[W_TILES]);
  v->nqt = p.nqt;
  return SA_OK;
}

// The windowed selector (search.py:276-319) over the refined candidates, its
// last CTA per head taking the argmin and writing the chosen full-length
// pattern's per-head parameters into the workspace views.
static int select_apply(const sa_prefill_desc* desc, const Plan& p, const Layout& L, const sa_prefill_view& V,
                        char* b, const void* q, const void* k, cudaStream_t st) {
  int32_t fam[SA_MAX_CAND], p1[SA_MAX_CAND], p2[SA_MAX_CAND];
  for (int c = 0; c < p.ncand; ++c) {
    fam[c] = desc->cand[c].family;
    p1[c] = desc->cand[c].p1;
    p2[c] = desc->cand[c].p2;
  }
  SelectApply ap{};
  for (int c = 0; c < p.ncand; ++c) ap.full[c] = p.cand[c];
  ap.family = V.family;
  ap.tri_w = const_cast<int32_t*>(V.index.tri_window);
  ap.tri_s = const_cast<int32_t*>(V.index.tri_sinks);
  ap.blk_b = const_cast<int32_t*>(V.index.blk_b);
  ap.counter = reinterpret_cast<int*>(b + L.off[W_SELCNT]);
  return launch_select(desc->batch, desc->heads, desc->kv_heads, p.n, std::min(desc->cal, p.n), desc->scale, q, k,
                       p.ncand, fam, p1, p2, V.choice, nullptr, V.errors, st, &ap);
}

extern "C" int sa_prefill_select(const sa_prefill_desc* desc, const void* q, const void* k, void* ws,
                                 size_t ws_bytes, void* stream) {
  Plan p;
  Layout L;
  int rc;
  if ((rc = make_plan(desc, &p, &L))) return rc;
  if (desc->mode != SA_MODE_AUTO) return fail(SA_ERR_SEARCH, "sa_prefill_select needs SA_MODE_AUTO");
  if (!q || !k || !ws) return fail(SA_ERR_DIMENSION, "null pointer argument");
  if (ws_bytes < L.total) return fail(SA_ERR_DIMENSION, "workspace too small (%zu < %zu)", ws_bytes, L.total);
  sa_prefill_view V;
  sa_prefill_views(desc, ws, &V);
  return select_apply(desc, p, L, V, reinterpret_cast<char*>(ws), q, k, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int sa_prefill(const sa_prefill_desc* desc, const void* q, const void* k, const void* v,
                          void* out, void* ws, size_t ws_bytes, void* stream) {
  Plan p;
  Layout L;
  int rc;
  if ((rc = make_plan(desc, &p, &L))) return rc;
  if (!q || !k || !v || !out || !ws) return fail(SA_ERR_DIMENSION, "null pointer argument");
  if (ws_bytes < L.total) return fail(SA_ERR_DIMENSION, "workspace too small (%zu < %zu)", ws_bytes, L.total);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  sa_prefill_view V;
  sa_prefill_views(desc, ws, &V);
  char* b = reinterpret_cast<char*>(ws);
  const int n = p.n;
  const int B = desc->batch, H = desc->heads, HK = desc->kv_heads;

  // AttnMatrices' finiteness scan (core.py:72-74) of q, k, v and the KvCache
  // fill (runtime.py:197): one HBM-bound kernel on a second side stream,
  // joined before this call's work completes.  By default it runs beside the
  // attention (which moves ~1 TB/s of its 8): 128-thread CTAs that fit into
  // the registers two attention CTAs leave on an SM, the attention launched
  // at top priority so it claims SMs first (32K auto layer: +25 us over no
  // scan / fill, against +55 us beside the estimators).
  const bool fill = desc->cache_capacity > 0 && desc->cache_k && desc->cache_v;
  if (fill && desc->cache_capacity < n)
    return fail(SA_ERR_CACHE_OVERFLOW, "cache of capacity %d cannot hold %d rows", desc->cache_capacity, n);
  static const int chk_mode = [] {
    const char* e = getenv("SA_CHECK_MODE");  // A/B: 0 both, 1 no scan, 2 no fill, 3 neither
    return e ? atoi(e) : 0;
  }();
  // Placement (SA_SCAN_AT): 0 = grid-stride kernel from the start, joined
  // before the attention; 1 = short-CTA kernel from the start, joined after
  // the attention; 2 = short-CTA kernel forked beside the attention (whose
  // persistent CTAs leave room for one per SM and launch at top priority).
  static const int scan_at = [] {
    const char* e = getenv("SA_SCAN_AT");
    return e ? atoi(e) : 2;
  }();
  SideStream* chk = (desc->check_flag || fill) ? side_stream() : nullptr;
  auto fork_scan = [&](bool chunked) -> int {
    cudaEventRecord(chk->fork2, st);
    cudaStreamWaitEvent(chk->s2, chk->fork2, 0);
    if (desc->check_flag) cudaMemsetAsync(desc->check_flag, 0, sizeof(int32_t), chk->s2);
    const long long nq = (long long)p.hh * n * kHeadDim, nkv = (long long)p.hk * n * kHeadDim;
    const int r = launch_scan_fill(q, (chk_mode & 1) ? 0 : nq, k, v, nkv, (long long)n * kHeadDim,
                                   (fill && !(chk_mode & 2)) ? desc->cache_k : nullptr,
                                   (fill && !(chk_mode & 2)) ? desc->cache_v : nullptr,
                                   (long long)std::max(desc->cache_capacity, 1) * kHeadDim, desc->check_flag,
                                   chk->s2, chunked);
    cudaEventRecord(chk->join2, chk->s2);
    return r;
  };
  if (chk && scan_at != 2 && (rc = fork_scan(scan_at == 1))) return rc;
  // The single Block-Cluster candidate's key pooling needs only K: it runs on
  // the side stream from the start, beside the selector.
  static const bool overlap = [] {
    const char* e = getenv("SA_OVERLAP_EST");
    return !(e && e[0] == '0');
  }();
  int nblk = 0, blk_c = -1;
  for (int c = 0; c < p.ncand; ++c)
    if (p.cand[c].family == SA_BLOCK_SPARSE) ++nblk, blk_c = c;
  SideStream* side = (overlap && p.any_block && (p.any_vs || nblk == 1)) ? side_stream() : nullptr;
  // Session 4: with the VS chain on a top-priority side stream and a 16 us
  // selector, the key pooling goes after the selection on the caller's stream
  // (32K layer 1.0835-1.0846 -> 1.0787-1.0821 ms); SA_KPOOL_EARLY=1 runs it on
  // the side stream from the start, beside the selector, as before.
  static const bool kpool_env = [] {
    const char* e = getenv("SA_KPOOL_EARLY");
    return e && e[0] == '1';
  }();
  const bool kpool_early = side && nblk == 1 && kpool_env;
  if (kpool_early) {
    cudaEventRecord(side->fork0, st);
    cudaStreamWaitEvent(side->s, side->fork0, 0);
    if (use_block_screen(p.cand[blk_c].p2))
      rc = launch_block_pool16(p.hk, n, p.cand[blk_c].p1, k, b + L.off[W_KP], true, nullptr, 0, side->s);
    else
      rc = launch_block_pool(p.hk, n, p.cand[blk_c].p1, 1, k, b + L.off[W_KP], nullptr, nullptr, 0, side->s);
    if (rc) return rc;
    cudaEventRecord(side->kdone, side->s);
  }
  // 1. per-head choice: preselected 0 = the selector runs here (its last CTA
  // per head applies the choice), 2 = sa_prefill_select already did that,
  // 1 = the caller wrote view.choice (composed wide-window selection): apply it
  int32_t* choice = nullptr;
  if (desc->mode == SA_MODE_AUTO) {
    choice = V.choice;
    if (desc->preselected == 0 && (rc = select_apply(desc, p, L, V, b, q, k, st))) return rc;
  }
  if (desc->mode != SA_MODE_AUTO || desc->preselected == 1) {
    ApplyArgs a{};
    a.hh = p.hh;
    a.ncand = p.ncand;
    for (int c = 0; c < p.ncand; ++c) a.cand[c] = p.cand[c];
    a.choice = choice;
    a.family = V.family;
    a.tri_w = const_cast<int32_t*>(V.index.tri_window);
    a.tri_s = const_cast<int32_t*>(V.index.tri_sinks);
    a.blk_b = const_cast<int32_t*>(V.index.blk_b);
    apply_choice_kernel<<<(p.hh + 127) / 128, 128, 0, st>>>(a);
    if ((rc = check_launch("apply_choice_kernel"))) return rc;
  }
  auto mark_on = [&](int e, cudaStream_t s) {
    if (desc->stage_events[e]) cudaEventRecord(reinterpret_cast<cudaEvent_t>(desc->stage_events[e]), s);
  };
  auto mark = [&](int e) { mark_on(e, st); };
  mark(0);
  // The VS and Block-Cluster estimators only share the per-head choice: with
  // both present the VS chain (latency-bound, few CTAs) runs on the side stream
  // beside the block GEMM (fork / join through events, graph-capturable).
  // SA_OVERLAP_EST=0 keeps everything on the caller's stream.
  cudaStream_t vs_st = st;
  const bool vs_side = side && p.any_vs;
  if (vs_side) {
    cudaEventRecord(side->fork, st);
    cudaStreamWaitEvent(side->s, side->fork, 0);
    vs_st = side->s;
  }
  // 2. vertical-slash estimator + stable top-k into bitmaps
  if (p.any_vs) {
    cudaMemsetAsync(const_cast<uint32_t*>(V.index.colbits), 0, (size_t)p.hh * p.vs_words * 4, vs_st);
    cudaMemsetAsync(const_cast<uint32_t*>(V.index.diagrev), 0, (size_t)p.hh * p.vs_words * 4, vs_st);
    // estimated scoring over the last q_est rows, in groups of <= 128 rows
    const int r_first = n - p.q_est;
    for (int g = 0; g < p.tail_groups; ++g) {
      const int r_hi = n - g * 128;
      const int r_lo = std::max(r_first, r_hi - 128);
      if ((rc = launch_score_tail(B, H, HK, n, desc->scale, q, k, r_lo, r_hi, V.col_scores,
                                  V.diag_scores, g > 0, V.family, SA_VERTICAL_SLASH,
                                  b + L.off[W_TAIL], p.tail_ws, vs_st)))
        return rc;
    }
    for (int c = 0; c < p.ncand; ++c) {
      if (p.cand[c].family != SA_VERTICAL_SLASH) continue;
      TopkArgs t{};
      t.scores = V.col_scores;
      t.ld = n;
      t.rows = p.hh;
      t.n = n;
      t.k = p.cand[c].p1;
      t.idx_out = V.col_idx;
      t.out_ld = p.max_kv;
      t.bits = const_cast<uint32_t*>(V.index.colbits);
      t.bits_ld = p.vs_words;
      t.bit_base = 0;
      t.bit_neg = 0;
      t.gate = choice ? choice : V.family;
      t.gate_sparse = desc->mode == SA_MODE_AUTO;  // a fixed VS layer keeps every row
      t.gate_div = 1;
      t.gate_val = choice ? c : SA_VERTICAL_SLASH;
      // diagonal rows in the same launch (rows >= hh)
      t.split = p.hh;
      t.scores2 = V.diag_scores;
      t.k2 = p.cand[c].p2;
      t.idx_out2 = V.diag_idx;
      t.out_ld2 = p.max_ks;
      t.bits2 = const_cast<uint32_t*>(V.index.diagrev);
      t.bit_base2 = n + 127;
      t.bit_neg2 = 1;
      if ((rc = launch_topk(t, vs_st))) return rc;
    }
  }
  mark_on(1, vs_st);
  // 3. block estimator
  if (p.any_block) {
    for (int c = 0; c < p.ncand; ++c) {
      if (p.cand[c].family != SA_BLOCK_SPARSE) continue;
      const int bs = p.cand[c].p1, kb = p.cand[c].p2;
      const int32_t* gate = choice ? choice : V.family;
      const int gval = choice ? c : SA_BLOCK_SPARSE;
      if (use_block_screen(kb)) {
        // k_b <= 8 (the auto search's Block(8, 1)): fp16 screen + exact refine (block_screen.cu)
        if ((rc = launch_block_pool16(p.hh, n, bs, q, b + L.off[W_QP], false, gate, gval, st))) return rc;
        if (kpool_early) {
          cudaStreamWaitEvent(st, side->kdone, 0);
        } else if ((rc = launch_block_pool16(p.hk, n, bs, k, b + L.off[W_KP], true, nullptr, 0, st))) {
          return rc;
        }
        if ((rc = launch_block_screen(B, H, HK, n, bs, kb, b + L.off[W_QP], b + L.off[W_KP],
                                      const_cast<int32_t*>(V.index.blk_idx), p.blk_head_stride,
                                      const_cast<int32_t*>(V.index.blk_row_off), p.blk_row_stride, gate, gval,
                                      b + L.off[W_BLKWS], p.blk_ws, st)))
          return rc;
        continue;
      }
      if ((rc = launch_block_pool(p.hh, n, bs, 0, q, b + L.off[W_QP], nullptr, gate, gval, st))) return rc;
      if (kpool_early) {
        cudaStreamWaitEvent(st, side->kdone, 0);
      } else if ((rc = launch_block_pool(p.hk, n, bs, 1, k, b + L.off[W_KP], nullptr, nullptr, 0, st))) {
        return rc;
      }
      if ((rc = launch_block_select(B, H, HK, n, bs, kb, desc->scale, b + L.off[W_QP],
                                    b + L.off[W_KP], const_cast<int32_t*>(V.index.blk_idx),
                                    p.blk_head_stride, const_cast<int32_t*>(V.index.blk_row_off),
                                    p.blk_row_stride, gate, gval, b + L.off[W_BLKWS], p.blk_ws, st)))
        return rc;
    }
  }
  if (side) {  // join the side stream (the tile lists need every index)
    cudaEventRecord(side->join, side->s);
    cudaStreamWaitEvent(st, side->join, 0);
  }
  mark(2);
  // 4. executed tiles + attention
  if ((rc = sa_build_tiles(&V.index, p.hh, n, V.tile_off, V.tile_cnt, V.tiles, stream))) return rc;
  mark(3);
  // SA_SCAN_AT=2: the scan is forked after the work-order kernel, just ahead of
  // the attention launch, so its short CTAs start once the attention's
  // persistent CTAs (launched early through PDL) hold their SM slots (32K:
  // 1.0952 vs 1.0934 ms forked before the work order, SA_SCAN_LATE=0; queueing
  // it after the attention launch measured 20 us slower)
  static const bool scan_late = [] {
    const char* e = getenv("SA_SCAN_LATE");
    return !(e && e[0] == '0');
  }();
  if (chk && scan_at == 2 && !(scan_late && !desc->stop_after_tiles) && (rc = fork_scan(true))) return rc;
  if (chk && (scan_at == 0 || desc->stop_after_tiles)) cudaStreamWaitEvent(st, chk->join2, 0);
  if (desc->stop_after_tiles) return SA_OK;
  // CTA order: auto layers mix heavy (VS, dense-like) and light (Block) heads,
  // so the non-empty items go longest-first (LPT); a uniform layer (dense or
  // one fixed pattern) keeps the kernel's kv-group-major order, heaviest query
  // tiles first in a group, so the items in flight share one group's K/V in L2
  // (dense / VS 4-8% faster at 64K-128K, equal at 32K; SA_ATTN_ORDER=0 / 1
  // forces either, for A/B)
  static const int order_env = [] {
    const char* e = getenv("SA_ATTN_ORDER");
    return e ? atoi(e) : -1;
  }();
  const bool lpt = order_env >= 0 ? order_env != 0 : desc->mode == SA_MODE_AUTO;
  int32_t* wbase = reinterpret_cast<int32_t*>(b + L.off[W_WORK]);
  int* counter = wbase;
  int32_t* n_work = wbase + 1;
  int32_t* work = wbase + 64;
  // GQA siblings adjacent within a cost bin (SA_SIBLING_ORDER=0: head-major, for A/B)
  static const bool sib = [] {
    const char* e = getenv("SA_SIBLING_ORDER");
    return !(e && e[0] == '0');
  }();
  if (lpt && (rc = launch_order_work(V.tile_cnt, p.hh * p.nqt, p.nqt, work, n_work, st, p.nqt,
                                     sib ? H / HK : 1, counter)))
    return rc;
  if (chk && scan_at == 2 && scan_late && (rc = fork_scan(true))) return rc;
  rc = launch_attn(B, H, HK, n, desc->scale, q, k, v, out, &V.index, V.tile_off, V.tile_cnt, V.tiles,
                   lpt ? work : nullptr, nullptr, st, desc->out_ld, counter, lpt ? n_work : nullptr, nullptr, 0,
                   lpt);
  mark(4);
  if (chk && scan_at != 0) cudaStreamWaitEvent(st, chk->join2, 0);
  return rc;
}
