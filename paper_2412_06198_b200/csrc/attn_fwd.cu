// attn_fwd.cu — tile-sparse causal FlashAttention forward for sm_100a.
//
// One kernel serves the three pattern families of the reference
// (patterns.py:353-435 vertical_slash_attention, which also runs the
// Triangular index per patterns.py:262-276/495-497, and patterns.py:438-484
// block_sparse_attention) plus the dense reference (core.py:138-154):
// the index is turned into a per-(head, query-tile) list of 128-key tiles,
// each tagged with a mask kind (sa_types.h), and the kernel evaluates logits
// only on listed tiles.  Inside a tile, positions outside the index get -inf
// before the row softmax, which reproduces "weights off the index are
// exactly 0" (patterns.py:353-435 docstring) and the column-wins dedupe
// (a position is one element of the union, evaluated once).
//
// Per CTA: one (head, 128-row query tile); every listed 128-key tile is
// processed as two 64-key sub-tiles u.  192 threads:
//   warps 0-3  softmax: thread r owns query row r (TMEM lane r)
//   warp  4    TMA producer: Q once, then K_u / V_u through a 5-slot 16 KB ring
//   warp  5    TMEM allocator + single-thread tcgen05.mma issuer
// TMEM (256 columns): S double buffer (2 x 64 fp32 columns, P = bf16 softmax
// aliased over the first 32 columns of its buffer) and O (128 columns).  The
// MMA warp issues QK(u+2) right after PV(u), so the tensor core computes the
// next logits while the softmax warps work on the current ones; two CTAs
// co-reside per SM (113 KB smem, 256 TMEM columns each) and hide each other's
// prologue/epilogue.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "sa_types.h"
#include "sm100_common.cuh"
#include "attn_mask.cuh"

namespace sa {

constexpr int kMaxPeers = 7;  // an 8-GPU NVSwitch domain

struct AttnArgs {
  CUtensorMap tmap_q;  // [HH, n, 128] bf16, box {64, 128, 1}, SW128
  CUtensorMap tmap_k;  // [HK, n, 128], box {64, 64, 1}
  CUtensorMap tmap_v;  // [HK, n, 128], box {64, 64, 1}
  CUtensorMap tmap_k8;  // gather maps (make_tmap_kv_gather): box = 8 rows x both d-halves, 2 KB
  CUtensorMap tmap_v8;
  __nv_bfloat16* out;
  long long out_batch_stride;  // elements between batches
  long long out_row_stride;    // elements between rows (H * 128 for (B, L, H*d))
  int n;
  int heads;     // query heads per batch
  int kv_heads;  // key/value heads per batch
  int nqt;       // query tiles = ceil(n / 128)
  int hh_total;  // batch * heads
  float scale_log2;
  const int32_t* tile_off;  // [hh_total * nqt]
  const int32_t* tile_cnt;  // [hh_total * nqt]
  const uint32_t* tiles;
  const int32_t* work;  // optional CTA -> (hh * nqt + qt) order; null = heavy-first default
  HeadIndexView idx;
  float* lse;  // optional [hh_total, n] natural-log row log-sum-exp
  unsigned long long* prof;  // SA_ATTN_PROF builds: per-role phase cycle counters [3 * 16]
  int* counter;              // optional work-item counter (zeroed before launch): dynamic fetch
  const int32_t* n_work;     // optional device count of `work` entries (default hh_total * nqt)
  int st256;                 // output rows 32-byte aligned: 256-bit stores
  int skip_dead;             // warps whose 32 rows are all masked out of a sub-tile write P = 0 only
  int epi_mode;              // experiment (SA_ATTN_EPI): 1 = full epilogue, 0 = no global stores, 2 = no O read
  CUtensorMap tmap_out;      // SA_ATTN_TMA_STORE: the output as {cols, n, B}, box {64, 128, 1}
  int tma_out;               // use it (no peer copies, TMA-compatible layout)
  int n_peers;               // > 0: every output row is also stored into these buffers (same layout),
  __nv_bfloat16* peer_out[kMaxPeers];  // other ranks' outputs mapped over NVLink (fused all-gather)
};

constexpr int kThreads = 192;     // softmax WG + producer + MMA warp
constexpr int kThreadsEwg = 384;  // + an epilogue WG (and two idle warps: warpgroup-aligned setmaxnreg)
constexpr int kDefaultPoly = 4;
#ifndef SA_PRODUCER_SLEEP_NS
#define SA_PRODUCER_SLEEP_NS 64
#endif
#ifndef SA_MMA_SLEEP_NS
#define SA_MMA_SLEEP_NS 16
#endif
// polling back-off of the producer / MMA warps (they share sub-partitions with softmax warps)
constexpr int kProducerSleepNs = SA_PRODUCER_SLEEP_NS;
#ifndef SA_EWG_SLEEP_NS
#define SA_EWG_SLEEP_NS 256
#endif
constexpr int kMmaSleepNs = SA_MMA_SLEEP_NS;
#ifdef SA_ATTN_PROF
constexpr bool kProf = true;
#else
constexpr bool kProf = false;
#endif
// phase timer: PT(k) adds the cycles since the previous mark to counter k
#define PT_INIT long long pt_last = kProf ? clock64() : 0; unsigned long long pc[16] = {0};
#define PT(k) do { if (kProf) { long long t_ = clock64(); pc[k] += t_ - pt_last; pt_last = t_; } } while (0)
#define PT_FLUSH(base) do { if (kProf && a.prof && lane_id() == 0) { \
    for (int k_ = 0; k_ < 16; ++k_) atomicAdd(a.prof + (base) + k_, pc[k_]); } } while (0)
constexpr uint32_t kTmemCols = 256;
constexpr uint32_t kColS = 0;    // S buffers at 0 and 64 (P aliased at their first 32 columns)
constexpr uint32_t kColO = 128;
constexpr int kSub = 64;         // keys per sub-tile
#ifndef SA_ATTN_TMA_STORE
#define SA_ATTN_TMA_STORE 0
#endif
// SA_ATTN_TMA_STORE: the epilogue writes each 64-column half of the output tile
// into a 16 KB shared-memory stage (taken from the K/V ring) and one thread
// TMA-stores it, instead of 8 x 32-byte global stores per thread
constexpr int kRing = SA_ATTN_TMA_STORE ? 4 : 5;  // K/V ring slots of 16 KB
constexpr int kSlotBytes = 16384;
constexpr int kSmemQ = 0;
constexpr int kSmemRing = 32768;
constexpr int kSmemStage = kSmemRing + kRing * kSlotBytes;          // TMA-store stage (1024-aligned)
constexpr int kSmemBar = kSmemStage + (SA_ATTN_TMA_STORE ? 16384 : 0);  // 114688
constexpr int kSmemL = kSmemBar + 256;     // EWG: the row sums l of the item handed to the epilogue WG
constexpr int kSmemBytes = kSmemBar + 256;  // + barriers; base is 1024-aligned (two CTAs per SM must fit)
constexpr int kSmemBytesEwg = kSmemL + 512;

enum Bar {
  B_Q = 0,                     // Q tile landed
  B_QE = 1,                    // every QK MMA of the item completed (Q buffer free)
  B_FULL0 = 2,                 // kRing
  B_EMPTY0 = B_FULL0 + kRing,  // kRing
  B_SF0 = B_EMPTY0 + kRing,    // 2
  B_PF0 = B_SF0 + 2,           // 2
  B_OF = B_PF0 + 2,            // final O of the item
  B_OE = B_OF + 1,             // epilogue has read O
  B_IF0 = B_OE + 1,            // 2: work-item slot published
  B_IE0 = B_IF0 + 2,           // 2: work-item slot consumed
  B_LF = B_IE0 + 2,            // EWG: row sums of the finished item in smem
  B_LE = B_LF + 1,             // EWG: the epilogue WG has read them
  B_NUM = B_LE + 1
};

// Work item idx -> (hh * nqt + qt): the caller's order (LPT), else kv-group-major
// (the group's K/V stays L2-resident), heaviest query tiles first in a group.
__device__ __forceinline__ int item_at(const AttnArgs& a, int idx) {
  if (a.work != nullptr) return a.work[idx];
  const int gs = a.heads / a.kv_heads;
  const int per_group = a.nqt * gs;
  const int g = idx / per_group, r = idx % per_group;
  const int qt = a.nqt - 1 - r / gs;
  const int hh_ = (g / a.kv_heads) * a.heads + (g % a.kv_heads) * gs + r % gs;
  return hh_ * a.nqt + qt;
}

// Persistent: each CTA (two per SM) walks work items (head, query tile).  The
// producer fetches the next item (an atomic counter over the LPT list, or a
// static stride) and publishes it through a two-slot shared-memory queue; the
// barrier phases run on across items, so the next item's Q load and first
// QK MMAs overlap the current item's last sub-tiles and epilogue.
//
// POLY > 0: every POLY-th exp pair of a row chunk runs on the FMA pipe
// (exp2_poly2) instead of MUFU, balancing the two pipes.
//
// EWG: a fourth role, an epilogue warpgroup (warps 4-7), takes the finished
// item's O out of TMEM, normalises, packs and stores it (and the peer copies)
// while the softmax warps already run the next item; registers are
// rebalanced with setmaxnreg (softmax 144, epilogue 56, producer / MMA 40).
template <int POLY, bool EWG>
__global__ void __launch_bounds__(EWG ? kThreadsEwg : kThreads, 2) attn_fwd_kernel(const __grid_constant__ AttnArgs a) {
  constexpr int kProdWarp = EWG ? 8 : 4;
  constexpr int kMmaWarp = EWG ? 9 : 5;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if ((smem_u32(smem) & 1023u) != 0u) __trap();  // SWIZZLE_128B tiles need 1024-byte alignment
  uint8_t* sQ = smem + kSmemQ;
  uint8_t* sRing = smem + kSmemRing;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kSmemBar);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + B_NUM);
  volatile int* sItem = reinterpret_cast<volatile int*>(tmem_holder + 4);  // [2]
  // per ring slot: 1 = gathered layout ([8-row block][half][8 rows][128 B]), 0 = [half][64 rows][128 B]
  volatile int* sLay = sItem + 2;  // [kRing]

  const long long t_entry = kProf ? clock64() : 0;
  const int warp = warp_id();

  if (threadIdx.x == 0) {
    mbar_init(&bars[B_Q], 1);
    mbar_init(&bars[B_QE], 1);
    for (int i = 0; i < kRing; ++i) {
      mbar_init(&bars[B_FULL0 + i], 1);
      mbar_init(&bars[B_EMPTY0 + i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars[B_SF0 + i], 1);
      mbar_init(&bars[B_PF0 + i], 128);
      mbar_init(&bars[B_IF0 + i], 1);
      mbar_init(&bars[B_IE0 + i], EWG ? 1 + 256 : 1 + 128);
    }
    mbar_init(&bars[B_OF], 1);
    mbar_init(&bars[B_OE], 128);
    mbar_init(&bars[B_LF], 128);
    mbar_init(&bars[B_LE], 128);
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc(tmem_holder, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_holder;
  // programmatic dependent launch: the prologue above overlapped the previous
  // kernel; everything below may read its results
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int n_items = a.n_work ? *a.n_work : a.hh_total * a.nqt;

  if (warp == kProdWarp) {
    // ------------------------------------------------------------ producer
    if constexpr (EWG) asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    const int lane = lane_id();
    if (lane == 0) {
      tma_prefetch(&a.tmap_q);
      tma_prefetch(&a.tmap_k);
      tma_prefetch(&a.tmap_v);
    }
    PT_INIT
    int rb = 0;  // ring items issued by this CTA so far
    for (int J = 0;; ++J) {
      // fetch and publish the next work item
      int idx = 0;
      if (lane == 0) idx = a.counter ? atomicAdd(a.counter, 1) : (int)blockIdx.x + J * (int)gridDim.x;
      idx = __shfl_sync(0xffffffffu, idx, 0);
      const int item = idx < n_items ? item_at(a, idx) : -1;
      if (J >= 2) mbar_wait_backoff<kProducerSleepNs>(&bars[B_IE0 + (J & 1)], ((J >> 1) - 1) & 1);
      if (lane == 0) {
        sItem[J & 1] = item;
        mbar_arrive(&bars[B_IF0 + (J & 1)]);
      }
      if (item < 0) break;
      const int hh = item / a.nqt, qt = item % a.nqt;
      const int hkv = (hh / a.heads) * a.kv_heads + (hh % a.heads) / (a.heads / a.kv_heads);
      const int cnt = a.tile_cnt[item];
      const int nsub = 2 * cnt;
      const uint32_t* tl = a.tiles + a.tile_off[item];
      // Q: the buffer is free once every QK MMA of the previous item completed
      if (J >= 1) mbar_wait_backoff<kProducerSleepNs>(&bars[B_QE], (J - 1) & 1);
      if (lane == 0) {
        mbar_arrive_expect_tx(&bars[B_Q], 32768);
        tma_load_3d(sQ, &a.tmap_q, &bars[B_Q], 0, qt * kTile, hh);
        tma_load_3d(sQ + 16384, &a.tmap_q, &bars[B_Q], 64, qt * kTile, hh);
      }
      const int bsz = a.idx.blk_b[hh];
      int slot_gk = 0;  // gather tiles: key block of slot `lane` (0 = placeholder, masked)
      // ring sequence: K_0, V_0, K_1, V_1, ... (sub-tiles u = 2 j + half)
      for (int i = 0; i < 2 * nsub; ++i) {
        const int u = i >> 1;
        const int g = rb + i;
        const int slot = g % kRing;
        const uint32_t e = tl[u >> 1];
        const uint32_t kind = tile_kind(e);
        if (kind == TK_GATHER && (i & 3) == 0) {
          const int gq = qt * (kTile / bsz) + lane;
          const int32_t* ro = a.idx.blk_row_off + (size_t)hh * a.idx.blk_row_stride;
          int gk = 0;
          if (lane < kTile / bsz && gq * bsz < a.n) {
            const int k = ro[gq] + (int)tile_ktile(e);
            if (k < ro[gq + 1]) {
              const int x = a.idx.blk_idx[k];
              if (x < gq) gk = x;
            }
          }
          slot_gk = gk;
        }
        PT(0);
        if (g >= kRing) mbar_wait_backoff<kProducerSleepNs>(&bars[B_EMPTY0 + slot], ((g / kRing) - 1) & 1);
        PT(1);
        uint8_t* dst = sRing + slot * kSlotBytes;
        // b = 64: a gathered sub-tile is one whole key block, loaded like a contiguous one
        const int gk64 = (kind == TK_GATHER && bsz == kSub) ? __shfl_sync(0xffffffffu, slot_gk, u & 1) : -1;
        if (kind != TK_GATHER || gk64 >= 0) {
          if (lane == 0) {
            const int row = gk64 >= 0 ? gk64 * kSub : (int)tile_ktile(e) * kTile + (u & 1) * kSub;
            const CUtensorMap* map = (i & 1) ? &a.tmap_v : &a.tmap_k;
            sLay[slot] = 0;
            mbar_arrive_expect_tx(&bars[B_FULL0 + slot], kSlotBytes);
            tma_load_3d(dst, map, &bars[B_FULL0 + slot], 0, row, hkv);
            tma_load_3d(dst + 8192, map, &bars[B_FULL0 + slot], 64, row, hkv);
          }
        } else {
          // 64 gathered keys = 8 boxes of 8 rows x both d-halves (2 KB each); lane -> box
          const int bx = lane & 7;
          const int key = (u & 1) * kSub + bx * 8;
          const int gk = __shfl_sync(0xffffffffu, slot_gk, key / bsz);
          const CUtensorMap* map = (i & 1) ? &a.tmap_v8 : &a.tmap_k8;
          if (lane == 0) {
            sLay[slot] = 1;
            mbar_arrive_expect_tx(&bars[B_FULL0 + slot], kSlotBytes);
          }
          __syncwarp();
          if (lane < 8) tma_load_4d(dst + bx * 2048, map, &bars[B_FULL0 + slot], 0, gk * bsz + key % bsz, 0, hkv);
        }
        PT(2);
        if (kProf) pc[15] += 1;
      }
      rb += 2 * nsub;
    }
    PT_FLUSH(32);
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    if constexpr (EWG) asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    const bool leader = elect_one();
    constexpr uint32_t idesc_qk = idesc_bf16_f32(128, kSub, 0, 0);
    constexpr uint32_t idesc_pv = idesc_bf16_f32(128, 128, 0, 1);
    const uint32_t q_addr = smem_u32(sQ);
    const uint32_t ring_addr = smem_u32(sRing);
    PT_INIT
    int rb = 0, sb = 0, pb = 0;  // ring items, S-buffer uses (per buffer), PV commits so far
    for (int J = 0;; ++J) {
      mbar_wait_backoff<kMmaSleepNs>(&bars[B_IF0 + (J & 1)], (J >> 1) & 1);
      // the elected lane reads the slot and releases it; the warp gets the item
      // by shuffle (every read of the slot precedes its own release)
      int item = 0;
      if (leader) {
        item = sItem[J & 1];
        mbar_arrive(&bars[B_IE0 + (J & 1)]);
      }
      item = __shfl_sync(0xffffffffu, item, __ffs(__ballot_sync(0xffffffffu, leader)) - 1);
      if (item < 0) break;
      const int nsub = 2 * a.tile_cnt[item];
      if (leader) {
        auto issue_qk = [&](int u) {
          const int g = rb + 2 * u, slot = g % kRing;
          PT(0);
          mbar_wait_backoff<kMmaSleepNs>(&bars[B_FULL0 + slot], (g / kRing) & 1);
          PT(1);
          tc_fence_after();
          const uint32_t k_addr = ring_addr + slot * kSlotBytes;
          // gathered slots interleave the d-halves per 8-key block (half at +1 KB, blocks 2 KB apart)
          const bool gl = sLay[slot] != 0;
          const uint32_t k_half = gl ? 1024u : 8192u, k_sbo = gl ? 2048u : 1024u;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            mma_ss(tbase + kColS + (u & 1) * kSub,
                   sdesc_sw128(q_addr + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                   sdesc_sw128(k_addr + (kk >> 2) * k_half + (kk & 3) * 32, 16, k_sbo), idesc_qk,
                   kk > 0 ? 1u : 0u);
          }
          mma_commit(&bars[B_EMPTY0 + slot]);
          mma_commit(&bars[B_SF0 + (u & 1)]);
          if (u == nsub - 1) mma_commit(&bars[B_QE]);  // last reader of Q
          PT(2);
        };
        mbar_wait_backoff<kMmaSleepNs>(&bars[B_Q], J & 1);
        tc_fence_after();
        if (nsub == 0) mma_commit(&bars[B_QE]);
        if (nsub > 0) issue_qk(0);
        if (nsub > 1) issue_qk(1);
        for (int u = 0; u < nsub; ++u) {
          PT(3);
          mbar_wait_backoff<kMmaSleepNs>(&bars[B_PF0 + (u & 1)], (sb + (u >> 1)) & 1);
          PT(4);
          const int g = rb + 2 * u + 1, slot = g % kRing;
          mbar_wait_backoff<kMmaSleepNs>(&bars[B_FULL0 + slot], (g / kRing) & 1);
          // PV(0) overwrites O: the previous item's epilogue must have read it
          if (u == 0 && J >= 1) mbar_wait_backoff<kMmaSleepNs>(&bars[B_OE], (J - 1) & 1);
          PT(5);
          tc_fence_after();
          const uint32_t v_addr = ring_addr + slot * kSlotBytes;
          const uint32_t p_addr = tbase + kColS + (u & 1) * kSub;
          const bool gl = sLay[slot] != 0;
          const uint32_t v_step = gl ? 4096u : 2048u, v_lbo = gl ? 1024u : 8192u, v_sbo = gl ? 2048u : 1024u;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            mma_ts(tbase + kColO, p_addr + kk * 8, sdesc_sw128(v_addr + kk * v_step, v_lbo, v_sbo),
                   idesc_pv, (u > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&bars[B_EMPTY0 + slot]);  // also "PV(u) has updated O" for a rescaling softmax
          PT(6);
          if (kProf) pc[15] += 1;
          if (u + 2 < nsub) issue_qk(u + 2);
        }
        mma_commit(&bars[B_OF]);
      }
      __syncwarp();
      rb += 2 * nsub;
      sb += nsub / 2;
      pb += nsub;
    }
    (void)pb;
    PT_FLUSH(16);
  } else if (EWG && warp >= 4 && warp < 8) {
    // ------------------------------------------------------------ epilogue WG
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
    const int r = threadIdx.x - 128;  // row of the tile = TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const volatile float* sL = reinterpret_cast<const volatile float*>(smem + kSmemL);
    for (int J = 0;; ++J) {
      mbar_wait_backoff<SA_EWG_SLEEP_NS>(&bars[B_IF0 + (J & 1)], (J >> 1) & 1);
      const int item = sItem[J & 1];
      mbar_arrive(&bars[B_IE0 + (J & 1)]);
      if (item < 0) break;
      const int hh = item / a.nqt, qt = item % a.nqt;
      const int bidx = hh / a.heads, h = hh % a.heads;
      const int i = qt * kTile + r;
      const bool valid = i < a.n && a.tile_cnt[item] > 0;  // cnt == 0: query tile not requested
      const long long ooff = (long long)bidx * a.out_batch_stride + (long long)i * a.out_row_stride +
                             (long long)h * kHeadDim;
      mbar_wait_backoff<SA_EWG_SLEEP_NS>(&bars[B_LF], J & 1);
      const float inv = 1.0f / sL[r];
      mbar_arrive(&bars[B_LE]);
      mbar_wait_backoff<SA_EWG_SLEEP_NS>(&bars[B_OF], J & 1);
      tc_fence_after();
      __nv_bfloat16* orow = a.out + ooff;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t o[32];
        tmem_ld32(tbase + lane_off + kColO + 32 * c, o);
        tmem_ld_wait();
        if (c == 3) {
          tc_fence_before();
          mbar_arrive(&bars[B_OE]);  // O may now be overwritten by the next item's PV(0)
        }
        if (valid) {
          uint32_t pk[16];
#pragma unroll
          for (int t = 0; t < 16; ++t)
            pk[t] = pack_bf16(__uint_as_float(o[2 * t]) * inv, __uint_as_float(o[2 * t + 1]) * inv);
          auto store = [&](__nv_bfloat16* row) {
            if (a.st256) {
#pragma unroll
              for (int t = 0; t < 2; ++t) st_global_v8(row + 32 * c + 16 * t, pk + 8 * t);
            } else {
              uint4* dst = reinterpret_cast<uint4*>(row + 32 * c);
#pragma unroll
              for (int t = 0; t < 4; ++t)
                dst[t] = make_uint4(pk[4 * t], pk[4 * t + 1], pk[4 * t + 2], pk[4 * t + 3]);
            }
          };
          store(orow);
#pragma unroll 1
          for (int pr = 0; pr < a.n_peers; ++pr) store(a.peer_out[pr] + ooff);
        }
      }
    }
    if (a.n_peers > 0) __threadfence_system();  // peer stores drained before the CTA retires
  } else if (warp < 4) {
    // ------------------------------------------------------------ softmax warps
    if constexpr (EWG) asm volatile("setmaxnreg.inc.sync.aligned.u32 144;\n" ::: "memory");
    const int r = threadIdx.x;  // 0..127
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    const float sl2 = a.scale_log2;
    PT_INIT
    if (kProf) { pc[10] += pt_last - t_entry; pc[12] += 1; }
    int sb = 0, pb = 0, rb = 0;  // S-buffer uses, PV count, ring positions (as the MMA warp counts them)
    // The next item's descriptor, row constants and first tile entries are
    // loaded before the current item's epilogue, hiding their latency.
    int item, cnt;
    const uint32_t* tl;
    RowConst rc;
    uint32_t raw[9];
    uint32_t e_cur, e_nxt;
    auto fetch_item = [&](int J) {
      mbar_wait(&bars[B_IF0 + (J & 1)], (J >> 1) & 1);
      item = sItem[J & 1];
      mbar_arrive(&bars[B_IE0 + (J & 1)]);
      if (item < 0) return;
      cnt = a.tile_cnt[item];
      tl = a.tiles + a.tile_off[item];
      const int hh_ = item / a.nqt, i_ = (item % a.nqt) * kTile + r;
      rc = row_const(a, hh_, i_);
      e_cur = cnt > 0 ? tl[0] : 0u;
      e_nxt = cnt > 1 ? tl[1] : 0u;
      mask_fetch(a, rc, hh_, i_, e_cur, raw);
    };
    fetch_item(0);
    for (int J = 0;; ++J) {
      if (item < 0) break;
      const int hh = item / a.nqt, qt = item % a.nqt;
      const int bidx = hh / a.heads, h = hh % a.heads;
      const int nsub = 2 * cnt;
      const int i = qt * kTile + r;
      const int cur_cnt = cnt;
      float m_used = -INFINITY;
      float l = 0.f;
      uint32_t msk[4] = {0u, 0u, 0u, 0u};
      uint32_t kind = TK_FULL;
      for (int u = 0; u < nsub; ++u) {
        const int half = u & 1;
        PT(0);
        if (half == 0) {
          const int t = u >> 1;
          kind = tile_kind(e_cur);
          if (kind != TK_FULL) mask_make(a, rc, i, qt, e_cur, raw, msk);
          // next tile's entry and mask words are loaded now, used one tile later
          if (t + 1 < cnt) mask_fetch(a, rc, hh, i, e_nxt, raw);
          e_cur = e_nxt;
          e_nxt = (t + 2 < cnt) ? tl[t + 2] : 0u;
        }
        PT(1);
        mbar_wait(&bars[B_SF0 + half], (sb + (u >> 1)) & 1);
        PT(2);
        tc_fence_after();
        const uint32_t s_col = tbase + lane_off + kColS + half * kSub;
        // Gathered / block-diagonal / causal-diagonal tiles leave half the rows
        // of a sub-tile with no visible key: such a warp skips the softmax and
        // only zeroes its P rows (the PV MMA still reads all 128), keeping m, l, O.
        if (kind != TK_FULL && a.skip_dead &&
            __all_sync(0xffffffffu, ((half ? msk[2] : msk[0]) | (half ? msk[3] : msk[1])) == 0u)) {
          uint32_t z[32];
#pragma unroll
          for (int t = 0; t < 32; ++t) z[t] = 0u;
          tmem_st32(s_col, z);
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(&bars[B_PF0 + half]);
          PT(7);
          continue;
        }
        uint32_t s[2][32];
        tmem_ld32(s_col, s[0]);
        tmem_ld32(s_col + 32, s[1]);
        tmem_ld_wait();
        PT(3);
        if (kind != TK_FULL) {
          // float selects on constant bit tests: ptxas emits R2P (7 mask bits
          // to predicates at once) + FSEL, about one instruction per logit
          const uint32_t m0 = half ? msk[2] : msk[0], m1 = half ? msk[3] : msk[1];
          // (one loop per mask word: interleaving the two words defeats the R2P match)
#pragma unroll
          for (int t = 0; t < 32; ++t)
            if (!(m0 & (1u << t))) s[0][t] = __float_as_uint(-INFINITY);
#pragma unroll
          for (int t = 0; t < 32; ++t)
            if (!(m1 & (1u << t))) s[1][t] = __float_as_uint(-INFINITY);
        }
        // row max: four independent FMNMX3 chains
        float mx;
        {
          float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int t = 0; t < 32; t += 4) {
              m4[2 * c] = fmax3(m4[2 * c], __uint_as_float(s[c][t]), __uint_as_float(s[c][t + 1]));
              m4[2 * c + 1] = fmax3(m4[2 * c + 1], __uint_as_float(s[c][t + 2]), __uint_as_float(s[c][t + 3]));
            }
          mx = fmax3(m4[0], m4[1], fmaxf(m4[2], m4[3]));
        }
        PT(4);
        const float mt = mx * sl2;
        // Lazy rescale: keep a stale max until the row max grows by > 2^8.  The
        // decision is per row but the TMEM round trip of O is warp-wide
        // (tcgen05.ld/st are .sync.aligned), so rows that need none use 1.
        const bool need = mt > m_used + 8.0f;
        if (__any_sync(0xffffffffu, need)) {
          const float alpha = need ? fast_exp2(m_used - mt) : 1.0f;  // 0 when m_used == -inf
          l *= alpha;
          if (u > 0) {
            // PV(u-1) may still be accumulating into O (PV(u-2) completed before
            // S_u): wait for the commit that releases V(u-1)'s ring slot.  That
            // slot cannot complete another phase before P(u) exists (its next
            // reader, QK(u+2), is issued after PV(u)), so the parity is exact.
            const int gv = rb + 2 * (u - 1) + 1;
            mbar_wait(&bars[B_EMPTY0 + gv % kRing], (gv / kRing) & 1);
            tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
              uint32_t o[32];
              tmem_ld32(tbase + lane_off + kColO + 32 * c, o);
              tmem_ld_wait();
#pragma unroll
              for (int t = 0; t < 32; t += 2) {
                const float2 v = fmul2(make_float2(__uint_as_float(o[t]), __uint_as_float(o[t + 1])),
                                       make_float2(alpha, alpha));
                o[t] = __float_as_uint(v.x);
                o[t + 1] = __float_as_uint(v.y);
              }
              tmem_st32(tbase + lane_off + kColO + 32 * c, o);
            }
            tmem_st_wait();
          }
          if (need) m_used = mt;
        }
        PT(5);
        const float moff = (m_used == -INFINITY) ? 0.f : m_used;
        // p = exp2(s * scale_log2 - m): FFMA2 + two MUFU.EX2; row sum in four FADD2 chains
        const float2 sc2 = make_float2(sl2, sl2);
        const float2 mo2 = make_float2(-moff, -moff);
        float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                         make_float2(0.f, 0.f)};
        uint32_t p[32];
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int t = 0; t < 32; t += 2) {
            float2 x = ffma2(make_float2(__uint_as_float(s[c][t]), __uint_as_float(s[c][t + 1])), sc2, mo2);
            if (POLY > 0 && ((t >> 1) % (POLY > 0 ? POLY : 1)) == (POLY > 0 ? POLY : 1) - 1) {
              x = exp2_poly2(x);
            } else {
              x.x = fast_exp2(x.x);
              x.y = fast_exp2(x.y);
            }
            acc[(t >> 1) & 3] = fadd2(acc[(t >> 1) & 3], x);
            p[c * 16 + (t >> 1)] = pack_bf16(x.x, x.y);
          }
        {
          const float2 a01 = fadd2(acc[0], acc[1]), a23 = fadd2(acc[2], acc[3]);
          const float2 t2 = fadd2(a01, a23);
          l += t2.x + t2.y;
        }
        PT(6);
        tmem_st32(s_col, p);  // P (bf16 pairs) over the first 32 columns of this S buffer
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&bars[B_PF0 + half]);
        PT(7);
        if (kProf) pc[15] += 1;
      }
      // ---------------------------------------------------------- epilogue
      fetch_item(J + 1);  // next item's loads in flight during this epilogue
      if constexpr (EWG) {
        // hand the row sum to the epilogue WG (its previous one has been read)
        if (J >= 1) mbar_wait(&bars[B_LE], (J - 1) & 1);
        reinterpret_cast<volatile float*>(smem + kSmemL)[r] = l;
        mbar_arrive(&bars[B_LF]);
        if (a.lse != nullptr && i < a.n && cur_cnt > 0)
          a.lse[(size_t)hh * a.n + i] = (m_used + log2f(l)) * 0.69314718055994531f;
        PT(9);
        sb += nsub / 2;
        pb += nsub;
        rb += 2 * nsub;
        continue;
      }
      mbar_wait(&bars[B_OF], J & 1);
      PT(8);
      tc_fence_after();
      const float inv = 1.0f / l;
      const bool valid = i < a.n && cur_cnt > 0;  // cnt == 0: query tile not requested
      if (SA_ATTN_TMA_STORE && a.tma_out) {
        // two 64-column halves through the swizzled stage; rows past n are
        // clipped by the TMA box bounds
        uint8_t* stage = smem + kSmemStage;
        const uint32_t st_addr = smem_u32(stage) + (uint32_t)r * 128u;
#pragma unroll 1
        for (int hf = 0; hf < 2; ++hf) {
          if (r == 0) bulk_wait_read0();  // the previous store has read the stage
          named_bar_sync(1, 128);
          uint32_t o[2][32];
          tmem_ld32(tbase + lane_off + kColO + 64 * hf, o[0]);
          tmem_ld32(tbase + lane_off + kColO + 64 * hf + 32, o[1]);
          tmem_ld_wait();
          if (hf == 1) {
            tc_fence_before();
            mbar_arrive(&bars[B_OE]);  // O may now be overwritten by the next item's PV(0)
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            uint32_t w[4];
#pragma unroll
            for (int t = 0; t < 4; ++t)
              w[t] = pack_bf16(__uint_as_float(o[j >> 2][(j & 3) * 8 + 2 * t]) * inv,
                               __uint_as_float(o[j >> 2][(j & 3) * 8 + 2 * t + 1]) * inv);
            st_shared_v4(st_addr + ((uint32_t)(j ^ (r & 7)) << 4), w[0], w[1], w[2], w[3]);
          }
          fence_proxy_async();
          named_bar_sync(1, 128);
          if (r == 0 && cur_cnt > 0) {
            tma_store_3d(&a.tmap_out, stage, h * kHeadDim + 64 * hf, qt * kTile, bidx);
            bulk_commit();
          }
        }
        if (valid && a.lse != nullptr) a.lse[(size_t)hh * a.n + i] = (m_used + log2f(l)) * 0.69314718055994531f;
        PT(9);
        sb += nsub / 2;
        pb += nsub;
        rb += 2 * nsub;
        continue;
      }
      const long long ooff = (long long)bidx * a.out_batch_stride + (long long)i * a.out_row_stride +
                             (long long)h * kHeadDim;
      __nv_bfloat16* orow = a.out + ooff;
      if (a.epi_mode == 2) {
        tc_fence_before();
        mbar_arrive(&bars[B_OE]);
      }
#pragma unroll 1
      for (int c = 0; c < (a.epi_mode == 2 ? 0 : 4); ++c) {
        uint32_t o[32];
        tmem_ld32(tbase + lane_off + kColO + 32 * c, o);
        tmem_ld_wait();
        if (c == 3) {
          tc_fence_before();
          mbar_arrive(&bars[B_OE]);  // O may now be overwritten by the next item's PV(0)
        }
        if (valid && a.epi_mode == 1) {
          uint32_t pk[16];
#pragma unroll
          for (int t = 0; t < 16; ++t)
            pk[t] = pack_bf16(__uint_as_float(o[2 * t]) * inv, __uint_as_float(o[2 * t + 1]) * inv);
          auto store = [&](__nv_bfloat16* row) {
            if (a.st256) {  // 32-byte stores: whole L2 sectors per lane
#pragma unroll
              for (int t = 0; t < 2; ++t) st_global_v8(row + 32 * c + 16 * t, pk + 8 * t);
            } else {
              uint4* dst = reinterpret_cast<uint4*>(row + 32 * c);
#pragma unroll
              for (int t = 0; t < 4; ++t)
                dst[t] = make_uint4(pk[4 * t], pk[4 * t + 1], pk[4 * t + 2], pk[4 * t + 3]);
            }
          };
          store(orow);
          // fused all-gather: the same bytes straight into every peer's output over NVLink
#pragma unroll 1
          for (int pr = 0; pr < a.n_peers; ++pr) store(a.peer_out[pr] + ooff);
        }
      }
      if (valid && a.lse != nullptr) a.lse[(size_t)hh * a.n + i] = (m_used + log2f(l)) * 0.69314718055994531f;
      PT(9);
      sb += nsub / 2;
      pb += nsub;
      rb += 2 * nsub;
    }
    if (SA_ATTN_TMA_STORE && a.tma_out && r == 0) bulk_wait0();  // every output store complete
    if (kProf) pc[11] += clock64() - t_entry;
    PT_FLUSH(0);
    if (!EWG && a.n_peers > 0) __threadfence_system();  // peer stores drained before the CTA retires
  } else if (EWG) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");  // warps 10-11: idle
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) tmem_dealloc(tbase, kTmemCols);
}

}  // namespace sa

// ------------------------------------------------------------------ C ABI
#include "api_common.h"
#include "internal.h"

static void* sa_attn_dbg_ptr = nullptr;

// Tool hook (not in the public header): in SA_ATTN_PROF builds the kernel adds
// its per-role phase cycles into p[0..48) (softmax, MMA, TMA producer).
extern "C" int sa_attn_profile_counters(void* p) { sa_attn_dbg_ptr = p; return 0; }

namespace sa {

int launch_attn(int batch, int heads, int kv_heads, int n, float scale, const void* q, const void* k,
                const void* v, void* out, const sa_head_index* index, const int32_t* tile_off,
                const int32_t* tile_cnt, const uint32_t* tiles, const int32_t* work, float* lse,
                cudaStream_t cs, long long out_ld, int* counter, const int32_t* n_work,
                void* const* peer_out, int n_peers, bool counter_zeroed) {
  if (batch < 1 || heads < 1 || kv_heads < 1 || n < 1)
    return fail(SA_ERR_DIMENSION, "need batch, heads, kv_heads, n >= 1");
  if (heads % kv_heads != 0)
    return fail(SA_ERR_DIMENSION, "heads=%d not a multiple of kv_heads=%d", heads, kv_heads);
  if (!(scale > 0.f) || !std::isfinite(scale))
    return fail(SA_ERR_DIMENSION, "scale must be positive and finite");
  if (!q || !k || !v || !out || !index || !tile_off || !tile_cnt || !tiles)
    return fail(SA_ERR_DIMENSION, "null pointer argument");
  AttnArgs a;
  memset(&a, 0, sizeof(a));
  int st;
  if ((st = make_tmap_3d_bf16(&a.tmap_q, q, kHeadDim, n, batch * heads, kTile))) return st;
  if ((st = make_tmap_3d_bf16(&a.tmap_k, k, kHeadDim, n, batch * kv_heads, kSub))) return st;
  if ((st = make_tmap_3d_bf16(&a.tmap_v, v, kHeadDim, n, batch * kv_heads, kSub))) return st;
  if ((st = make_tmap_kv_gather(&a.tmap_k8, k, n, batch * kv_heads))) return st;
  if ((st = make_tmap_kv_gather(&a.tmap_v8, v, n, batch * kv_heads))) return st;
  a.out = reinterpret_cast<__nv_bfloat16*>(out);
  a.out_row_stride = out_ld > 0 ? out_ld : (long long)heads * kHeadDim;
  a.out_batch_stride = (long long)n * a.out_row_stride;
  if (a.out_row_stride % 8 != 0 || (reinterpret_cast<uintptr_t>(out) & 15) != 0)
    return fail(SA_ERR_DIMENSION, "output rows must be 16-byte aligned (out_ld %% 8 == 0)");
  a.st256 = (a.out_row_stride % 16 == 0 && (reinterpret_cast<uintptr_t>(out) & 31) == 0) ? 1 : 0;
  static const int skip_dead = [] {
    const char* e = getenv("SA_ATTN_SKIP");  // A/B: 0 = every warp runs the softmax of every sub-tile
    return e ? atoi(e) : 1;
  }();
  a.skip_dead = skip_dead;
  static const int epi_mode = [] {
    const char* e = getenv("SA_ATTN_EPI");  // experiment only: output left unwritten when != 1
    return e ? atoi(e) : 1;
  }();
  a.epi_mode = epi_mode;
  if (n_peers < 0 || n_peers > kMaxPeers || (n_peers > 0 && !peer_out))
    return fail(SA_ERR_DIMENSION, "n_peers must be in [0, %d]", kMaxPeers);
  a.n_peers = n_peers;
  for (int p = 0; p < n_peers; ++p) {
    const uintptr_t pp = reinterpret_cast<uintptr_t>(peer_out[p]);
    if (!pp || (pp & 15) != 0) return fail(SA_ERR_DIMENSION, "peer output %d null or not 16-byte aligned", p);
    if ((pp & 31) != 0) a.st256 = 0;
    a.peer_out[p] = reinterpret_cast<__nv_bfloat16*>(peer_out[p]);
  }
  a.n = n;
  a.heads = heads;
  a.kv_heads = kv_heads;
  a.nqt = (n + kTile - 1) / kTile;
  if (SA_ATTN_TMA_STORE && n_peers == 0) {
    if ((st = make_tmap_out_bf16(&a.tmap_out, out, a.out_row_stride, n, batch, a.out_row_stride))) return st;
    a.tma_out = 1;
  }
  a.hh_total = batch * heads;
  a.scale_log2 = scale * 1.4426950408889634f;
  a.tile_off = tile_off;
  a.tile_cnt = tile_cnt;
  a.tiles = tiles;
  a.work = work;
  a.counter = counter;
  a.n_work = n_work;
  // (a memset between the work-order kernel and this launch would defeat PDL:
  // callers whose previous kernel already zeroed the counter say so)
  if (counter && !counter_zeroed) cudaMemsetAsync(counter, 0, sizeof(int), cs);
  a.idx = *index;
  a.lse = lse;
  a.prof = reinterpret_cast<unsigned long long*>(sa_attn_dbg_ptr);
  // exp split between MUFU and the FMA pipe (SA_ATTN_POLY overrides, for tuning)
  static const int poly = [] {
    const char* e = getenv("SA_ATTN_POLY");
    const int v = e ? atoi(e) : kDefaultPoly;
    return (v == 0 || v == 2 || v == 3 || v == 4 || v == 8) ? v : kDefaultPoly;
  }();
  // SA_ATTN_EWG=1: an epilogue warpgroup takes the output stores off the
  // softmax warps (384-thread CTAs).  Opt-in: measured slower (32K auto
  // attention 0.869 vs 0.828 ms, Block(8,1) 0.217 vs 0.209, VS 8.0 vs 7.7;
  // DESIGN.md), though removing the epilogue outright would save 4.6%.
  static const bool ewg = [] {
    const char* e = getenv("SA_ATTN_EWG");
    return e && e[0] == '1';
  }();
  static std::atomic<uint64_t> attr_done{0};
  once_per_device(attr_done, [] {
#define SA_ATTR(P)                                                                                           \
  cudaFuncSetAttribute(attn_fwd_kernel<P, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes); \
  cudaFuncSetAttribute(attn_fwd_kernel<P, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytesEwg);
    SA_ATTR(0) SA_ATTR(2) SA_ATTR(3) SA_ATTR(4) SA_ATTR(8)
#undef SA_ATTR
  });
  // persistent: two CTAs per SM (113 KB shared memory and 256 TMEM columns each)
  const int num_sms = device_sm_count();
  static const int per_sm = [] {
    const char* e = getenv("SA_ATTN_CTAS");  // A/B: CTAs per SM (default 2)
    const int v = e ? atoi(e) : 2;
    return v == 1 ? 1 : 2;
  }();
  const int grid = (int)std::min<long long>((long long)per_sm * num_sms, (long long)a.hh_total * a.nqt);
  // the need_weights path derives weights from lse: keep exact MUFU exps there
  void (*kern)(AttnArgs);
  switch (lse != nullptr ? 0 : poly) {
    case 2: kern = ewg ? attn_fwd_kernel<2, true> : attn_fwd_kernel<2, false>; break;
    case 3: kern = ewg ? attn_fwd_kernel<3, true> : attn_fwd_kernel<3, false>; break;
    case 4: kern = ewg ? attn_fwd_kernel<4, true> : attn_fwd_kernel<4, false>; break;
    case 8: kern = ewg ? attn_fwd_kernel<8, true> : attn_fwd_kernel<8, false>; break;
    default: kern = ewg ? attn_fwd_kernel<0, true> : attn_fwd_kernel<0, false>; break;
  }
  // programmatic dependent launch: the CTAs become resident and run their
  // prologue (barriers, TMEM, tensor-map prefetch) while the previous kernel
  // in the stream (the work-order kernel) finishes; griddepcontrol.wait in the
  // kernel orders every global read after it (SA_PDL=0: plain launch)
  static const bool pdl = [] {
    const char* e = getenv("SA_PDL");
    return !(e && e[0] == '0');
  }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(ewg ? kThreadsEwg : kThreads);
  cfg.dynamicSmemBytes = ewg ? kSmemBytesEwg : kSmemBytes;
  cfg.stream = cs;
  // highest scheduling priority: when a short-CTA kernel (the finiteness scan /
  // cache fill) runs beside it, freed SM slots go to attention CTAs first
  static const int prio = [] {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    const char* e = getenv("SA_ATTN_PRIO");  // A/B: 0 = stream priority
    return (e && e[0] == '0') ? 1 : hi;
  }();
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl && counter_zeroed) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (prio <= 0) {
    attr[na].id = cudaLaunchAttributePriority;
    attr[na].val.priority = prio;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  cudaLaunchKernelEx(&cfg, kern, a);
  return check_launch("attn_fwd_kernel");
}

}  // namespace sa

extern "C" int sa_attn_sparse(int batch, int heads, int kv_heads, int n, float scale,
                              const void* q, const void* k, const void* v, void* out,
                              const sa_head_index* index, const int32_t* tile_off,
                              const int32_t* tile_cnt, const uint32_t* tiles, float* lse,
                              void* stream) {
  return sa::launch_attn(batch, heads, kv_heads, n, scale, q, k, v, out, index, tile_off, tile_cnt,
                         tiles, nullptr, lse, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int sa_attn_sparse_work(int batch, int heads, int kv_heads, int n, float scale, const void* q,
                                   const void* k, const void* v, void* out, const sa_head_index* index,
                                   const int32_t* tile_off, const int32_t* tile_cnt, const uint32_t* tiles,
                                   const int32_t* work, const int32_t* n_work, int32_t* counter, long long out_ld,
                                   void* stream) {
  // the persistent kernel fetches items through `counter` (zeroed on the stream)
  if (!work || !n_work || !counter) return sa::fail(SA_ERR_DIMENSION, "null work list or counter");
  return sa::launch_attn(batch, heads, kv_heads, n, scale, q, k, v, out, index, tile_off, tile_cnt, tiles, work,
                         nullptr, reinterpret_cast<cudaStream_t>(stream), out_ld, counter, n_work);
}

extern "C" int sa_attn_sparse_work_peers(int batch, int heads, int kv_heads, int n, float scale, const void* q,
                                         const void* k, const void* v, void* out, void* const* peer_out,
                                         int n_peers, const sa_head_index* index, const int32_t* tile_off,
                                         const int32_t* tile_cnt, const uint32_t* tiles, const int32_t* work,
                                         const int32_t* n_work, int32_t* counter, long long out_ld,
                                         void* stream) {
  if (!work || !n_work || !counter) return sa::fail(SA_ERR_DIMENSION, "null work list or counter");
  return sa::launch_attn(batch, heads, kv_heads, n, scale, q, k, v, out, index, tile_off, tile_cnt, tiles, work,
                         nullptr, reinterpret_cast<cudaStream_t>(stream), out_ld, counter, n_work, peer_out,
                         n_peers);
}
