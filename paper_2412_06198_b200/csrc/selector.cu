// selector.cu — the kernel-aware per-head pattern selector, on device.
//
// Reference: search.py:276-319 (select_pattern_windowed) -> search.py:209-258
// (select_pattern, scoring="exact", metric="weights").  For every head, the
// trailing `cal` rows form a standalone causal sub-problem (search.py:304-306).
// The kernel computes its dense weights (core.py:138-154), realises each
// refined candidate with exact scoring (patterns.py:324-343 at n = cal), forms
// the candidate's sparse weights (softmax restricted to the realised
// positions, patterns.py:353-484) and the Frobenius distance to the dense
// weights in float64 (core.py:179-186), then takes the strict-< argmin in
// candidate order (search.py:245-250: the earlier candidate wins ties).
//
// One CTA per (head, candidate), everything in shared memory (cal <= 64, d <= 128).  The
// family id written per head indexes the caller's candidate list; the host
// has already refined the candidates and rescaled them to n (search.py:
// 236-241, 261-273 — data-independent integer math).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "api_common.h"
#include "internal.h"
#include "sa_types.h"

namespace sa {

constexpr int kCalMax = 64;
constexpr int kSelThreads = 512;

struct SelectArgs {
  const __nv_bfloat16* q;  // [HH, n, 128]
  const __nv_bfloat16* k;  // [HK, n, 128]
  int n, heads, kv_heads, hh_total;
  int cal;
  float scale;
  int ncand;
  int cand_fam[SA_MAX_CAND];  // family of candidate c (0 tri, 1 vs, 2 block)
  int cand_p1[SA_MAX_CAND];   // tri window / vs k_v / block b
  int cand_p2[SA_MAX_CAND];   // tri sinks / vs k_s / block k_b
  int32_t* choice_out;  // [HH] index of the chosen candidate
  int32_t* family_out;  // [HH] family of the chosen candidate (optional)
  double* err_out;      // [HH, SA_MAX_CAND] Frobenius errors (optional)
  int apply;            // SelectApply below is set
  SelectApply ap;
};

struct SelectSmem {
  float q[kCalMax][132];  // 16-byte rows: the logit loop reads float4 along d
  float k[kCalMax][132];
  float L[kCalMax][kCalMax + 1];   // scaled causal logits
  float Wd[kCalMax][kCalMax + 1];  // dense weights
  double colscore[kCalMax];
  double diagscore[kCalMax];
  float pq[kCalMax][129];  // pooled q (block candidate)
  float pk[kCalMax][129];
  float BL[kCalMax][kCalMax + 1];  // pooled logits
  unsigned char colsel[kCalMax];
  unsigned char diagsel[kCalMax];
  unsigned char blksel[kCalMax][kCalMax];
  double red[kSelThreads / 32];
  // bf16 copies of the windows for the tensor-core logits (rows padded to 272 B:
  // conflict-free ldmatrix)
  __align__(16) __nv_bfloat16 q16[kCalMax][136];
  __align__(16) __nv_bfloat16 k16[kCalMax][136];
};

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One CTA per (head, candidate): blockIdx.x = head, blockIdx.y = candidate.
// The dense part (logits, dense weights) is recomputed by each candidate's CTA
// so the candidates run in parallel; rows are processed one warp per row with
// shuffle reductions.  Writes err[hh, c]; select_argmin_kernel picks per head.
__global__ void __launch_bounds__(kSelThreads) select_kernel(SelectArgs a) {
  extern __shared__ __align__(16) unsigned char sraw[];
  SelectSmem& S = *reinterpret_cast<SelectSmem*>(sraw);
  const int hh = blockIdx.x;
  const int ci = blockIdx.y;
  const int bidx = hh / a.heads, h = hh % a.heads;
  const int hkv = bidx * a.kv_heads + h / (a.heads / a.kv_heads);
  const int cal = a.cal, n = a.n;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int kWarps = kSelThreads / 32;
  const __nv_bfloat16* qb = a.q + ((size_t)hh * n + (n - cal)) * kHeadDim;
  const __nv_bfloat16* kb = a.k + ((size_t)hkv * n + (n - cal)) * kHeadDim;
  {
    // 16-byte loads, all issued before any is consumed (one memory latency)
    constexpr int kVec = kCalMax * kHeadDim / 8 / kSelThreads;  // uint4 per thread per matrix
    uint4 qv[kVec], kv[kVec];
#pragma unroll
    for (int u = 0; u < kVec; ++u) {
      const int e = tid + u * kSelThreads;  // uint4 index: row e / 16, columns 8 (e % 16) ..
      const bool ok = e < cal * (kHeadDim / 8);
      qv[u] = ok ? __ldg(reinterpret_cast<const uint4*>(qb) + e) : make_uint4(0, 0, 0, 0);
      kv[u] = ok ? __ldg(reinterpret_cast<const uint4*>(kb) + e) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < kVec; ++u) {
      const int e = tid + u * kSelThreads;  // every row of the bf16 copies (zeros past cal)
      *reinterpret_cast<uint4*>(&S.q16[e / (kHeadDim / 8)][8 * (e % (kHeadDim / 8))]) = qv[u];
      *reinterpret_cast<uint4*>(&S.k16[e / (kHeadDim / 8)][8 * (e % (kHeadDim / 8))]) = kv[u];
      if (e < cal * (kHeadDim / 8)) {
        const int r = e / (kHeadDim / 8), d = 8 * (e % (kHeadDim / 8));
        const uint32_t qw[4] = {qv[u].x, qv[u].y, qv[u].z, qv[u].w};
        const uint32_t kw[4] = {kv[u].x, kv[u].y, kv[u].z, kv[u].w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float2 a2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&qw[t]));
          const float2 b2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&kw[t]));
          S.q[r][d + 2 * t] = a2.x;
          S.q[r][d + 2 * t + 1] = a2.y;
          S.k[r][d + 2 * t] = b2.x;
          S.k[r][d + 2 * t + 1] = b2.y;
        }
      }
    }
  }
  __syncthreads();
  // dense causal logits on the tensor cores (mma.sync m16n8k16, bf16 in, fp32
  // accumulate: the products of bf16 values are exact, only the summation
  // order differs from a sequential fp32 dot): warp w owns rows 16 (w / 4) ..
  // + 15 and columns 16 (w % 4) .. + 15
  {
    static_assert(kCalMax == 64 && kWarps == 16, "one 16 x 16 logit block per warp");
    const int mb = wid >> 2, nb = wid & 3;
    const int g = lane >> 2, t = lane & 3;
    float c[2][4] = {};
#pragma unroll
    for (int ks = 0; ks < kHeadDim / 16; ++ks) {
      uint32_t af[4], bq[4];
      const uint32_t aaddr =
          static_cast<uint32_t>(__cvta_generic_to_shared(&S.q16[16 * mb + (lane & 15)][16 * ks + (lane >> 4) * 8]));
      asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                   : "=r"(af[0]), "=r"(af[1]), "=r"(af[2]), "=r"(af[3])
                   : "r"(aaddr));
      const uint32_t baddr = static_cast<uint32_t>(__cvta_generic_to_shared(
          &S.k16[16 * nb + ((lane >> 4) << 3) + (lane & 7)][16 * ks + ((lane >> 3) & 1) * 8]));
      asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                   : "=r"(bq[0]), "=r"(bq[1]), "=r"(bq[2]), "=r"(bq[3])
                   : "r"(baddr));
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+f"(c[nt][0]), "+f"(c[nt][1]), "+f"(c[nt][2]), "+f"(c[nt][3])
            : "r"(af[0]), "r"(af[1]), "r"(af[2]), "r"(af[3]), "r"(bq[2 * nt]), "r"(bq[2 * nt + 1]));
    }
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          const int r = 16 * mb + g + 8 * h, cc = 16 * nb + 8 * nt + 2 * t + x;
          if (r < cal && cc < cal) S.L[r][cc] = (cc <= r) ? c[nt][2 * h + x] * a.scale : 0.f;
        }
  }
  __syncthreads();
  // dense weights (core.py:138-154): one warp per row, the warp's rows
  // (wid, wid + 16, ...) side by side so their shuffle / exp latencies overlap
  {
    constexpr int kR = kCalMax / kWarps;
    float l[kR][2], mx[kR], e[kR][2], sm[kR];
#pragma unroll
    for (int i = 0; i < kR; ++i) {
      const int r = wid + kWarps * i;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int c = lane + 32 * t;
        l[i][t] = (r < cal && c <= r && c < cal) ? S.L[r][c] : -INFINITY;
      }
      mx[i] = fmaxf(l[i][0], l[i][1]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int i = 0; i < kR; ++i) mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], o));
#pragma unroll
    for (int i = 0; i < kR; ++i) {
      const int r = wid + kWarps * i;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int c = lane + 32 * t;
        e[i][t] = (r < cal && c <= r && c < cal) ? expf(l[i][t] - mx[i]) : 0.f;
      }
      sm[i] = e[i][0] + e[i][1];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int i = 0; i < kR; ++i) sm[i] += __shfl_xor_sync(0xffffffffu, sm[i], o);
#pragma unroll
    for (int i = 0; i < kR; ++i) {
      const int r = wid + kWarps * i;
      if (r < cal) {
        if (lane < cal) S.Wd[r][lane] = e[i][0] / sm[i];
        if (lane + 32 < cal) S.Wd[r][lane + 32] = e[i][1] / sm[i];
      }
    }
  }
  __syncthreads();

  // (selects, not a dynamic index, so the parameter arrays stay in constant space)
  const int fam = ci == 0 ? a.cand_fam[0] : (ci == 1 ? a.cand_fam[1] : a.cand_fam[2]);
  const int p1 = ci == 0 ? a.cand_p1[0] : (ci == 1 ? a.cand_p1[1] : a.cand_p1[2]);
  const int p2 = ci == 0 ? a.cand_p2[0] : (ci == 1 ? a.cand_p2[1] : a.cand_p2[2]);
  if (fam == FAM_VS) {
    // exact scoring over all cal rows (patterns.py:182-202), float64 sums;
    // 8 threads per column / offset j, each over every 8th row, lane-reduced
    static_assert(kSelThreads >= 8 * kCalMax, "one 8-lane group per column");
    const int j = tid >> 3, part = tid & 7;
    double cs = 0.0, ds = 0.0;
    if (j < cal)
      for (int r = part; r < cal; r += 8) {
        cs += (double)S.Wd[r][j];
        if (r >= j) ds += (double)S.Wd[r][r - j];
      }
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      cs += __shfl_xor_sync(0xffffffffu, cs, o);
      ds += __shfl_xor_sync(0xffffffffu, ds, o);
    }
    if (part == 0 && j < cal) {
      S.colscore[j] = cs;
      S.diagscore[j] = ds;
    }
    __syncthreads();
    // stable top-k by rank (patterns.py:231-234): selected iff #{better} < k
    const int kv = min(p1, cal), ks = min(p2, cal);
    int bc = 0, bd = 0;
    if (j < cal) {
      const double vc = S.colscore[j], vd = S.diagscore[j];
      for (int i = part; i < cal; i += 8) {
        bc += (S.colscore[i] > vc) || (S.colscore[i] == vc && i < j);
        bd += (S.diagscore[i] > vd) || (S.diagscore[i] == vd && i < j);
      }
    }
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      bc += __shfl_xor_sync(0xffffffffu, bc, o);
      bd += __shfl_xor_sync(0xffffffffu, bd, o);
    }
    if (part == 0 && j < cal) {
      S.colsel[j] = bc < kv;
      S.diagsel[j] = bd < ks;
    }
    __syncthreads();
  } else if (fam == FAM_BLOCK) {
    const int b = min(p1, cal);
    const int nb = (cal + b - 1) / b;
    const int kbk = min(p2, nb);
    for (int e = tid; e < nb * kHeadDim; e += kSelThreads) {
      const int g = e / kHeadDim, d = e % kHeadDim;
      const int r0 = g * b, r1 = min(cal, r0 + b);
      float sq = 0.f, sk = 0.f;
      for (int r = r0; r < r1; ++r) {
        sq += S.q[r][d];
        sk += S.k[r][d];
      }
      S.pq[g][d] = sq / (float)(r1 - r0);
      S.pk[g][d] = sk / (float)(r1 - r0);
    }
    __syncthreads();
    for (int e = tid; e < nb * nb; e += kSelThreads) {
      const int g = e / nb, c = e % nb;
      float acc = 0.f;
      for (int d = 0; d < kHeadDim; ++d) acc = fmaf(S.pq[g][d], S.pk[c][d], acc);
      S.BL[g][c] = acc * a.scale;
    }
    __syncthreads();
    for (int e = tid; e < nb * nb; e += kSelThreads) {
      const int g = e / nb, c = e % nb;
      bool sel = false;
      if (c <= g) {
        const int keff = min(kbk, g + 1);
        int better = 0;
        const float v = S.BL[g][c];
        for (int i = 0; i <= g; ++i) better += (S.BL[g][i] > v) || (S.BL[g][i] == v && i < c);
        sel = (better < keff) || (c == g);
      }
      S.blksel[g][c] = sel;
    }
    __syncthreads();
  }
  // sparse weights per row vs dense, squared error in float64 (core.py:179-186);
  // the candidate's mask is evaluated in place; the warp's rows side by side,
  // each thread's float64 partial summed in row order as before
  double part = 0.0;
  {
    constexpr int kR = kCalMax / kWarps;
    auto in_mask = [&](int r, int c) -> bool {
      if (c > r) return false;
      if (fam == FAM_TRI) return (r - c < p1) || (c < p2) || (r == c);
      if (fam == FAM_VS) return S.colsel[c] || S.diagsel[r - c] || (r == c);
      const int b = min(p1, cal);
      return S.blksel[r / b][c / b];
    };
    float lv[kR][2], mx[kR], ev[kR][2], sm[kR];
    bool mv[kR][2];
#pragma unroll
    for (int i = 0; i < kR; ++i) {
      const int r = wid + kWarps * i;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int c = lane + 32 * t;
        mv[i][t] = r < cal && c < cal && in_mask(r, c);
        lv[i][t] = mv[i][t] ? S.L[r][c] : -INFINITY;
      }
      mx[i] = fmaxf(lv[i][0], lv[i][1]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int i = 0; i < kR; ++i) mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], o));
#pragma unroll
    for (int i = 0; i < kR; ++i) {
#pragma unroll
      for (int t = 0; t < 2; ++t) ev[i][t] = mv[i][t] ? expf(lv[i][t] - mx[i]) : 0.f;
      sm[i] = ev[i][0] + ev[i][1];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int i = 0; i < kR; ++i) sm[i] += __shfl_xor_sync(0xffffffffu, sm[i], o);
#pragma unroll
    for (int i = 0; i < kR; ++i) {
      const int r = wid + kWarps * i;
      if (r < cal) {
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int c = lane + 32 * t;
          if (c < cal) {
            const float w = mv[i][t] ? ev[i][t] / sm[i] : 0.f;
            const double dlt = (double)w - (double)S.Wd[r][c];
            part += dlt * dlt;
          }
        }
      }
    }
  }
  part = warp_sum(part);
  if (lane == 0) S.red[wid] = part;
  __syncthreads();
  if (tid == 0) {
    double tot = 0.0;
    for (int w = 0; w < kWarps; ++w) tot += S.red[w];
    a.err_out[(size_t)hh * SA_MAX_CAND + ci] = sqrt(tot);
    if (a.apply) {
      // the head's last candidate CTA: strict-< argmin in candidate order
      // (search.py:245-250; NaN never wins, all-NaN -> candidate 0) and the
      // chosen pattern's per-head parameters (what apply_choice_kernel writes)
      __threadfence();
      if (atomicAdd(&a.ap.counter[hh], 1) == a.ncand - 1) {
        a.ap.counter[hh] = 0;
        __threadfence();
        double best = INFINITY;
        int bc = 0;
        for (int c = 0; c < a.ncand; ++c) {
          const double e = __ldcg(&a.err_out[(size_t)hh * SA_MAX_CAND + c]);
          if (e < best) {
            best = e;
            bc = c;
          }
        }
        a.choice_out[hh] = bc;
        if (a.family_out) a.family_out[hh] = a.cand_fam[bc];
        const sa_pattern pf = a.ap.full[bc];
        a.ap.family[hh] = pf.family;
        a.ap.tri_w[hh] = pf.family == SA_TRIANGULAR ? pf.p1 : 1;
        a.ap.tri_s[hh] = pf.family == SA_TRIANGULAR ? pf.p2 : 0;
        a.ap.blk_b[hh] = pf.family == SA_BLOCK_SPARSE ? pf.p1 : 1;
      }
    }
  }
}

// strict-< argmin in candidate order (search.py:245-250: earlier wins ties)
struct CandFamilies {
  int f[SA_MAX_CAND];
};
__global__ void select_argmin_kernel(const double* err, int hh_total, int ncand, int32_t* choice_out,
                                     int32_t* family_out, CandFamilies fam) {
  const int hh = blockIdx.x * blockDim.x + threadIdx.x;
  if (hh >= hh_total) return;
  double best = INFINITY;
  int best_c = 0;
  for (int c = 0; c < ncand; ++c) {
    const double e = err[(size_t)hh * SA_MAX_CAND + c];
    if (e < best) {
      best = e;
      best_c = c;
    }
  }
  choice_out[hh] = best_c;
  if (family_out) family_out[hh] = fam.f[best_c];
}

}  // namespace sa

namespace sa {
int launch_select(int batch, int heads, int kv_heads, int n, int cal, float scale, const void* q,
                  const void* k, int ncand, const int32_t* cand_fam, const int32_t* cand_p1,
                  const int32_t* cand_p2, int32_t* choice_out, int32_t* family_out,
                  double* err_out, cudaStream_t stream, const SelectApply* apply) {
  if (batch < 1 || heads < 1 || kv_heads < 1 || heads % kv_heads)
    return fail(SA_ERR_DIMENSION, "bad head layout");
  if (cal < 1 || cal > n) return fail(SA_ERR_SEARCH, "cal_window must be in [1, %d], got %d", n, cal);
  if (cal > kCalMax) return fail(SA_ERR_SEARCH, "device selector supports cal_window <= %d", kCalMax);
  if (ncand < 1 || ncand > SA_MAX_CAND)
    return fail(SA_ERR_SEARCH, "candidate list must hold 1..%d patterns", SA_MAX_CAND);
  SelectArgs a{};
  a.q = reinterpret_cast<const __nv_bfloat16*>(q);
  a.k = reinterpret_cast<const __nv_bfloat16*>(k);
  a.n = n;
  a.heads = heads;
  a.kv_heads = kv_heads;
  a.hh_total = batch * heads;
  a.cal = cal;
  a.scale = scale;
  a.ncand = ncand;
  for (int c = 0; c < ncand; ++c) {
    a.cand_fam[c] = cand_fam[c];
    a.cand_p1[c] = cand_p1[c];
    a.cand_p2[c] = cand_p2[c];
    if (cand_fam[c] < 0 || cand_fam[c] > 2) return fail(SA_ERR_SEARCH, "unknown candidate family");
  }
  a.choice_out = choice_out;
  a.family_out = family_out;
  a.err_out = err_out;
  static std::atomic<uint64_t> attr_done{0};
  once_per_device(attr_done, [] {
    cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SelectSmem));
  });
  if (!a.err_out) {  // callers that do not want the errors still need a scratch row per head
    // per (thread, device): a buffer freed while another stream uses it would race
    struct Scratch {
      double* p = nullptr;
      int heads = 0;
    };
    static thread_local Scratch tab[64];
    Scratch& s = tab[current_device() & 63];
    if (s.heads < a.hh_total) {
      if (s.p) cudaFree(s.p);
      if (cudaMalloc(&s.p, (size_t)a.hh_total * SA_MAX_CAND * sizeof(double)) != cudaSuccess)
        return fail(SA_ERR_CUDA, "selector scratch allocation failed");
      s.heads = a.hh_total;
    }
    a.err_out = s.p;
  }
  if (apply) {
    if (!choice_out || !apply->counter) return fail(SA_ERR_DIMENSION, "selector apply needs choice and counter");
    a.apply = 1;
    a.ap = *apply;
    cudaMemsetAsync(apply->counter, 0, (size_t)a.hh_total * sizeof(int), stream);
  }
  select_kernel<<<dim3(a.hh_total, ncand), kSelThreads, sizeof(SelectSmem), stream>>>(a);
  int rc = check_launch("select_kernel");
  if (rc || apply) return rc;
  CandFamilies fams{};
  for (int c = 0; c < ncand; ++c) fams.f[c] = a.cand_fam[c];
  select_argmin_kernel<<<(a.hh_total + 127) / 128, 128, 0, stream>>>(a.err_out, a.hh_total, ncand, choice_out,
                                                                    family_out, fams);
  return check_launch("select_argmin_kernel");
}
}  // namespace sa

extern "C" int sa_select_windowed(int batch, int heads, int kv_heads, int n, int cal, float scale,
                                  const void* q, const void* k, int ncand,
                                  const int32_t* cand_fam_host, const int32_t* cand_p1_host,
                                  const int32_t* cand_p2_host, int32_t* choice_out,
                                  int32_t* family_out, double* err_out, void* stream) {
  return sa::launch_select(batch, heads, kv_heads, n, cal, scale, q, k, ncand, cand_fam_host,
                           cand_p1_host, cand_p2_host, choice_out, family_out, err_out,
                           reinterpret_cast<cudaStream_t>(stream));
}

// search.py:245-250: per row the strict-< argmin over the candidates' errors
// (the earlier candidate wins ties; NaN never wins; all-NaN -> candidate 0).
namespace sa {
__global__ void select_family_kernel(const double* err, long long ld, int rows, int ncand, int32_t* out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  double best = INFINITY;
  int bc = 0;
  for (int c = 0; c < ncand; ++c) {
    const double e = err[(size_t)r * ld + c];
    if (e < best) {
      best = e;
      bc = c;
    }
  }
  out[r] = bc;
}
}  // namespace sa

extern "C" int sa_select_family(const double* err, long long ld, int rows, int ncand, int32_t* choice_out,
                                void* stream) {
  using namespace sa;
  if (rows < 0 || ncand < 1 || ld < ncand) return fail(SA_ERR_SEARCH, "bad error matrix shape");
  if (rows == 0) return SA_OK;
  if (!err || !choice_out) return fail(SA_ERR_DIMENSION, "null pointer");
  select_family_kernel<<<(rows + 255) / 256, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(err, ld, rows, ncand,
                                                                                              choice_out);
  return check_launch("select_family_kernel");
}
