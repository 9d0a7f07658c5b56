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
// One CTA per head, everything in shared memory (cal <= 64, d <= 128).  The
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
constexpr int kSelThreads = 256;

struct SelectArgs {
  const __nv_bfloat16* q;  // [HH, n, 128]
  const __nv_bfloat16* k;  // [HK, n, 128]
  int n, heads, kv_heads, hh_total;
  int cal;
  float scale;
  int ncand;
  int cand_fam[3];  // family of candidate c (0 tri, 1 vs, 2 block)
  int cand_p1[3];   // tri window / vs k_v / block b
  int cand_p2[3];   // tri sinks / vs k_s / block k_b
  int32_t* choice_out;  // [HH] index of the chosen candidate
  int32_t* family_out;  // [HH] family of the chosen candidate (optional)
  double* err_out;      // [HH, 3] Frobenius errors (optional)
};

struct SelectSmem {
  float q[kCalMax][129];
  float k[kCalMax][129];
  float L[kCalMax][kCalMax + 1];   // scaled causal logits
  float Wd[kCalMax][kCalMax + 1];  // dense weights
  unsigned char M[kCalMax][kCalMax];  // candidate mask
  double colscore[kCalMax];
  double diagscore[kCalMax];
  float pq[kCalMax][129];  // pooled q (block candidate)
  float pk[kCalMax][129];
  float BL[kCalMax][kCalMax + 1];  // pooled logits
  unsigned char colsel[kCalMax];
  unsigned char diagsel[kCalMax];
  unsigned char blksel[kCalMax][kCalMax];
  double red[kSelThreads];
};

__device__ __forceinline__ double block_sum(double v, double* red) {
  red[threadIdx.x] = v;
  __syncthreads();
  for (int s = kSelThreads / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  const double r = red[0];
  __syncthreads();
  return r;
}

// stable top-k by rank: selected iff #{better} < k, better = larger score or
// equal score at a lower index (patterns.py:231-234)
__device__ __forceinline__ bool rank_selected(const double* s, int len, int j, int k) {
  int better = 0;
  const double v = s[j];
  for (int i = 0; i < len; ++i) better += (s[i] > v) || (s[i] == v && i < j);
  return better < k;
}

__global__ void __launch_bounds__(kSelThreads) select_kernel(SelectArgs a) {
  extern __shared__ __align__(16) unsigned char sraw[];
  SelectSmem& S = *reinterpret_cast<SelectSmem*>(sraw);
  const int hh = blockIdx.x;
  const int bidx = hh / a.heads, h = hh % a.heads;
  const int hkv = bidx * a.kv_heads + h / (a.heads / a.kv_heads);
  const int cal = a.cal, n = a.n;
  const int tid = threadIdx.x;
  const __nv_bfloat16* qb = a.q + ((size_t)hh * n + (n - cal)) * kHeadDim;
  const __nv_bfloat16* kb = a.k + ((size_t)hkv * n + (n - cal)) * kHeadDim;
  for (int e = tid; e < cal * kHeadDim; e += kSelThreads) {
    const int r = e / kHeadDim, d = e % kHeadDim;
    S.q[r][d] = __bfloat162float(qb[e]);
    S.k[r][d] = __bfloat162float(kb[e]);
  }
  __syncthreads();
  // dense logits, causal
  for (int e = tid; e < cal * cal; e += kSelThreads) {
    const int r = e / cal, c = e % cal;
    float acc = 0.f;
    if (c <= r) {
#pragma unroll 8
      for (int d = 0; d < kHeadDim; ++d) acc = fmaf(S.q[r][d], S.k[c][d], acc);
    }
    S.L[r][c] = acc * a.scale;
  }
  __syncthreads();
  // dense weights: one thread per row
  for (int r = tid; r < cal; r += kSelThreads) {
    float mx = -INFINITY;
    for (int c = 0; c <= r; ++c) mx = fmaxf(mx, S.L[r][c]);
    float sum = 0.f;
    for (int c = 0; c <= r; ++c) {
      const float e = expf(S.L[r][c] - mx);
      S.Wd[r][c] = e;
      sum += e;
    }
    for (int c = 0; c < cal; ++c) S.Wd[r][c] = (c <= r) ? S.Wd[r][c] / sum : 0.f;
  }
  __syncthreads();

  double best = INFINITY;
  int best_c = 0;
  for (int ci = 0; ci < a.ncand; ++ci) {
    const int fam = a.cand_fam[ci];
    const int p1 = a.cand_p1[ci], p2 = a.cand_p2[ci];
    if (fam == FAM_VS) {
      // exact scoring over all cal rows (patterns.py:182-202), float64 sums
      for (int j = tid; j < cal; j += kSelThreads) {
        double cs = 0.0, ds = 0.0;
        for (int r = 0; r < cal; ++r) cs += (double)S.Wd[r][j];
        for (int r = j; r < cal; ++r) ds += (double)S.Wd[r][r - j];
        S.colscore[j] = cs;
        S.diagscore[j] = ds;
      }
      __syncthreads();
      const int kv = min(p1, cal), ks = min(p2, cal);
      for (int j = tid; j < cal; j += kSelThreads) {
        S.colsel[j] = rank_selected(S.colscore, cal, j, kv);
        S.diagsel[j] = rank_selected(S.diagscore, cal, j, ks);
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
    // candidate mask
    for (int e = tid; e < cal * cal; e += kSelThreads) {
      const int r = e / cal, c = e % cal;
      bool m = false;
      if (c <= r) {
        if (fam == FAM_TRI) {
          m = (r - c < p1) || (c < p2) || (r == c);
        } else if (fam == FAM_VS) {
          m = S.colsel[c] || S.diagsel[r - c] || (r == c);
        } else {
          const int b = min(p1, cal);
          m = S.blksel[r / b][c / b];
        }
      }
      S.M[r][c] = m;
    }
    __syncthreads();
    // sparse weights per row vs dense, squared error in float64
    double part = 0.0;
    for (int r = tid; r < cal; r += kSelThreads) {
      float mx = -INFINITY;
      for (int c = 0; c <= r; ++c)
        if (S.M[r][c]) mx = fmaxf(mx, S.L[r][c]);
      float sum = 0.f;
      for (int c = 0; c <= r; ++c)
        if (S.M[r][c]) sum += expf(S.L[r][c] - mx);
      for (int c = 0; c < cal; ++c) {
        float w = 0.f;
        if (c <= r && S.M[r][c]) w = expf(S.L[r][c] - mx) / sum;
        const double dlt = (double)w - (double)S.Wd[r][c];
        part += dlt * dlt;
      }
    }
    const double err = sqrt(block_sum(part, S.red));
    if (tid == 0) {
      if (a.err_out) a.err_out[(size_t)hh * 3 + ci] = err;
    }
    if (err < best) {
      best = err;
      best_c = ci;
    }
    __syncthreads();
  }
  if (tid == 0) {
    a.choice_out[hh] = best_c;
    if (a.family_out) a.family_out[hh] = a.cand_fam[best_c];
  }
}

}  // namespace sa

namespace sa {
int launch_select(int batch, int heads, int kv_heads, int n, int cal, float scale, const void* q,
                  const void* k, int ncand, const int32_t* cand_fam, const int32_t* cand_p1,
                  const int32_t* cand_p2, int32_t* choice_out, int32_t* family_out,
                  double* err_out, cudaStream_t stream) {
  if (batch < 1 || heads < 1 || kv_heads < 1 || heads % kv_heads)
    return fail(SA_ERR_DIMENSION, "bad head layout");
  if (cal < 1 || cal > n) return fail(SA_ERR_SEARCH, "cal_window must be in [1, %d], got %d", n, cal);
  if (cal > kCalMax) return fail(SA_ERR_SEARCH, "device selector supports cal_window <= %d", kCalMax);
  if (ncand < 1 || ncand > 3) return fail(SA_ERR_SEARCH, "candidate list must hold 1..3 patterns");
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
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(SelectSmem));
    attr = true;
  }
  select_kernel<<<a.hh_total, kSelThreads, sizeof(SelectSmem), stream>>>(a);
  return check_launch("select_kernel");
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
