// api_common.h — error state and helpers shared by the extern "C" entry points.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <string>

#include "sparseattn_b200.h"

namespace sa {

void set_error(const char* fmt, ...);
int fail(int status, const char* fmt, ...);

// Encode a 3-D bf16 tensor map over a [d2, d1, d0=128] row-major tensor,
// box {64, box_rows, 1}, 128-byte swizzle.
int make_tmap_3d_bf16(CUtensorMap* map, const void* base, int d0, int d1, int d2, int box_rows);
int make_tmap_kv_gather(CUtensorMap* map, const void* base, int n, int groups);
int make_tmap_out_bf16(CUtensorMap* map, void* base, long long cols, int n, int batch, long long row_stride);

inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(SA_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return SA_OK;
}

}  // namespace sa
