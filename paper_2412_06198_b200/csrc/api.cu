// api.cu — extern "C" boundary (include/sparseattn_b200.h): argument checks
// mapped to the reference's exception classes, tensor-map encoding, launches.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "api_common.h"
#include "sa_types.h"

namespace sa {


static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

int fail(int status, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return status;
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

int make_tmap_3d_bf16(CUtensorMap* map, const void* base, int d0, int d1, int d2, int box_rows) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return fail(SA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)d2};
  cuuint64_t strides[2] = {(cuuint64_t)d0 * 2, (cuuint64_t)d0 * 2 * (cuuint64_t)d1};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SA_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return SA_OK;
}

// The attention output [B][n][row_stride] bf16 as a 3-D map {cols, n, B} with
// box {64 cols, 128 rows, 1}: TMA stores clip rows past n inside each batch.
int make_tmap_out_bf16(CUtensorMap* map, void* base, long long cols, int n, int batch, long long row_stride) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return fail(SA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)n, (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)row_stride * 2, (cuuint64_t)row_stride * 2 * (cuuint64_t)n};
  cuuint32_t box[3] = {64, 128, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SA_ERR_CUDA, "cuTensorMapEncodeTiled (out) failed (%d)", (int)r);
  return SA_OK;
}

// K/V viewed as [groups][n rows][2 d-halves][64] with the halves as the box's
// outer dim: one box {64, 8, 2} = 8 rows x both halves = 2 KB, laid out in
// shared memory as [half][8 rows][128 B] (two SWIZZLE_128B atoms).
int make_tmap_kv_gather(CUtensorMap* map, const void* base, int n, int groups) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return fail(SA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[4] = {64, (cuuint64_t)n, 2, (cuuint64_t)groups};
  cuuint64_t strides[3] = {256, 128, (cuuint64_t)n * 256};
  cuuint32_t box[4] = {64, 8, 2, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SA_ERR_CUDA, "cuTensorMapEncodeTiled (gather map) failed (%d)", (int)r);
  return SA_OK;
}

}  // namespace sa

extern "C" {

const char* sa_last_error(void) { return sa::g_last_error.c_str(); }

int sa_version(void) { return 1; }

// CUDA IPC for the fused output all-gather (multigpu.PeerOutputs): a rank's
// output buffer is its own cudaMalloc allocation, so the opened mapping starts
// at the buffer (no sub-allocation offset to carry).
int sa_ipc_alloc(size_t bytes, void** ptr, void* handle) {
  if (!ptr || !handle || bytes == 0) return sa::fail(SA_ERR_DIMENSION, "sa_ipc_alloc: bad arguments");
  if (sizeof(cudaIpcMemHandle_t) > SA_IPC_HANDLE_BYTES) return sa::fail(SA_ERR_CUDA, "IPC handle size");
  cudaError_t e = cudaMalloc(ptr, bytes);
  if (e != cudaSuccess) return sa::fail(SA_ERR_CUDA, "cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e));
  cudaIpcMemHandle_t h;
  e = cudaIpcGetMemHandle(&h, *ptr);
  if (e != cudaSuccess) {
    cudaFree(*ptr);
    *ptr = nullptr;
    return sa::fail(SA_ERR_CUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
  }
  memset(handle, 0, SA_IPC_HANDLE_BYTES);
  memcpy(handle, &h, sizeof(h));
  return SA_OK;
}

int sa_ipc_free(void* ptr) {
  const cudaError_t e = cudaFree(ptr);
  return e == cudaSuccess ? SA_OK : sa::fail(SA_ERR_CUDA, "cudaFree: %s", cudaGetErrorString(e));
}

int sa_ipc_open(const void* handle, void** ptr) {
  if (!ptr || !handle) return sa::fail(SA_ERR_DIMENSION, "sa_ipc_open: bad arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  const cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? SA_OK : sa::fail(SA_ERR_CUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
}

int sa_ipc_close(void* ptr) {
  const cudaError_t e = cudaIpcCloseMemHandle(ptr);
  return e == cudaSuccess ? SA_OK : sa::fail(SA_ERR_CUDA, "cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
}

}  // extern "C"
