// common.cuh -- error plumbing shared by the libbnff translation units.
#pragma once
#include <cstdarg>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../include/bnff.h"

namespace bnff {

// thread-local last-error message returned by bnff_last_error()
char* last_error_buf();

inline int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(last_error_buf(), 512, fmt, ap);
  va_end(ap);
  return code;
}
inline int set_cuda_error(cudaError_t e, const char* where) {
  return set_error(BNFF_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}
inline int check_launch(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, where);
  return BNFF_OK;
}

}  // namespace bnff

// sum over pixels of the (optionally BN_DX-transformed) gradient -> dbias (fp32, c);
// scratch holds [bnff_sum_tiles(pixels)][2][c] partials
extern "C" int bnff_dbias_scratch(int32_t dtype, bnff_view dy, bnff_view dy_x, int32_t dy_pro,
                                  bnff_coef coef, float* scratch, float* dbias, void* stream);
