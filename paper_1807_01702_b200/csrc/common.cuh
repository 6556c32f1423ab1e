// common.cuh -- error plumbing shared by the libbnff translation units.
#pragma once
#include <cstdarg>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../include/bnff.h"

// 3xTF32 MMAs with a stacked B operand (2 MMAs per K step instead of 3); -DBNFF_TF32_STACK=0
// restores the three-MMA issue for A/B timing
#ifndef BNFF_TF32_STACK
#define BNFF_TF32_STACK 1
#endif

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
                                  bnff_coef coef, double* scratch, float* dbias, void* stream);

// wgrad32.cu / wconv.cu internals shared with igemm.cu's bnff_conv_wgrad
extern "C" int64_t bnff_wgrad_f32_ws(int32_t n, int32_t h, int32_t w, int32_t kh, int32_t c_in, int32_t c_out);
extern "C" int bnff_wgrad_f32_partials(bnff_view x, int32_t x_pro, bnff_coef x_coef, bnff_view dy, bnff_view dy_x,
                                       int32_t dy_pro, bnff_coef dy_coef, int32_t kh, float* ws, int32_t want_db,
                                       int32_t* splits_out, void* stream);
extern "C" int bnff_wgrad_reduce(const float* ws, int32_t splits, int32_t taps, int32_t cin, int32_t cout,
                                 int32_t cin_real, float* dw, const float* wsb, float* dbias, void* stream);

#include <cstdlib>
#include <utility>

namespace bnff {
// ---------------------------------------------------------------------------
// programmatic dependent launch (PDL): every libbnff kernel is launched with
// programmatic stream serialization, triggers its dependents at entry and waits
// (griddepcontrol.wait) before touching data produced by earlier launches, so the
// next kernel's launch and prologue overlap this kernel's tail.  BNFF_PDL=0 disables.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
inline int pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BNFF_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v;
}
template <typename... KArgs, typename... Args>
inline void launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                   Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
}  // namespace bnff
