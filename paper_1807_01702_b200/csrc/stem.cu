// stem.cu -- channel-poor stem convolution (the DenseNet/ResNet 7x7/s2 conv over the
// 3-channel image, graph.py:358-375 of the reference) recast as a dense GEMM.
//
// The image is stored NHWC with its 3 channels padded to 8 (16 B per pixel).  Read as an
// implicit GEMM directly, every output pixel gathers 49 16-byte chunks of which 5/8 are
// padding (K = 392 for 147 real taps*channels) and the gather is latency-bound.  Here one
// HBM-bound pass writes the packed patch matrix col[p][k], k = (ky*kw + kx)*c + ci
// (K = 147 padded to 160), after which the forward conv is a 1x1 conv over col (the
// window-shift tcgen05 kernel, with its bias / sub-BN1 statistics epilogue) and the
// weight gradient is that 1x1 conv's wgrad; two tiny kernels move the weights between
// the reference layout (co, ci, kh, kw) and the (co, k) matrix.
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "sm100.cuh"
#include "common.cuh"

namespace bnff {
namespace stem {

// one CTA: tp consecutive output pixels of one output row.  The kh input rows the tile
// touches are staged in shared memory as 16-byte pixels; a per-CTA table maps each patch
// column k to its element offset in that stage (-1: K padding), so every thread builds
// whole 16-byte chunks of patch rows (8 table-driven shared loads) and stores them
// coalesced.
template <typename T>
__global__ void __launch_bounds__(256) im2col_kernel(const T* __restrict__ x, long long x_rs,
                                                     int h, int w, int oh, int ow, int kh, int kw,
                                                     int stride, int pad, int creal, int kpad, int tp,
                                                     T* __restrict__ col, long long col_rs) {
  griddep_launch();
  constexpr int EPP = 16 / (int)sizeof(T);  // elements per stored pixel / per 16-byte chunk
  extern __shared__ uint4 tile[];  // [kh][tw] 16-byte pixels (8 bf16 / 4 fp32), then int koff[kpad]
  const int tpr = (ow + tp - 1) / tp;
  const int b = blockIdx.x;
  const int row = b / tpr;  // img * oh + oy
  const int ox0 = (b - row * tpr) * tp;
  const int img = row / oh, oy = row - img * oh;
  const int tw = (tp - 1) * stride + kw;
  const int ix0 = ox0 * stride - pad, iy0 = oy * stride - pad;
  const int K = kh * kw * creal;
  const int np = min(tp, ow - ox0);
  int* koff = reinterpret_cast<int*>(tile + kh * tw);
  for (int k = threadIdx.x; k < kpad; k += blockDim.x) {
    int o = -1;
    if (k < K) {
      const int tap = k / creal, ci = k - tap * creal;
      const int ky = tap / kw, kx = tap - ky * kw;
      o = (ky * tw + kx) * EPP + ci;
    }
    koff[k] = o;
  }
  griddep_wait();
  for (int i = threadIdx.x; i < kh * tw; i += blockDim.x) {
    const int ky = i / tw, t = i - ky * tw;
    const int iy = iy0 + ky, ix = ix0 + t;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (iy >= 0 && iy < h && ix >= 0 && ix < w)
      v = __ldg(reinterpret_cast<const uint4*>(x + ((long long)(img * h + iy) * w + ix) * x_rs));
    tile[i] = v;
  }
  __syncthreads();
  const unsigned short* ts = reinterpret_cast<const unsigned short*>(tile);
  const uint32_t* tw32 = reinterpret_cast<const uint32_t*>(tile);
  const int cpp = kpad / EPP;  // 16-byte chunks per patch row
  const long long p0 = (long long)row * ow + ox0;
  for (int i = threadIdx.x; i < np * cpp; i += blockDim.x) {
    const int p = i / cpp, j = i - p * cpp;
    const int pb = p * stride * EPP;
    uint32_t v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if constexpr (EPP == 8) {
        const int o0 = koff[j * 8 + 2 * e], o1 = koff[j * 8 + 2 * e + 1];
        const uint32_t lo = o0 >= 0 ? ts[o0 + pb] : 0u, hi = o1 >= 0 ? ts[o1 + pb] : 0u;
        v[e] = lo | (hi << 16);
      } else {
        const int o = koff[j * 4 + e];
        v[e] = o >= 0 ? tw32[o + pb] : 0u;
      }
    }
    *reinterpret_cast<uint4*>(col + (p0 + p) * col_rs + j * EPP) = make_uint4(v[0], v[1], v[2], v[3]);
  }
}

// w (co, ci, kh, kw) fp32 -> w2 (co, kpad) fp32, k = (ky*kw + kx)*ci_n + ci; zero tail
__global__ void weight_to_cols_kernel(const float* __restrict__ w, int co_n, int ci_n, int kh, int kw,
                                      int kpad, float* __restrict__ w2) {
  griddep_launch();
  griddep_wait();
  const int K = kh * kw * ci_n;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < co_n * kpad; i += gridDim.x * blockDim.x) {
    const int co = i / kpad, k = i - co * kpad;
    float v = 0.f;
    if (k < K) {
      const int tap = k / ci_n, ci = k - tap * ci_n;
      v = w[((long long)co * ci_n + ci) * kh * kw + tap];
    }
    w2[i] = v;
  }
}

// dw2 (co, kpad) -> dw (co, ci, kh, kw): the inverse gather for the weight gradient
__global__ void cols_to_weight_kernel(const float* __restrict__ dw2, int co_n, int ci_n, int kh, int kw,
                                      int kpad, float* __restrict__ dw) {
  griddep_launch();
  griddep_wait();
  const int taps = kh * kw;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < co_n * ci_n * taps; i += gridDim.x * blockDim.x) {
    const int tap = i % taps;
    const int t = i / taps;
    const int ci = t % ci_n, co = t / ci_n;
    dw[i] = dw2[(long long)co * kpad + tap * ci_n + ci];
  }
}

// input gradient of the stem conv through its patch matrix: dx[n, iy, ix, ci] = sum over the
// (ky, kx) taps whose output (oy, ox) = ((iy + pad - ky) / s, (ix + pad - kx) / s) is an
// integer position inside the map of dcol[n, oy, ox, (ky*kw + kx)*creal + ci] (col2im as a
// deterministic gather).  One CTA per input row: for each of the <= ceil(kh/s) (ky, oy) pairs
// that reach the row, the kw*creal contiguous patch entries of every output column are staged
// in shared memory (each dcol element is read exactly once over the grid, in contiguous runs),
// then one thread per (column, channel) sums its taps in fixed order; storage channels beyond
// creal are written as zeros.
template <typename T>
__global__ void __launch_bounds__(256) col2im_kernel(const T* __restrict__ dcol, long long col_rs, int n, int h,
                                                     int w, int oh, int ow, int kh, int kw, int stride, int pad,
                                                     int creal, int cstore, T* __restrict__ dx, long long dx_rs) {
  griddep_launch();
  constexpr int EC = 16 / (int)sizeof(T);  // elements per 16-byte chunk
  extern __shared__ uint4 cbuf[];          // [pairs][ow][NC chunks]: the aligned chunks covering a run
  const int row = blockIdx.x;
  const int img = row / h, iy = row - img * h;
  const int E = kw * creal;                // one ky's run of patch entries
  const int NC = (E + 2 * EC - 2) / EC;    // chunks that can cover a run at any alignment
  int pky[8], poy[8], np = 0;
  for (int ky = 0; ky < kh && np < 8; ++ky) {
    const int ty = iy + pad - ky;
    if (ty < 0 || ty % stride) continue;
    const int oy = ty / stride;
    if (oy >= oh) continue;
    pky[np] = ky;
    poy[np] = oy;
    ++np;
  }
  griddep_wait();
  for (int p = 0; p < np; ++p) {  // 16-byte loads of the aligned chunks around each run
    const int c0 = pky[p] * E / EC;
    const T* src = dcol + ((long long)img * oh + poy[p]) * ow * col_rs + (long long)c0 * EC;
    uint4* dst = cbuf + p * ow * NC;
    for (int i = threadIdx.x; i < ow * NC; i += blockDim.x) {
      const int ox = i / NC, c = i - ox * NC;
      dst[i] = (c0 + c) * EC < col_rs ? *reinterpret_cast<const uint4*>(src + (long long)ox * col_rs + c * EC)
                                       : make_uint4(0, 0, 0, 0);
    }
  }
  __syncthreads();
  const T* sb = reinterpret_cast<const T*>(cbuf);
  T* out = dx + (long long)row * w * dx_rs;
  // one thread per input column: its <= ceil(kw/s) horizontal taps per staged (ky, oy) pair,
  // every real channel in registers, one 16-byte store of the whole stored pixel
  for (int ix = threadIdx.x; ix < w; ix += blockDim.x) {
    float acc[EC];
#pragma unroll
    for (int c = 0; c < EC; ++c) acc[c] = 0.f;
    const int kx0 = (ix + pad) % stride;
    for (int p = 0; p < np; ++p) {
      const int off0 = pky[p] * E - (pky[p] * E / EC) * EC;  // run start inside its first chunk
      const T* b = sb + (p * ow * NC) * EC + off0;
      for (int kx = kx0; kx < kw; kx += stride) {
        const int tx = ix + pad - kx;
        if (tx < 0) break;
        const int ox = tx / stride;
        if (ox >= ow) continue;
        const T* e = b + ox * NC * EC + kx * creal;
#pragma unroll
        for (int c = 0; c < EC; ++c)
          if (c < creal) acc[c] += (float)e[c];
      }
    }
    if (cstore == EC) {
      __align__(16) T v[EC];
#pragma unroll
      for (int c = 0; c < EC; ++c) v[c] = (T)acc[c];
      *reinterpret_cast<uint4*>(out + (long long)ix * dx_rs) = *reinterpret_cast<const uint4*>(v);
    } else {
      for (int c = 0; c < cstore; ++c) out[(long long)ix * dx_rs + c] = (T)(c < EC ? acc[c] : 0.f);
    }
  }
}



// ---------------------------------------------------------------------------
// strided convolutions (ResNet's stride-2 3x3s) on the window GEMM: a patch matrix per conv
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void ld16(const T* p, float (&f)[16 / sizeof(T)]) {
  const uint4 r = __ldg(reinterpret_cast<const uint4*>(p));
  if constexpr (sizeof(T) == 2) {
    f[0] = bf16lo(r.x); f[1] = bf16hi(r.x); f[2] = bf16lo(r.y); f[3] = bf16hi(r.y);
    f[4] = bf16lo(r.z); f[5] = bf16hi(r.z); f[6] = bf16lo(r.w); f[7] = bf16hi(r.w);
  } else {
    f[0] = __uint_as_float(r.x); f[1] = __uint_as_float(r.y); f[2] = __uint_as_float(r.z); f[3] = __uint_as_float(r.w);
  }
}
template <typename T>
__device__ __forceinline__ void st16(T* p, const float (&f)[16 / sizeof(T)]) {
  uint4 o;
  if constexpr (sizeof(T) == 2) {
    o.x = pack_bf16(f[0], f[1]); o.y = pack_bf16(f[2], f[3]); o.z = pack_bf16(f[4], f[5]); o.w = pack_bf16(f[6], f[7]);
  } else {
    o = make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]), __float_as_uint(f[3]));
  }
  *reinterpret_cast<uint4*>(p) = o;
}

// col[p][(ky*kw + kx)*C + c] = pro(x)[n, oy*s + ky - pad, ox*s + kx - pad, c], zero outside the map
// (padding applies after the normalize/ReLU prologue, fused.py:133-138).  pro: 0 none, 1 ReLU,
// 2 BN+ReLU as the window kernels compute it: max(fmaf(x, s, b - m*s), 0).  One thread per
// 16-byte chunk of a (pixel, tap) run.
template <typename T>
__global__ void __launch_bounds__(256) im2col_s_kernel(const T* __restrict__ x, long long x_rs, int n, int h,
                                                       int w, int C, int oh, int ow, int kh, int kw, int stride,
                                                       int pad, int pro, const float* __restrict__ cm,
                                                       const float* __restrict__ cs, const float* __restrict__ cb,
                                                       T* __restrict__ col, long long col_rs) {
  griddep_launch();
  griddep_wait();
  constexpr int EC = 16 / (int)sizeof(T);
  const int cpc = C / EC;
  const long long total = (long long)n * oh * ow * kh * kw * cpc;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(i % cpc);
    long long t = i / cpc;
    const int tap = (int)(t % (kh * kw));
    const long long p = t / (kh * kw);
    const int ox = (int)(p % ow);
    const long long q = p / ow;
    const int oy = (int)(q % oh);
    const int img = (int)(q / oh);
    const int iy = oy * stride + tap / kw - pad, ix = ox * stride + tap % kw - pad;
    const int c0 = j * EC;
    float f[EC];
    if (iy >= 0 && iy < h && ix >= 0 && ix < w) {
      ld16(x + ((long long)(img * h + iy) * w + ix) * x_rs + c0, f);
      if (pro == 2) {
#pragma unroll
        for (int e = 0; e < EC; ++e) {
          const float sc = __ldg(cs + c0 + e);
          f[e] = fmaxf(fmaf(f[e], sc, __ldg(cb + c0 + e) - __ldg(cm + c0 + e) * sc), 0.f);
        }
      } else if (pro == 1) {
#pragma unroll
        for (int e = 0; e < EC; ++e) f[e] = fmaxf(f[e], 0.f);
      }
    } else {
#pragma unroll
      for (int e = 0; e < EC; ++e) f[e] = 0.f;
    }
    st16(col + p * col_rs + tap * C + c0, f);
  }
}

// dx[n, iy, ix, c] = epi(sum over the taps that reach (iy, ix) of dcol[p(oy, ox)][(ky*kw + kx)*C + c])
// in fixed tap order; epi: 0 plain, 1 CLIP (x > 0), 2 NRC mask (fmaf(x, s, b - m*s) > 0, the
// window kernels' ReLU decision).  One thread per 16-byte chunk of an input pixel.
template <typename T>
__global__ void __launch_bounds__(256) col2im_s_kernel(const T* __restrict__ dcol, long long col_rs, int n, int h,
                                                       int w, int C, int oh, int ow, int kh, int kw, int stride,
                                                       int pad, int epi, const T* __restrict__ xm, long long xm_rs,
                                                       const float* __restrict__ cm, const float* __restrict__ cs,
                                                       const float* __restrict__ cb, T* __restrict__ dx,
                                                       long long dx_rs) {
  griddep_launch();
  griddep_wait();
  constexpr int EC = 16 / (int)sizeof(T);
  const int cpc = C / EC;
  const long long total = (long long)n * h * w * cpc;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(i % cpc);
    const long long pix = i / cpc;
    const int ix = (int)(pix % w);
    const long long q = pix / w;
    const int iy = (int)(q % h);
    const int img = (int)(q / h);
    const int c0 = j * EC;
    float acc[EC];
#pragma unroll
    for (int e = 0; e < EC; ++e) acc[e] = 0.f;
    for (int ky = (iy + pad) % stride; ky < kh; ky += stride) {
      const int ty = iy + pad - ky;
      if (ty < 0) break;
      const int oy = ty / stride;
      if (oy >= oh) continue;
      for (int kx = (ix + pad) % stride; kx < kw; kx += stride) {
        const int tx = ix + pad - kx;
        if (tx < 0) break;
        const int ox = tx / stride;
        if (ox >= ow) continue;
        float f[EC];
        ld16(dcol + (((long long)img * oh + oy) * ow + ox) * col_rs + (ky * kw + kx) * C + c0, f);
#pragma unroll
        for (int e = 0; e < EC; ++e) acc[e] += f[e];
      }
    }
    if (epi) {
      float xv[EC];
      ld16(xm + pix * xm_rs + c0, xv);
#pragma unroll
      for (int e = 0; e < EC; ++e) {
        bool keep;
        if (epi == 1) {
          keep = xv[e] > 0.f;
        } else {
          const float sc = __ldg(cs + c0 + e);
          keep = fmaf(xv[e], sc, __ldg(cb + c0 + e) - __ldg(cm + c0 + e) * sc) > 0.f;
        }
        acc[e] = keep ? acc[e] : 0.f;
      }
    }
    st16(dx + pix * dx_rs + c0, acc);
  }
}

}  // namespace stem
}  // namespace bnff

using namespace bnff;

extern "C" int bnff_im2col(int32_t dtype, bnff_view x, int32_t c_real, int32_t kh, int32_t kw,
                           int32_t stride, int32_t pad, bnff_view col, void* stream) {
  if (dtype != BNFF_BF16 && dtype != BNFF_F32) return set_error(BNFF_ERR_UNSUPPORTED, "im2col: dtype");
  const int epp = dtype == BNFF_F32 ? 4 : 8;  // one 16-byte pixel
  if (x.c != epp || c_real < 1 || c_real > epp)
    return set_error(BNFF_ERR_UNSUPPORTED, "im2col: input must be stored with %d channels (got %lld)", epp,
                     (long long)x.c);
  if (kh < 1 || kw < 1 || stride < 1 || pad < 0) return set_error(BNFF_ERR_SHAPE, "im2col: bad conv geometry");
  const long long oh = (x.h + 2 * pad - kh) / stride + 1, ow = (x.w + 2 * pad - kw) / stride + 1;
  if (col.n != x.n || col.h != oh || col.w != ow)
    return set_error(BNFF_ERR_SHAPE, "im2col: col (%lld,%lld,%lld) != (%lld,%lld,%lld)", (long long)col.n,
                     (long long)col.h, (long long)col.w, (long long)x.n, oh, ow);
  if (col.c % epp || col.c < (long long)kh * kw * c_real || col.row_stride % epp || x.row_stride % epp)
    return set_error(BNFF_ERR_SHAPE, "im2col: col channels %lld must be a multiple of %d >= %d",
                     (long long)col.c, epp, kh * kw * c_real);
  const int tp = ow <= 128 ? (int)ow : 64;
  const int tw = (tp - 1) * stride + kw;
  const size_t smem = (size_t)kh * tw * 16 + (size_t)col.c * 4;
  if (smem > 200 * 1024) return set_error(BNFF_ERR_UNSUPPORTED, "im2col: window too large");
  const long long blocks = x.n * oh * ((ow + tp - 1) / tp);
  if (blocks == 0) return BNFF_OK;
  cudaError_t e = cudaSuccess;
  if (dtype == BNFF_F32) {
    if (smem > 48 * 1024)
      e = cudaFuncSetAttribute(stem::im2col_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return set_cuda_error(e, "im2col attr");
    launch(stem::im2col_kernel<float>, dim3((unsigned)blocks), dim3(256), smem, (cudaStream_t)stream,
           (const float*)x.ptr, (long long)x.row_stride, (int)x.h, (int)x.w, (int)oh, (int)ow, kh, kw, stride,
           pad, c_real, (int)col.c, tp, (float*)col.ptr, (long long)col.row_stride);
  } else {
    if (smem > 48 * 1024)
      e = cudaFuncSetAttribute(stem::im2col_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem);
    if (e != cudaSuccess) return set_cuda_error(e, "im2col attr");
    launch(stem::im2col_kernel<__nv_bfloat16>, dim3((unsigned)blocks), dim3(256), smem, (cudaStream_t)stream,
           (const __nv_bfloat16*)x.ptr, (long long)x.row_stride, (int)x.h, (int)x.w, (int)oh, (int)ow, kh, kw,
           stride, pad, c_real, (int)col.c, tp, (__nv_bfloat16*)col.ptr, (long long)col.row_stride);
  }
  return check_launch("im2col");
}

extern "C" int bnff_weight_to_cols(const float* w, int32_t c_out, int32_t c_in, int32_t kh, int32_t kw,
                                   int32_t kpad, float* w2, void* stream) {
  if (kpad < c_in * kh * kw) return set_error(BNFF_ERR_SHAPE, "weight_to_cols: kpad too small");
  const int n = c_out * kpad;
  launch(stem::weight_to_cols_kernel, dim3((n + 255) / 256), dim3(256), 0, (cudaStream_t)stream, w, c_out,
         c_in, kh, kw, kpad, w2);
  return check_launch("weight_to_cols");
}

extern "C" int bnff_cols_to_weight(const float* dw2, int32_t c_out, int32_t c_in, int32_t kh, int32_t kw,
                                   int32_t kpad, float* dw, void* stream) {
  if (kpad < c_in * kh * kw) return set_error(BNFF_ERR_SHAPE, "cols_to_weight: kpad too small");
  const int n = c_out * c_in * kh * kw;
  launch(stem::cols_to_weight_kernel, dim3((n + 255) / 256), dim3(256), 0, (cudaStream_t)stream, dw2, c_out,
         c_in, kh, kw, kpad, dw);
  return check_launch("cols_to_weight");
}

extern "C" int bnff_col2im(int32_t dtype, bnff_view dcol, int32_t c_real, int32_t kh, int32_t kw, int32_t stride,
                           int32_t pad, bnff_view dx, void* stream) {
  if (dtype != BNFF_BF16 && dtype != BNFF_F32) return set_error(BNFF_ERR_UNSUPPORTED, "col2im: dtype");
  if (kh < 1 || kw < 1 || stride < 1 || pad < 0 || c_real < 1 || c_real > dx.c)
    return set_error(BNFF_ERR_SHAPE, "col2im: bad conv geometry");
  const long long oh = (dx.h + 2 * pad - kh) / stride + 1, ow = (dx.w + 2 * pad - kw) / stride + 1;
  if (dcol.n != dx.n || dcol.h != oh || dcol.w != ow || dcol.c < (long long)kh * kw * c_real)
    return set_error(BNFF_ERR_SHAPE, "col2im: dcol (%lld,%lld,%lld,%lld) vs dx", (long long)dcol.n,
                     (long long)dcol.h, (long long)dcol.w, (long long)dcol.c);
  const long long rows = dx.n * dx.h;
  if (rows == 0) return BNFF_OK;
  const int np_max = (kh + stride - 1) / stride;
  const int ec = dtype == BNFF_F32 ? 4 : 8;
  const int nc = (kw * c_real + 2 * ec - 2) / ec;
  if (dcol.row_stride % ec) return set_error(BNFF_ERR_UNSUPPORTED, "col2im: dcol rows not 16-byte aligned");
  if (c_real > ec || dx.row_stride % ec)
    return set_error(BNFF_ERR_UNSUPPORTED, "col2im: the image must be stored as one 16-byte pixel");
  const size_t smem = (size_t)np_max * ow * nc * 16;
  if (np_max > 8 || smem > 200 * 1024) return set_error(BNFF_ERR_UNSUPPORTED, "col2im: window too large");
  cudaError_t e = cudaSuccess;
  if (dtype == BNFF_F32) {
    if (smem > 48 * 1024)
      e = cudaFuncSetAttribute(stem::col2im_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return set_cuda_error(e, "col2im attr");
    launch(stem::col2im_kernel<float>, dim3((unsigned)rows), dim3(256), smem, (cudaStream_t)stream,
           (const float*)dcol.ptr, (long long)dcol.row_stride, (int)dx.n, (int)dx.h, (int)dx.w, (int)oh, (int)ow, kh,
           kw, stride, pad, c_real, (int)dx.c, (float*)dx.ptr, (long long)dx.row_stride);
  } else {
    if (smem > 48 * 1024)
      e = cudaFuncSetAttribute(stem::col2im_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem);
    if (e != cudaSuccess) return set_cuda_error(e, "col2im attr");
    launch(stem::col2im_kernel<__nv_bfloat16>, dim3((unsigned)rows), dim3(256), smem, (cudaStream_t)stream,
           (const __nv_bfloat16*)dcol.ptr, (long long)dcol.row_stride, (int)dx.n, (int)dx.h, (int)dx.w, (int)oh,
           (int)ow, kh, kw, stride, pad, c_real, (int)dx.c, (__nv_bfloat16*)dx.ptr, (long long)dx.row_stride);
  }
  return check_launch("col2im");
}

static inline int grid256(long long work) {
  long long b = (work + 255) / 256;
  return (int)(b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b));
}

extern "C" int bnff_im2col_s(int32_t dtype, bnff_view x, int32_t kh, int32_t kw, int32_t stride, int32_t pad,
                             int32_t pro, bnff_coef pcoef, bnff_view col, void* stream) {
  if (dtype != BNFF_BF16 && dtype != BNFF_F32) return set_error(BNFF_ERR_UNSUPPORTED, "im2col_s: dtype");
  const int ec = dtype == BNFF_F32 ? 4 : 8;
  if (x.c % ec || x.row_stride % ec || col.row_stride % ec)
    return set_error(BNFF_ERR_UNSUPPORTED, "im2col_s: channels must fill 16-byte chunks");
  const long long oh = (x.h + 2 * pad - kh) / stride + 1, ow = (x.w + 2 * pad - kw) / stride + 1;
  if (col.n != x.n || col.h != oh || col.w != ow || col.c < (long long)kh * kw * x.c)
    return set_error(BNFF_ERR_SHAPE, "im2col_s: col (%lld,%lld,%lld,%lld)", (long long)col.n, (long long)col.h,
                     (long long)col.w, (long long)col.c);
  if (pro == BNFF_PRO_BN_RELU && (!pcoef.a || !pcoef.b || !pcoef.c))
    return set_error(BNFF_ERR_STATE, "im2col_s: missing normalisation tables");
  const int p = pro == BNFF_PRO_BN_RELU ? 2 : (pro == BNFF_PRO_RELU ? 1 : 0);
  const long long work = x.n * oh * ow * kh * kw * (x.c / ec);
  if (dtype == BNFF_F32)
    launch(stem::im2col_s_kernel<float>, dim3(grid256(work)), dim3(256), 0, (cudaStream_t)stream, (const float*)x.ptr,
           (long long)x.row_stride, (int)x.n, (int)x.h, (int)x.w, (int)x.c, (int)oh, (int)ow, kh, kw, stride, pad, p,
           pcoef.a, pcoef.b, pcoef.c, (float*)col.ptr, (long long)col.row_stride);
  else
    launch(stem::im2col_s_kernel<__nv_bfloat16>, dim3(grid256(work)), dim3(256), 0, (cudaStream_t)stream,
           (const __nv_bfloat16*)x.ptr, (long long)x.row_stride, (int)x.n, (int)x.h, (int)x.w, (int)x.c, (int)oh,
           (int)ow, kh, kw, stride, pad, p, pcoef.a, pcoef.b, pcoef.c, (__nv_bfloat16*)col.ptr,
           (long long)col.row_stride);
  return check_launch("im2col_s");
}

extern "C" int bnff_col2im_s(int32_t dtype, bnff_view dcol, int32_t kh, int32_t kw, int32_t stride, int32_t pad,
                             int32_t epi, bnff_view x, bnff_coef ecoef, bnff_view dx, void* stream) {
  if (dtype != BNFF_BF16 && dtype != BNFF_F32) return set_error(BNFF_ERR_UNSUPPORTED, "col2im_s: dtype");
  const int ec = dtype == BNFF_F32 ? 4 : 8;
  if (dx.c % ec || dx.row_stride % ec || dcol.row_stride % ec)
    return set_error(BNFF_ERR_UNSUPPORTED, "col2im_s: channels must fill 16-byte chunks");
  const long long oh = (dx.h + 2 * pad - kh) / stride + 1, ow = (dx.w + 2 * pad - kw) / stride + 1;
  if (dcol.n != dx.n || dcol.h != oh || dcol.w != ow || dcol.c < (long long)kh * kw * dx.c)
    return set_error(BNFF_ERR_SHAPE, "col2im_s: dcol vs dx");
  const int e = epi == BNFF_DG_NRC ? 2 : (epi == BNFF_DG_CLIP ? 1 : 0);
  if (e && (!x.ptr || x.n != dx.n || x.h != dx.h || x.w != dx.w || x.c != dx.c))
    return set_error(BNFF_ERR_SHAPE, "col2im_s: mask input");
  if (e == 2 && (!ecoef.a || !ecoef.b || !ecoef.c)) return set_error(BNFF_ERR_STATE, "col2im_s: missing tables");
  if (epi != BNFF_DG_PLAIN && epi != BNFF_DG_CLIP && epi != BNFF_DG_NRC)
    return set_error(BNFF_ERR_UNSUPPORTED, "col2im_s: epilogue %d", epi);
  const long long work = dx.n * dx.h * dx.w * (dx.c / ec);
  if (dtype == BNFF_F32)
    launch(stem::col2im_s_kernel<float>, dim3(grid256(work)), dim3(256), 0, (cudaStream_t)stream,
           (const float*)dcol.ptr, (long long)dcol.row_stride, (int)dx.n, (int)dx.h, (int)dx.w, (int)dx.c, (int)oh,
           (int)ow, kh, kw, stride, pad, e, (const float*)x.ptr, (long long)x.row_stride, ecoef.a, ecoef.b, ecoef.c,
           (float*)dx.ptr, (long long)dx.row_stride);
  else
    launch(stem::col2im_s_kernel<__nv_bfloat16>, dim3(grid256(work)), dim3(256), 0, (cudaStream_t)stream,
           (const __nv_bfloat16*)dcol.ptr, (long long)dcol.row_stride, (int)dx.n, (int)dx.h, (int)dx.w, (int)dx.c,
           (int)oh, (int)ow, kh, kw, stride, pad, e, (const __nv_bfloat16*)x.ptr, (long long)x.row_stride, ecoef.a,
           ecoef.b, ecoef.c, (__nv_bfloat16*)dx.ptr, (long long)dx.row_stride);
  return check_launch("col2im_s");
}
