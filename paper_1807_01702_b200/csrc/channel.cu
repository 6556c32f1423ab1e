// channel.cu -- HBM-bound kernels of the restructured-BN path (sm_100a).
//
// Everything here streams NHWC views with 128-bit loads/stores (8 bf16 / 4 f32
// per access, consecutive threads on consecutive channel chunks of a pixel) and
// reduces per-channel quantities deterministically: per-tile partials written
// to a [tiles][2][C] buffer, then combined in a fixed order in float64.
#include <cstdint>
#include <cstdio>
#include <type_traits>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "sm100.cuh"
#include "common.cuh"

namespace bnff {

static thread_local char g_err[512] = "";
char* last_error_buf() { return g_err; }

// ---------------------------------------------------------------------------
// vector access helpers
// ---------------------------------------------------------------------------
template <typename T> struct VecIO;
template <> struct VecIO<__nv_bfloat16> {
  static constexpr int V = 8;
  __device__ static __forceinline__ void load(const void* base, long long off, float (&f)[8]) {
    const uint4 r = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(base) + off));
    f[0] = bf16lo(r.x); f[1] = bf16hi(r.x); f[2] = bf16lo(r.y); f[3] = bf16hi(r.y);
    f[4] = bf16lo(r.z); f[5] = bf16hi(r.z); f[6] = bf16lo(r.w); f[7] = bf16hi(r.w);
  }
  __device__ static __forceinline__ void store(void* base, long long off, const float (&f)[8]) {
    uint4 o;
    o.x = pack_bf16(f[0], f[1]); o.y = pack_bf16(f[2], f[3]);
    o.z = pack_bf16(f[4], f[5]); o.w = pack_bf16(f[6], f[7]);
    *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(base) + off) = o;
  }
  __device__ static __forceinline__ float round(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }
};
template <> struct VecIO<float> {
  static constexpr int V = 4;
  __device__ static __forceinline__ void load(const void* base, long long off, float (&f)[4]) {
    const float4 r = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(base) + off));
    f[0] = r.x; f[1] = r.y; f[2] = r.z; f[3] = r.w;
  }
  __device__ static __forceinline__ void store(void* base, long long off, const float (&f)[4]) {
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(base) + off) = make_float4(f[0], f[1], f[2], f[3]);
  }
  __device__ static __forceinline__ float round(float v) { return v; }
};

struct View {
  const void* p;
  long long rs;
};

__device__ __forceinline__ void unpack8f(const uint4& r, float* f) {
  f[0] = bf16lo(r.x); f[1] = bf16hi(r.x); f[2] = bf16lo(r.y); f[3] = bf16hi(r.y);
  f[4] = bf16lo(r.z); f[5] = bf16hi(r.z); f[6] = bf16lo(r.w); f[7] = bf16hi(r.w);
}

__device__ __forceinline__ float bn_dx_elem(float dt, float x, int c, const bnff_coef& cf) {
  const float xh = __fmul_rn(__fsub_rn(x, __ldg(cf.a + c)), __ldg(cf.b + c));
  const float t = __fsub_rn(__fsub_rn(dt, __ldg(cf.c + c)), __fmul_rn(xh, __ldg(cf.d + c)));
  return __fmul_rn(__ldg(cf.e + c), t);
}

// partials [tiles][2][C] -> float64 totals, one launch: block = 32 channels x 8 row
// groups; every (row group, channel) sum is a fixed-order loop, then a fixed-order
// combine of the 8 groups (bitwise deterministic)
__device__ __forceinline__ void reduce_two(const double* __restrict__ part, int tiles, int C, int c,
                                           double& o1, double& o2) {
  // block = 32 channels x 16 row groups; loads of one thread are independent (unrolled)
  __shared__ double sh[2][16][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  double a = 0.0, b = 0.0;
  if (c < C) {
    double va[12], vb[12];
#pragma unroll
    for (int u = 0; u < 12; ++u) {
      const int t = ty + 16 * u;
      va[u] = t < tiles ? part[((long long)t * 2 + 0) * C + c] : 0.0;
      vb[u] = t < tiles ? part[((long long)t * 2 + 1) * C + c] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 12; ++u) { a += (double)va[u]; b += (double)vb[u]; }
    for (int t = ty + 16 * 12; t < tiles; t += 16) {
      a += (double)part[((long long)t * 2 + 0) * C + c];
      b += (double)part[((long long)t * 2 + 1) * C + c];
    }
  }
  sh[0][ty][tx] = a;
  sh[1][ty][tx] = b;
  __syncthreads();
  o1 = o2 = 0.0;
  if (ty == 0) {
    for (int k = 0; k < 16; ++k) { o1 += sh[0][k][tx]; o2 += sh[1][k][tx]; }
  }
}

__global__ void __launch_bounds__(512) stats_finalize_kernel(const double* __restrict__ part, int tiles, int C,
                                                             long long count, double* sum, double* sumsq,
                                                             double* mean, double* var) {
  griddep_launch();
  griddep_wait();
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  double s1, s2;
  reduce_two(part, tiles, C, c, s1, s2);
  if ((threadIdx.x >> 5) == 0 && c < C) {
    sum[c] = s1;
    sumsq[c] = s2;
    if (mean && var) {  // ChannelStats.from_sums (ops.py:109-113): population var, clamped
      const double m = s1 / (double)count;
      mean[c] = m;
      const double v = s2 / (double)count - m * m;
      var[c] = v > 0.0 ? v : 0.0;
    }
  }
}

// stats_finalize of one freshly produced piece (channels [c_off, c_off + c_new) of a block)
// fused with the next consumer's bn_coeffs over all c_total channels (ICF: concat_stats +
// ChannelStats.from_sums + inv_std, ops.py:109-143; one launch instead of two)
__global__ void __launch_bounds__(512) finalize_coeffs_kernel(
    const double* __restrict__ part, int tiles, int c_new, long long count, double* sum, double* sumsq,
    double* mean, double* var, int c_off, int c_total, const double* mean_all, const double* var_all,
    const float* gamma, const float* beta, float eps, float* mean32, float* scale32, float* beta32,
    float* inv32) {
  griddep_launch();
  griddep_wait();
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  const int cl = (c >= c_off && c < c_off + c_new) ? c - c_off : c_new;  // piece column or none
  double s1, s2;
  reduce_two(part, tiles, c_new, cl, s1, s2);
  if ((threadIdx.x >> 5) == 0 && c < c_total) {
    double m, v;
    if (cl < c_new) {  // ChannelStats.from_sums (ops.py:109-113): population var, clamped
      sum[cl] = s1;
      sumsq[cl] = s2;
      m = s1 / (double)count;
      v = s2 / (double)count - m * m;
      v = v > 0.0 ? v : 0.0;
      mean[cl] = m;
      var[cl] = v;
    } else {
      m = mean_all[c];
      v = var_all[c];
    }
    const double vv = v > 0.0 ? v : 0.0;
    const double inv = 1.0 / sqrt(vv + (double)eps);
    mean32[c] = (float)m;
    if (scale32) scale32[c] = (float)((double)gamma[c] * inv);
    if (beta32) beta32[c] = beta[c];
    if (inv32) inv32[c] = (float)inv;
  }
}

__global__ void __launch_bounds__(512) dx_coeffs_fused_kernel(
    const double* __restrict__ part, int tiles, int C, long long count, const double* mean,
    const double* var, const float* gamma, float eps, double* dgamma64, double* dbeta64, float* k1,
    float* k2, float* g, float* mean32, float* inv32, float* dgamma32, float* dbeta32, float* acc_a,
    float* acc_b, int acc_init) {
  griddep_launch();
  griddep_wait();
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  double dbeta, dgamma;
  reduce_two(part, tiles, C, c, dbeta, dgamma);
  if ((threadIdx.x >> 5) == 0 && c < C) {
    dbeta64[c] = dbeta;
    dgamma64[c] = dgamma;
    const double v = var[c] > 0.0 ? var[c] : 0.0;
    const double inv = 1.0 / sqrt(v + (double)eps);
    k1[c] = (float)(dbeta / (double)count);
    k2[c] = (float)(dgamma / (double)count);
    g[c] = (float)((double)gamma[c] * inv);
    mean32[c] = (float)mean[c];
    inv32[c] = (float)inv;
    if (dgamma32) dgamma32[c] = (float)dgamma;
    if (dbeta32) dbeta32[c] = (float)dbeta;
    if (acc_a) {  // ICF block-gradient fold: per-channel remainder g*(k1 + xhat*k2)
      const float gf = (float)((double)gamma[c] * inv);
      const float a = gf * (float)(dbeta / (double)count), b = gf * (float)(dgamma / (double)count);
      acc_a[c] = acc_init ? a : acc_a[c] + a;
      acc_b[c] = acc_init ? b : acc_b[c] + b;
    }
  }
}

__global__ void stats_from_sums_kernel(int C, long long count, const double* sum, const double* sumsq,
                                       double* mean, double* var) {
  griddep_launch();
  griddep_wait();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const double m = sum[c] / (double)count;
  mean[c] = m;
  const double v = sumsq[c] / (double)count - m * m;
  var[c] = v > 0.0 ? v : 0.0;
}

// partials -> float64 totals of one slot (kept for the centred-variance path)
__global__ void reduce_parts_kernel(const double* __restrict__ part, int tiles, int C, int slot,
                                    double* __restrict__ out) {
  griddep_launch();
  griddep_wait();
  __shared__ double sh[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + tx;
  double acc = 0.0;
  if (c < C)
    for (int t = ty; t < tiles; t += 8) acc += (double)part[((long long)t * 2 + slot) * C + c];
  sh[ty][tx] = acc;
  __syncthreads();
  if (ty == 0 && c < C) {
    double s = 0.0;
    for (int k = 0; k < 8; ++k) s += sh[k][tx];
    out[c] = s;
  }
}

__global__ void bn_coeffs_kernel(int C, const double* mean, const double* var, const float* gamma,
                                 const float* beta, float eps, float* mean32, float* scale32,
                                 float* beta32, float* inv32) {
  griddep_launch();
  griddep_wait();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const double v = var[c] > 0.0 ? var[c] : 0.0;
  const double inv = 1.0 / sqrt(v + (double)eps);
  mean32[c] = (float)mean[c];
  if (scale32) scale32[c] = (float)((double)gamma[c] * inv);
  if (beta32) beta32[c] = beta[c];
  if (inv32) inv32[c] = (float)inv;
}

__global__ void dx_coeffs_kernel(int C, long long count, const double* dsum, const double* dsum2,
                                 const double* mean, const double* var, const float* gamma,
                                 float eps, float* k1, float* k2, float* g, float* mean32,
                                 float* inv32, float* dgamma32, float* dbeta32) {
  griddep_launch();
  griddep_wait();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const double v = var[c] > 0.0 ? var[c] : 0.0;
  const double inv = 1.0 / sqrt(v + (double)eps);
  const double dbeta = dsum[c], dgamma = dsum2[c];
  k1[c] = (float)(dbeta / (double)count);
  k2[c] = (float)(dgamma / (double)count);
  g[c] = (float)((double)gamma[c] * inv);
  mean32[c] = (float)mean[c];
  inv32[c] = (float)inv;
  if (dgamma32) dgamma32[c] = (float)dgamma;
  if (dbeta32) dbeta32[c] = (float)dbeta;
}

// ---------------------------------------------------------------------------
// elementwise families (grid-stride over pixels x chunks)
// ---------------------------------------------------------------------------
// Row x chunk mapping shared by the streaming kernels: a thread owns one 16-byte
// channel chunk j (fixed, so its per-channel coefficients live in registers) and
// walks pixel rows; rows are split across the block (tpr per iteration) and grid.
struct RowChunk {
  int cpr, tpr, j, lane;
  bool active;
  __device__ RowChunk(int C, int V) {
    cpr = C / V;
    tpr = cpr >= (int)blockDim.x ? 1 : (int)blockDim.x / cpr;
    j = (int)threadIdx.x % cpr;
    lane = (int)threadIdx.x / cpr;
    active = lane < tpr;
  }
};
__host__ inline int rowchunk_grid(long long pixels, int C, int V) {
  const int cpr = C / V;
  const int tpr = cpr >= 256 ? 1 : 256 / cpr;
  long long b = (pixels + tpr - 1) / tpr;
  const long long cap = 148 * 8;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

template <typename T>
__global__ void __launch_bounds__(256) bn_apply_kernel(View x, View y, long long pixels, int C,
                                                       bnff_coef cf, int relu) {
  griddep_launch();
  griddep_wait();
  constexpr int V = VecIO<T>::V;
  const RowChunk rc(C, V);
  if (!rc.active) return;
  for (int jj = rc.j; jj < rc.cpr; jj += (int)blockDim.x) {
    const int c0 = jj * V;
    float a[V], b[V], c[V];
#pragma unroll
    for (int k = 0; k < V; ++k) { a[k] = __ldg(cf.a + c0 + k); b[k] = __ldg(cf.b + c0 + k); c[k] = __ldg(cf.c + c0 + k); }
    for (long long r = (long long)blockIdx.x * rc.tpr + rc.lane; r < pixels; r += (long long)gridDim.x * rc.tpr) {
      float f[V];
      VecIO<T>::load(x.p, r * x.rs + c0, f);
#pragma unroll
      for (int k = 0; k < V; ++k) {
        float t = __fadd_rn(__fmul_rn(__fsub_rn(f[k], a[k]), b[k]), c[k]);  // bn_fwd op order
        f[k] = relu ? fmaxf(t, 0.f) : t;
      }
      VecIO<T>::store(const_cast<void*>(y.p), r * y.rs + c0, f);
    }
    if (rc.cpr < (int)blockDim.x) break;
  }
}

struct TermDev {
  View g, x;
  int deferred;
  bnff_coef cf;
};

// deferred BN dx coefficients of one chunk.  fp32 storage: the reference's exact op
// order g*((dt - k1) - xhat*k2), xhat = (x-mean)*inv.  bf16 storage: the same affine
// map refactored as g*dt + B*x + C (two FMAs; rounding far below bf16 resolution).
template <typename T, int V>
struct DxCoef {
  float m[V], inv[V], k1[V], k2[V], g[V];
  __device__ void load(const bnff_coef& cf, int c0) {
#pragma unroll
    for (int k = 0; k < V; ++k) {
      m[k] = __ldg(cf.a + c0 + k); inv[k] = __ldg(cf.b + c0 + k); k1[k] = __ldg(cf.c + c0 + k);
      k2[k] = __ldg(cf.d + c0 + k); g[k] = __ldg(cf.e + c0 + k);
    }
    if constexpr (sizeof(T) == 2) {
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const float B = -g[k] * k2[k] * inv[k];
        const float Cc = g[k] * (k2[k] * inv[k] * m[k] - k1[k]);
        k1[k] = B;
        k2[k] = Cc;
      }
    }
  }
  __device__ __forceinline__ float apply(float dt, float x, int k) const {
    if constexpr (sizeof(T) == 2) {
      return fmaf(dt, g[k], fmaf(x, k1[k], k2[k]));
    } else {
      const float xh = __fmul_rn(__fsub_rn(x, m[k]), inv[k]);
      const float t = __fsub_rn(__fsub_rn(dt, k1[k]), __fmul_rn(xh, k2[k]));
      return __fmul_rn(g[k], t);
    }
  }
};

template <typename T>
__global__ void __launch_bounds__(256) grad_sum_kernel(View out, long long pixels, int C, int accumulate,
                                                       TermDev t0, TermDev t1, int nterms) {
  griddep_launch();
  griddep_wait();
  constexpr int V = VecIO<T>::V;
  const RowChunk rc(C, V);
  if (!rc.active) return;
  for (int jj = rc.j; jj < rc.cpr; jj += (int)blockDim.x) {
    const int c0 = jj * V;
    DxCoef<T, V> d0, d1;
    if (t0.deferred) d0.load(t0.cf, c0);
    if (nterms > 1 && t1.deferred) d1.load(t1.cf, c0);
    for (long long r = (long long)blockIdx.x * rc.tpr + rc.lane; r < pixels; r += (long long)gridDim.x * rc.tpr) {
      float acc[V], v[V], xv[V];
      VecIO<T>::load(t0.g.p, r * t0.g.rs + c0, v);
      if (t0.deferred) VecIO<T>::load(t0.x.p, r * t0.x.rs + c0, xv);
#pragma unroll
      for (int k = 0; k < V; ++k) acc[k] = t0.deferred ? d0.apply(v[k], xv[k], k) : v[k];
      if (nterms > 1) {
        VecIO<T>::load(t1.g.p, r * t1.g.rs + c0, v);
        if (t1.deferred) VecIO<T>::load(t1.x.p, r * t1.x.rs + c0, xv);
#pragma unroll
        for (int k = 0; k < V; ++k) {
          // each resolved term is rounded to storage precision (the reference materialises it)
          const float a = VecIO<T>::round(acc[k]);
          const float b = VecIO<T>::round(t1.deferred ? d1.apply(v[k], xv[k], k) : v[k]);
          acc[k] = a + b;
        }
      }
      if (accumulate) {
        VecIO<T>::load(out.p, r * out.rs + c0, v);
#pragma unroll
        for (int k = 0; k < V; ++k) acc[k] = v[k] + VecIO<T>::round(acc[k]);
      }
      VecIO<T>::store(const_cast<void*>(out.p), r * out.rs + c0, acc);
    }
    if (rc.cpr < (int)blockDim.x) break;
  }
}

// ---------------------------------------------------------------------------
// K5: channel sums -> partials [tiles][2][C]
// ---------------------------------------------------------------------------
constexpr int kSumThreads = 256;
constexpr int kMaxTiles = 1184;  // 8 x 148

__host__ __device__ inline int sum_tiles(long long pixels) {
  long long t = (pixels + 31) / 32;
  return (int)(t < kMaxTiles ? (t < 1 ? 1 : t) : kMaxTiles);
}

// 16-byte channel columns per CTA of channel_sums: all of them, unless the map is so small
// that the row tiles alone leave SMs idle -- then groups of >= 32 columns (>= 4 x 148 CTAs)
inline int sum_col_width(int dtype, int c, int tiles) {
  const int cpr = c / (dtype == BNFF_F32 ? 4 : 8);
  const int want = (4 * 148 + tiles - 1) / tiles;
  int groups = cpr / 32;
  if (groups > want) groups = want;
  if (groups < 1) groups = 1;
  return (cpr + groups - 1) / groups;
}

// mode 0: (x, x^2); mode 1: (dy, dy*xhat) xhat=(x-a)*b; mode 2: (dy', 0) with dy'
// = dy or BN_DX(dy, x) when coef.e != null; mode 3: (centred^2, 0) with a = mean (double).
// Grid: x = row tiles (the partial rows), y = channel groups of `cw` 16-byte columns (small
// maps with many channels get more CTAs).  Four rows per thread in flight (two for MODE 2), then a
// fixed-order pairwise tree over the threads sharing a column (bitwise deterministic).
template <typename T, int MODE>
__global__ void __launch_bounds__(kSumThreads, 3) channel_sums_kernel(View xv, View dyv, long long pixels, int C,
                                                                      int cw, bnff_coef cf, const double* mean64,
                                                                      double* part) {
  constexpr int mode = MODE;
  griddep_launch();
  griddep_wait();
  constexpr int V = VecIO<T>::V;
  // fp32 data accumulates in float64 (the reference's bn_stats_onepass sums in f64,
  // ops.py:231-237); bf16 values (8-bit significands) accumulate in fp32
  using Acc = typename std::conditional<sizeof(T) == 4, double, float>::type;
  __shared__ Acc sh[2][V][kSumThreads];
  const int cpr = C / V;
  const int tiles = gridDim.x;
  const long long rows_per_tile = (pixels + tiles - 1) / tiles;
  const long long r_begin = blockIdx.x * rows_per_tile;
  const long long r_end = min(pixels, r_begin + rows_per_tile);
  const int g_lo = blockIdx.y * cw, g_hi = min(cpr, g_lo + cw);
  const bool two = mode == 1 || (mode == 2 && cf.e != nullptr);  // a second operand (x) per row
  const View pv = (mode == 0 || mode == 3) ? xv : dyv;
  for (int cbase = g_lo; cbase < g_hi; cbase += kSumThreads) {
    const int ccount = min(kSumThreads, g_hi - cbase);
    const int rows_per_iter = kSumThreads / ccount;
    const int tcol = threadIdx.x % ccount, trow = threadIdx.x / ccount;
    const bool active = trow < rows_per_iter;
    const int c0 = (cbase + tcol) * V;
    Acc s1[V], s2[V];
#pragma unroll
    for (int i = 0; i < V; ++i) s1[i] = s2[i] = Acc(0);
    if (active) {
      // per-channel coefficients hoisted out of the row loop
      float ca[V], cb[V];
      double m64[V];
      DxCoef<T, V> dxc;
      if (mode == 1) {
#pragma unroll
        for (int i = 0; i < V; ++i) { ca[i] = __ldg(cf.a + c0 + i); cb[i] = __ldg(cf.b + c0 + i); }
      } else if (mode == 2 && two) {
        dxc.load(cf, c0);
      } else if (mode == 3) {
#pragma unroll
        for (int i = 0; i < V; ++i) m64[i] = mean64[c0 + i];
      }
      auto acc = [&](const float (&v)[V], const float (&x)[V]) {
#pragma unroll
        for (int i = 0; i < V; ++i) {
          if (mode == 0) {
            s1[i] += (Acc)v[i];
            s2[i] += (Acc)v[i] * (Acc)v[i];
          } else if (mode == 1) {
            const float xh = __fmul_rn(__fsub_rn(x[i], ca[i]), cb[i]);
            s1[i] += (Acc)v[i];
            s2[i] += (Acc)v[i] * (Acc)xh;
          } else if (mode == 2) {
            s1[i] += (Acc)(two ? dxc.apply(v[i], x[i], i) : v[i]);
          } else {
            const Acc d = (Acc)((double)v[i] - m64[i]);
            s1[i] += d * d;
          }
        }
      };
      // rows in flight per thread (the deferred-dx dbias keeps five coefficient vectors live)
      constexpr int U = MODE == 2 ? 2 : 4;
      long long r = r_begin + trow;
      for (; r + (U - 1) * rows_per_iter < r_end; r += U * rows_per_iter) {
        float v[U][V], x[U][V];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          VecIO<T>::load(pv.p, (r + u * rows_per_iter) * pv.rs + c0, v[u]);
          if (two) VecIO<T>::load(xv.p, (r + u * rows_per_iter) * xv.rs + c0, x[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc(v[u], x[u]);
      }
      for (; r < r_end; r += rows_per_iter) {
        float v[V], x[V];
        VecIO<T>::load(pv.p, r * pv.rs + c0, v);
        if (two) VecIO<T>::load(xv.p, r * xv.rs + c0, x);
        acc(v, x);
      }
    }
#pragma unroll
    for (int i = 0; i < V; ++i) {
      sh[0][i][threadIdx.x] = s1[i];
      sh[1][i][threadIdx.x] = s2[i];
    }
    __syncthreads();
    // fixed-order pairwise tree over the rows_per_iter threads of each column
    for (int n = rows_per_iter; n > 1;) {
      const int h = (n + 1) >> 1;
      if (active && trow < n - h) {
        const int o = threadIdx.x + h * ccount;
#pragma unroll
        for (int i = 0; i < V; ++i) {
          sh[0][i][threadIdx.x] += sh[0][i][o];
          sh[1][i][threadIdx.x] += sh[1][i][o];
        }
      }
      n = h;
      __syncthreads();
    }
    if (threadIdx.x < ccount) {
      const int cc = (cbase + threadIdx.x) * V;
#pragma unroll
      for (int i = 0; i < V; ++i) {
        part[((long long)blockIdx.x * 2 + 0) * C + cc + i] = sh[0][i][threadIdx.x];
        part[((long long)blockIdx.x * 2 + 1) * C + cc + i] = sh[1][i][threadIdx.x];
      }
    }
    __syncthreads();
  }
}

// bf16 fast path of grad_sum: raw 16-byte loads of U rows in flight before any math,
// deferred terms in the two-FMA form (DxCoef<bf16>)
template <int U, int NT>
__global__ void __launch_bounds__(256, 2) grad_sum_bf16_kernel(View out, long long pixels, int C, int accumulate,
                                                            TermDev t0, TermDev t1, int nterms_) {
  griddep_launch();
  griddep_wait();
  constexpr int nterms = NT;
  (void)nterms_;
  constexpr int V = 8;
  const RowChunk rc(C, V);
  if (!rc.active) return;
  for (int jj = rc.j; jj < rc.cpr; jj += (int)blockDim.x) {
    const int c0 = jj * V;
    DxCoef<__nv_bfloat16, V> d0, d1;
    if (t0.deferred) d0.load(t0.cf, c0);
    if (nterms > 1 && t1.deferred) d1.load(t1.cf, c0);
    const long long step = (long long)gridDim.x * rc.tpr;
    for (long long r = (long long)blockIdx.x * rc.tpr + rc.lane; r < pixels; r += U * step) {
      uint4 g0[U], x0[U], g1[U], x1[U], ov[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long rr = r + u * step;
        if (rr < pixels) {
          g0[u] = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(t0.g.p) + rr * t0.g.rs + c0));
          if (t0.deferred)
            x0[u] = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(t0.x.p) + rr * t0.x.rs + c0));
          if (nterms > 1) {
            g1[u] = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(t1.g.p) + rr * t1.g.rs + c0));
            if (t1.deferred)
              x1[u] = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(t1.x.p) + rr * t1.x.rs + c0));
          }
          if (accumulate)
            ov[u] = *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(out.p) + rr * out.rs + c0);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long rr = r + u * step;
        if (rr >= pixels) break;
        float a[V], v[V], xv[V];
        unpack8f(g0[u], v);
        if (t0.deferred) {
          unpack8f(x0[u], xv);
#pragma unroll
          for (int k = 0; k < V; ++k) a[k] = d0.apply(v[k], xv[k], k);
        } else {
#pragma unroll
          for (int k = 0; k < V; ++k) a[k] = v[k];
        }
        if (nterms > 1) {
          unpack8f(g1[u], v);
          if (t1.deferred) {
            unpack8f(x1[u], xv);
#pragma unroll
            for (int k = 0; k < V; ++k) v[k] = d1.apply(v[k], xv[k], k);
          }
#pragma unroll
          for (int k = 0; k < V; ++k) a[k] = VecIO<__nv_bfloat16>::round(a[k]) + VecIO<__nv_bfloat16>::round(v[k]);
        }
        if (accumulate) {
          unpack8f(ov[u], v);
#pragma unroll
          for (int k = 0; k < V; ++k) a[k] = v[k] + VecIO<__nv_bfloat16>::round(a[k]);
        }
        VecIO<__nv_bfloat16>::store(const_cast<void*>(out.p), rr * out.rs + c0, a);
      }
    }
    if (rc.cpr < (int)blockDim.x) break;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) relu_kernel(View x, View dy, View out, long long pixels, int C, int bwd) {
  griddep_launch();
  griddep_wait();
  constexpr int V = VecIO<T>::V;
  const RowChunk rc(C, V);
  if (!rc.active) return;
  for (int jj = rc.j; jj < rc.cpr; jj += (int)blockDim.x) {
    const int c0 = jj * V;
    for (long long r = (long long)blockIdx.x * rc.tpr + rc.lane; r < pixels; r += (long long)gridDim.x * rc.tpr) {
      float f[V], g[V];
      VecIO<T>::load(x.p, r * x.rs + c0, f);
      if (bwd) {
        VecIO<T>::load(dy.p, r * dy.rs + c0, g);
#pragma unroll
        for (int k = 0; k < V; ++k) f[k] = f[k] > 0.f ? g[k] : 0.f;
      } else {
#pragma unroll
        for (int k = 0; k < V; ++k) f[k] = fmaxf(f[k], 0.f);
      }
      VecIO<T>::store(const_cast<void*>(out.p), r * out.rs + c0, f);
    }
    if (rc.cpr < (int)blockDim.x) break;
  }
}

// avgpool forward with optional statistics of the written output (same tiling
// as channel_sums: tile = range of output pixels)
template <typename T>
__global__ void avgpool_fwd_kernel(View x, View y, int n, int h, int w, int oh, int ow, int C, int k,
                                   double* part) {
  griddep_launch();
  griddep_wait();
  constexpr int V = VecIO<T>::V;
  using Acc = typename std::conditional<sizeof(T) == 4, double, float>::type;  // f64 for fp32 data
  __shared__ Acc sh[2][kSumThreads][V];
  const long long pixels = (long long)n * oh * ow;
  const int cpr = C / V;
  const int tiles = gridDim.x;
  const long long rows_per_tile = (pixels + tiles - 1) / tiles;
  const long long r_begin = blockIdx.x * rows_per_tile;
  const long long r_end = min(pixels, r_begin + rows_per_tile);
  const float inv = 1.f / (float)(k * k);
  for (int cbase = 0; cbase < cpr; cbase += kSumThreads) {
    const int ccount = min(kSumThreads, cpr - cbase);
    const int rows_per_iter = kSumThreads / ccount;
    const int tcol = threadIdx.x % ccount, trow = threadIdx.x / ccount;
    const int c0 = (cbase + tcol) * V;
    Acc s1[V], s2[V];
#pragma unroll
    for (int i = 0; i < V; ++i) s1[i] = s2[i] = Acc(0);
    if (trow < rows_per_iter) {
      for (long long r = r_begin + trow; r < r_end; r += rows_per_iter) {
        const int img = (int)(r / ((long long)oh * ow));
        const int rem = (int)(r - (long long)img * oh * ow);
        const int oy = rem / ow, ox = rem - oy * ow;
        float acc[V];
#pragma unroll
        for (int i = 0; i < V; ++i) acc[i] = 0.f;
        if (k == 2) {  // the transitions and the stem: four independent 16-byte loads in flight
          const long long s0 = ((long long)img * h + oy * 2) * w + ox * 2;
          float f0[V], f1[V], f2[V], f3[V];
          VecIO<T>::load(x.p, s0 * x.rs + c0, f0);
          VecIO<T>::load(x.p, (s0 + 1) * x.rs + c0, f1);
          VecIO<T>::load(x.p, (s0 + w) * x.rs + c0, f2);
          VecIO<T>::load(x.p, (s0 + w + 1) * x.rs + c0, f3);
#pragma unroll
          for (int i = 0; i < V; ++i) acc[i] = ((f0[i] + f1[i]) + f2[i]) + f3[i];
        } else {
          for (int dy = 0; dy < k; ++dy)
            for (int dx = 0; dx < k; ++dx) {
              float f[V];
              const long long src = ((long long)img * h + oy * k + dy) * w + ox * k + dx;
              VecIO<T>::load(x.p, src * x.rs + c0, f);
#pragma unroll
              for (int i = 0; i < V; ++i) acc[i] += f[i];
            }
        }
#pragma unroll
        for (int i = 0; i < V; ++i) acc[i] = VecIO<T>::round(acc[i] * inv);
        VecIO<T>::store(const_cast<void*>(y.p), r * y.rs + c0, acc);
#pragma unroll
        for (int i = 0; i < V; ++i) {
          s1[i] += (Acc)(acc[i]);
          s2[i] += (Acc)acc[i] * (Acc)(acc[i]);
        }
      }
    }
    if (part == nullptr) continue;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      sh[0][threadIdx.x][i] = s1[i];
      sh[1][threadIdx.x][i] = s2[i];
    }
    __syncthreads();
    if (threadIdx.x < ccount) {
      Acc a[V], b[V];
#pragma unroll
      for (int i = 0; i < V; ++i) a[i] = b[i] = Acc(0);
      for (int rr = 0; rr < rows_per_iter; ++rr)
#pragma unroll
        for (int i = 0; i < V; ++i) {
          a[i] += sh[0][rr * ccount + threadIdx.x][i];
          b[i] += sh[1][rr * ccount + threadIdx.x][i];
        }
      const int cc = (cbase + threadIdx.x) * V;
#pragma unroll
      for (int i = 0; i < V; ++i) {
        part[((long long)blockIdx.x * 2 + 0) * C + cc + i] = a[i];
        part[((long long)blockIdx.x * 2 + 1) * C + cc + i] = b[i];
      }
    }
    __syncthreads();
  }
}

// large windows without statistics (the global head pool, ops.py:428-441 with k = h):
// one CTA per output pixel, the k*k window split over thread groups that each sum a
// fixed strided subset of window positions, then combined in group order (deterministic)
template <typename T>
__global__ void __launch_bounds__(256) avgpool_wide_kernel(View x, View y, int h, int w, int oh, int ow,
                                                           int C, int k) {
  griddep_launch();
  griddep_wait();
  constexpr int V = VecIO<T>::V;
  __shared__ float sh[256][V];
  const int cpr = C / V;
  const int groups = cpr >= 256 ? 1 : 256 / cpr;
  const int j = threadIdx.x % cpr, g = threadIdx.x / cpr;
  const int r = blockIdx.x;
  const int img = r / (oh * ow), rem = r - img * oh * ow;
  const int oy = rem / ow, ox = rem - oy * ow;
  const float inv = 1.f / (float)(k * k);
  for (int jj = j; jj < cpr; jj += (cpr >= 256 ? 256 : cpr)) {
    float acc[V];
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] = 0.f;
    if (g < groups) {
      int t = g;
      for (; t + 3 * groups < k * k; t += 4 * groups) {  // four loads in flight, summed in order
        float f[4][V];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int tt = t + u * groups, dy = tt / k, dx = tt - dy * k;
          VecIO<T>::load(x.p, (((long long)img * h + oy * k + dy) * w + ox * k + dx) * x.rs + jj * V, f[u]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int i = 0; i < V; ++i) acc[i] += f[u][i];
      }
      for (; t < k * k; t += groups) {
        const int dy = t / k, dx = t - dy * k;
        float f[V];
        VecIO<T>::load(x.p, (((long long)img * h + oy * k + dy) * w + ox * k + dx) * x.rs + jj * V, f);
#pragma unroll
        for (int i = 0; i < V; ++i) acc[i] += f[i];
      }
    }
#pragma unroll
    for (int i = 0; i < V; ++i) sh[threadIdx.x][i] = acc[i];
    __syncthreads();
    if (g == 0) {
      for (int q = 1; q < groups; ++q)
#pragma unroll
        for (int i = 0; i < V; ++i) acc[i] += sh[q * cpr + j][i];
#pragma unroll
      for (int i = 0; i < V; ++i) acc[i] = VecIO<T>::round(acc[i] * inv);
      VecIO<T>::store(const_cast<void*>(y.p), (long long)r * y.rs + jj * V, acc);
    }
    __syncthreads();
  }
}


// ---------------------------------------------------------------------------
// norm -> ReLU -> k x k average pool (the stem and any sub-BN2 -> ReLU -> AvgPool chain whose
// consumer is not a conv, graph.py:358-375): forward reads the conv output once and writes
// only the pooled map (+ its sub-BN1 partials); backward writes the BN-input gradient dt1 =
// ReLU'(bn(x)) * spread(dy)/k^2 and its (sum dt1, sum dt1*xhat) partials in the same pass
// (avgpool_bwd + relu_bwd + bn_bwd sums, ops.py:271-274, 314-319, 443-454).
// ---------------------------------------------------------------------------
template <typename T>
__global__ void norm_relu_pool_fwd_kernel(View x, View y, int n, int h, int w, int oh, int ow, int C, int k,
                                          bnff_coef cf, double* part) {
  griddep_launch();
  griddep_wait();
  constexpr int V = VecIO<T>::V;
  using Acc = typename std::conditional<sizeof(T) == 4, double, float>::type;  // f64 for fp32 data
  __shared__ Acc sh[2][kSumThreads][V];
  const long long pixels = (long long)n * oh * ow;
  const int cpr = C / V;
  const int tiles = gridDim.x;
  const long long rows_per_tile = (pixels + tiles - 1) / tiles;
  const long long r_begin = blockIdx.x * rows_per_tile;
  const long long r_end = min(pixels, r_begin + rows_per_tile);
  const float inv = 1.f / (float)(k * k);
  for (int cbase = 0; cbase < cpr; cbase += kSumThreads) {
    const int ccount = min(kSumThreads, cpr - cbase);
    const int rows_per_iter = kSumThreads / ccount;
    const int tcol = threadIdx.x % ccount, trow = threadIdx.x / ccount;
    const int c0 = (cbase + tcol) * V;
    Acc s1[V], s2[V];
    float ma[V], sc[V], be[V];
#pragma unroll
    for (int i = 0; i < V; ++i) s1[i] = s2[i] = Acc(0);
    if (trow < rows_per_iter) {
#pragma unroll
      for (int i = 0; i < V; ++i) {
        ma[i] = __ldg(cf.a + c0 + i);
        sc[i] = __ldg(cf.b + c0 + i);
        be[i] = __ldg(cf.c + c0 + i);
      }
      for (long long r = r_begin + trow; r < r_end; r += rows_per_iter) {
        const int img = (int)(r / ((long long)oh * ow));
        const int rem = (int)(r - (long long)img * oh * ow);
        const int oy = rem / ow, ox = rem - oy * ow;
        float acc[V];
#pragma unroll
        for (int i = 0; i < V; ++i) acc[i] = 0.f;
        for (int dy = 0; dy < k; ++dy)
          for (int dx = 0; dx < k; ++dx) {
            float f[V];
            const long long src = ((long long)img * h + oy * k + dy) * w + ox * k + dx;
            VecIO<T>::load(x.p, src * x.rs + c0, f);
#pragma unroll
            for (int i = 0; i < V; ++i)  // bn_fwd op order (ops.py:246-249), ReLU, in the storage precision
              acc[i] += VecIO<T>::round(fmaxf(__fadd_rn(__fmul_rn(__fsub_rn(f[i], ma[i]), sc[i]), be[i]), 0.f));
          }
#pragma unroll
        for (int i = 0; i < V; ++i) acc[i] = VecIO<T>::round(acc[i] * inv);
        VecIO<T>::store(const_cast<void*>(y.p), r * y.rs + c0, acc);
#pragma unroll
        for (int i = 0; i < V; ++i) {
          s1[i] += (Acc)(acc[i]);
          s2[i] += (Acc)acc[i] * (Acc)(acc[i]);
        }
      }
    }
    if (part == nullptr) continue;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      sh[0][threadIdx.x][i] = s1[i];
      sh[1][threadIdx.x][i] = s2[i];
    }
    __syncthreads();
    if (threadIdx.x < ccount) {
      Acc a[V], b[V];
#pragma unroll
      for (int i = 0; i < V; ++i) a[i] = b[i] = Acc(0);
      for (int rr = 0; rr < rows_per_iter; ++rr)
#pragma unroll
        for (int i = 0; i < V; ++i) {
          a[i] += sh[0][rr * ccount + threadIdx.x][i];
          b[i] += sh[1][rr * ccount + threadIdx.x][i];
        }
      const int cc = (cbase + threadIdx.x) * V;
#pragma unroll
      for (int i = 0; i < V; ++i) {
        part[((long long)blockIdx.x * 2 + 0) * C + cc + i] = a[i];
        part[((long long)blockIdx.x * 2 + 1) * C + cc + i] = b[i];
      }
    }
    __syncthreads();
  }
}

template <typename T>
__global__ void pool_relu_bn_bwd_kernel(View dyp, View x, View dr, int n, int h, int w, int oh, int ow, int C,
                                        int k, bnff_coef cf, double* part) {
  griddep_launch();
  griddep_wait();
  constexpr int V = VecIO<T>::V;
  using Acc = typename std::conditional<sizeof(T) == 4, double, float>::type;  // f64 for fp32 data
  __shared__ Acc sh[2][kSumThreads][V];
  const long long pixels = (long long)n * h * w;
  const int cpr = C / V;
  const int tiles = gridDim.x;
  const long long rows_per_tile = (pixels + tiles - 1) / tiles;
  const long long r_begin = blockIdx.x * rows_per_tile;
  const long long r_end = min(pixels, r_begin + rows_per_tile);
  const float inv = 1.f / (float)(k * k);
  for (int cbase = 0; cbase < cpr; cbase += kSumThreads) {
    const int ccount = min(kSumThreads, cpr - cbase);
    const int rows_per_iter = kSumThreads / ccount;
    const int tcol = threadIdx.x % ccount, trow = threadIdx.x / ccount;
    const int c0 = (cbase + tcol) * V;
    Acc s1[V], s2[V];
    float ma[V], sc[V], be[V], iv[V];
#pragma unroll
    for (int i = 0; i < V; ++i) s1[i] = s2[i] = Acc(0);
    if (trow < rows_per_iter) {
#pragma unroll
      for (int i = 0; i < V; ++i) {
        ma[i] = __ldg(cf.a + c0 + i);
        sc[i] = __ldg(cf.b + c0 + i);
        be[i] = __ldg(cf.c + c0 + i);
        iv[i] = __ldg(cf.d + c0 + i);
      }
      for (long long r = r_begin + trow; r < r_end; r += rows_per_iter) {
        const int img = (int)(r / ((long long)h * w));
        const int rem = (int)(r - (long long)img * h * w);
        const int yy = rem / w, xx = rem - yy * w;
        float xf[V], d[V];
        VecIO<T>::load(x.p, r * x.rs + c0, xf);
        const int py = yy / k, px = xx / k;
        if (py < oh && px < ow) {
          VecIO<T>::load(dyp.p, (((long long)img * oh + py) * ow + px) * dyp.rs + c0, d);
        } else {
#pragma unroll
          for (int i = 0; i < V; ++i) d[i] = 0.f;
        }
#pragma unroll
        for (int i = 0; i < V; ++i) {
          const float z = __fadd_rn(__fmul_rn(__fsub_rn(xf[i], ma[i]), sc[i]), be[i]);
          d[i] = VecIO<T>::round(z > 0.f ? VecIO<T>::round(d[i] * inv) : 0.f);
          const float xh = __fmul_rn(__fsub_rn(xf[i], ma[i]), iv[i]);
          s1[i] += (Acc)(d[i]);
          s2[i] += (Acc)d[i] * (Acc)(xh);
        }
        VecIO<T>::store(const_cast<void*>(dr.p), r * dr.rs + c0, d);
      }
    }
#pragma unroll
    for (int i = 0; i < V; ++i) {
      sh[0][threadIdx.x][i] = s1[i];
      sh[1][threadIdx.x][i] = s2[i];
    }
    __syncthreads();
    if (threadIdx.x < ccount) {
      Acc a[V], b[V];
#pragma unroll
      for (int i = 0; i < V; ++i) a[i] = b[i] = Acc(0);
      for (int rr = 0; rr < rows_per_iter; ++rr)
#pragma unroll
        for (int i = 0; i < V; ++i) {
          a[i] += sh[0][rr * ccount + threadIdx.x][i];
          b[i] += sh[1][rr * ccount + threadIdx.x][i];
        }
      const int cc = (cbase + threadIdx.x) * V;
#pragma unroll
      for (int i = 0; i < V; ++i) {
        part[((long long)blockIdx.x * 2 + 0) * C + cc + i] = a[i];
        part[((long long)blockIdx.x * 2 + 1) * C + cc + i] = b[i];
      }
    }
    __syncthreads();
  }
}

template <typename T>
__global__ void avgpool_bwd_kernel(View dy, View dx, int n, int h, int w, int oh, int ow, int C, int k) {
  griddep_launch();
  griddep_wait();
  constexpr int V = VecIO<T>::V;
  const int cpr = C / V;
  const long long total = (long long)n * h * w * cpr;
  const float inv = 1.f / (float)(k * k);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / cpr;
    const int c0 = (int)(i - r * cpr) * V;
    const int img = (int)(r / ((long long)h * w));
    const int rem = (int)(r - (long long)img * h * w);
    const int y = rem / w, x = rem - y * w;
    float f[V];
    if (y < oh * k && x < ow * k) {
      const long long src = ((long long)img * oh + y / k) * ow + x / k;
      VecIO<T>::load(dy.p, src * dy.rs + c0, f);
#pragma unroll
      for (int q = 0; q < V; ++q) f[q] = f[q] / (float)(k * k);
    } else {
#pragma unroll
      for (int q = 0; q < V; ++q) f[q] = 0.f;
    }
    (void)inv;
    VecIO<T>::store(const_cast<void*>(dx.p), r * dx.rs + c0, f);
  }
}

template <typename T>
__global__ void ews_kernel(View a, View b, View y, long long pixels, int C, int Cb) {
  griddep_launch();
  griddep_wait();
  constexpr int V = VecIO<T>::V;
  const int cpr = C / V;
  const long long total = pixels * cpr;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / cpr;
    const int c0 = (int)(i - r * cpr) * V;
    float f[V], g[V];
    VecIO<T>::load(a.p, r * a.rs + c0, f);
    if (c0 < Cb) {
      VecIO<T>::load(b.p, r * b.rs + c0, g);
#pragma unroll
      for (int q = 0; q < V; ++q) f[q] += g[q];
    }
    VecIO<T>::store(const_cast<void*>(y.p), r * y.rs + c0, f);
  }
}

template <typename T>
__global__ void copy_kernel(View s, View d, long long pixels, int C) {
  griddep_launch();
  griddep_wait();
  constexpr int V = VecIO<T>::V;
  const int cpr = C / V;
  const long long total = pixels * cpr;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / cpr;
    const int c0 = (int)(i - r * cpr) * V;
    float f[V];
    VecIO<T>::load(s.p, r * s.rs + c0, f);
    VecIO<T>::store(const_cast<void*>(d.p), r * d.rs + c0, f);
  }
}

template <typename T>
__global__ void nchw_to_nhwc_kernel(const float* src, long long n, long long c, long long h, long long w,
                                    View d, int Cs) {
  griddep_launch();
  griddep_wait();
  const long long total = n * h * w * Cs;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int ch = (int)(i % Cs);
    const long long pix = i / Cs;
    const long long img = pix / (h * w), rem = pix - img * h * w;
    const float v = ch < c ? src[(img * c + ch) * h * w + rem] : 0.f;
    T* dst = reinterpret_cast<T*>(const_cast<void*>(d.p)) + pix * d.rs + ch;
    if constexpr (sizeof(T) == 2) *dst = __float2bfloat16_rn(v);
    else *dst = v;
  }
}

// one thread per pixel when the stored pixel is exactly 16 bytes (8 bf16 / 4 f32): the
// c planes are read coalesced across consecutive pixels, one vector store per pixel
template <typename T>
__global__ void nchw_to_nhwc_px16_kernel(const float* __restrict__ src, long long n, int c, long long hw,
                                         View d) {
  griddep_launch();
  griddep_wait();
  constexpr int V = 16 / sizeof(T);
  const long long total = n * hw;
  for (long long pix = blockIdx.x * (long long)blockDim.x + threadIdx.x; pix < total;
       pix += (long long)gridDim.x * blockDim.x) {
    const long long img = pix / hw, rem = pix - img * hw;
    float f[V];
#pragma unroll
    for (int ch = 0; ch < V; ++ch) f[ch] = ch < c ? __ldg(src + (img * c + ch) * hw + rem) : 0.f;
    VecIO<T>::store(const_cast<void*>(d.p), pix * d.rs, f);
  }
}

template <typename T>
__global__ void nhwc_to_nchw_kernel(View s, long long n, long long c, long long h, long long w, float* dst) {
  griddep_launch();
  griddep_wait();
  const long long total = n * c * h * w;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long hw = i % (h * w);
    const long long t = i / (h * w);
    const int ch = (int)(t % c);
    const long long img = t / c;
    const T v = reinterpret_cast<const T*>(s.p)[(img * h * w + hw) * s.rs + ch];
    if constexpr (sizeof(T) == 2) dst[i] = __bfloat162float(v);
    else dst[i] = v;
  }
}

__global__ void sgd_kernel(float* w, const float* g, long long n, float lr) {
  griddep_launch();
  griddep_wait();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    w[i] = __fsub_rn(w[i], __fmul_rn(lr, g[i]));  // w - lr*g, two roundings (no FMA contraction)
}

template <typename T>
__global__ void pack_weights_kernel(const float* w, int co_n, int ci_n, int ci_s, int taps, int kpad,
                                    int kpad_t, T* wp, T* wt) {
  griddep_launch();
  griddep_wait();
  // forward pack [co][tap*ci_s + ci], transposed pack [ci][tap*co_n + co]
  const long long tot_f = (long long)co_n * kpad;
  const long long tot_t = (long long)ci_s * kpad_t;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot_f + tot_t;
       i += (long long)gridDim.x * blockDim.x) {
    float v = 0.f;
    if (i < tot_f) {
      const int co = (int)(i / kpad), k = (int)(i - (long long)co * kpad);
      const int tap = k / ci_s, ci = k - tap * ci_s;
      if (tap < taps && ci < ci_n) v = w[((long long)co * ci_n + ci) * taps + tap];
      if (wp) {
        if constexpr (sizeof(T) == 2) wp[i] = __float2bfloat16_rn(v);
        else wp[i] = v;
      }
    } else {
      const long long j = i - tot_f;
      const int ci = (int)(j / kpad_t), k = (int)(j - (long long)ci * kpad_t);
      const int tap = k / co_n, co = k - tap * co_n;
      if (tap < taps && ci < ci_n) v = w[((long long)co * ci_n + ci) * taps + tap];
      if (wt) {
        if constexpr (sizeof(T) == 2) wt[j] = __float2bfloat16_rn(v);
        else wt[j] = v;
      }
    }
  }
}

inline int grid_for(long long work, int threads = 256) {
  long long b = (work + threads - 1) / threads;
  const long long cap = 148 * 16;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

inline View vw(const bnff_view& v) { return View{v.ptr, (long long)v.row_stride}; }

inline int check_view(int dtype, const bnff_view& v, const char* what) {
  const int vec = dtype == BNFF_BF16 ? 8 : 4;
  if (dtype != BNFF_BF16 && dtype != BNFF_F32) return set_error(BNFF_ERR_UNSUPPORTED, "dtype %d", dtype);
  if (v.ptr == nullptr) return set_error(BNFF_ERR_STATE, "%s: null pointer", what);
  if (v.c % vec != 0 || v.row_stride % vec != 0 || (reinterpret_cast<uintptr_t>(v.ptr) & 15))
    return set_error(BNFF_ERR_UNSUPPORTED, "%s: c=%lld rs=%lld must be multiples of %d, 16B aligned", what,
                     (long long)v.c, (long long)v.row_stride, vec);
  return BNFF_OK;
}

inline bool same_dims(const bnff_view& a, const bnff_view& b) {
  return a.n == b.n && a.h == b.h && a.w == b.w && a.c == b.c;
}

}  // namespace bnff

using namespace bnff;

#define BNFF_DISPATCH(dtype, KERNEL, GRID, BLOCK, SMEM, STREAM, ...)                         \
  do {                                                                                       \
    if ((dtype) == BNFF_BF16) launch(KERNEL<__nv_bfloat16>, dim3(GRID), dim3(BLOCK), SMEM, STREAM, __VA_ARGS__); \
    else launch(KERNEL<float>, dim3(GRID), dim3(BLOCK), SMEM, STREAM, __VA_ARGS__);                          \
  } while (0)

extern "C" const char* bnff_last_error(void) { return g_err; }
extern "C" int bnff_version(void) { return 100; }
extern "C" int bnff_device_ok(void) {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return major == 10 && minor == 0 ? 1 : 0;
}

extern "C" int32_t bnff_sum_tiles(int64_t pixels) { return sum_tiles(pixels); }

template <typename T>
static void launch_sums_t(int mode, dim3 grid, cudaStream_t st, View x, View dy, long long pixels, int c, int cw,
                          bnff_coef cf, const double* mean, double* part) {
  switch (mode) {
    case 0: launch(channel_sums_kernel<T, 0>, grid, dim3(kSumThreads), 0, st, x, dy, pixels, c, cw, cf, mean, part); break;
    case 1: launch(channel_sums_kernel<T, 1>, grid, dim3(kSumThreads), 0, st, x, dy, pixels, c, cw, cf, mean, part); break;
    case 2: launch(channel_sums_kernel<T, 2>, grid, dim3(kSumThreads), 0, st, x, dy, pixels, c, cw, cf, mean, part); break;
    default: launch(channel_sums_kernel<T, 3>, grid, dim3(kSumThreads), 0, st, x, dy, pixels, c, cw, cf, mean, part);
  }
}
static void launch_sums(int dtype, int mode, dim3 grid, cudaStream_t st, View x, View dy, long long pixels, int c,
                        int cw, bnff_coef cf, const double* mean, double* part) {
  if (dtype == BNFF_BF16) launch_sums_t<__nv_bfloat16>(mode, grid, st, x, dy, pixels, c, cw, cf, mean, part);
  else launch_sums_t<float>(mode, grid, st, x, dy, pixels, c, cw, cf, mean, part);
}

extern "C" int bnff_channel_sums(int32_t dtype, int32_t mode, bnff_view x, bnff_view dy, bnff_coef coef,
                                 double* part, void* stream) {
  int rc;
  const bnff_view& shape = (mode == 0) ? x : dy;
  if ((rc = check_view(dtype, shape, "channel_sums"))) return rc;
  if ((mode == 1 || (mode == 2 && coef.e)) && (rc = check_view(dtype, x, "channel_sums x"))) return rc;
  if (mode == 1 && !same_dims(x, dy)) return set_error(BNFF_ERR_SHAPE, "channel_sums: x/dy dims differ");
  const long long pixels = shape.n * shape.h * shape.w;
  const int tiles = sum_tiles(pixels);
  const int cw = sum_col_width(dtype, (int)shape.c, tiles);
  const dim3 grid(tiles, (unsigned)((shape.c / (dtype == BNFF_F32 ? 4 : 8) + cw - 1) / cw));
  launch_sums(dtype, mode, grid, (cudaStream_t)stream, vw(x), vw(dy), pixels, (int)shape.c, cw, coef, nullptr, part);
  return check_launch("channel_sums");
}

extern "C" int bnff_stats_finalize(const double* part, int32_t tiles, int32_t c, int64_t count, double* sum,
                                   double* sumsq, double* mean, double* var, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  launch(stats_finalize_kernel, dim3((c + 31) / 32), dim3(512), 0, st, part, tiles, c, count, sum, sumsq, mean, var);
  return check_launch("stats_finalize");
}

extern "C" int bnff_centered_var(int32_t dtype, bnff_view x, const double* mean, double* part, void* stream) {
  int rc;
  if ((rc = check_view(dtype, x, "centered_var"))) return rc;
  const long long pixels = x.n * x.h * x.w;
  const int tiles = sum_tiles(pixels);
  bnff_coef cf{};
  const int cw = sum_col_width(dtype, (int)x.c, tiles);
  const dim3 grid(tiles, (unsigned)((x.c / (dtype == BNFF_F32 ? 4 : 8) + cw - 1) / cw));
  launch_sums(dtype, 3, grid, (cudaStream_t)stream, vw(x), vw(x), pixels, (int)x.c, cw, cf, mean, part);
  return check_launch("centered_var");
}

extern "C" int bnff_var_finalize(const double* part, int32_t tiles, int32_t c, int64_t count, double* var,
                                 void* stream);

namespace bnff {
__global__ void scale_kernel(double* v, int c, double s) {
  griddep_launch();
  griddep_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < c) v[i] = v[i] * s;
}
}  // namespace bnff

namespace bnff {
// centred partials -> var = sum(d^2) * (1/count) (ops.py:227), and -- when gamma is given --
// the fp32 prologue tables of bn_coeffs from (mean, var): the unfused BN's second pass
// ends in one launch
__global__ void __launch_bounds__(512) var_finalize_kernel(const double* __restrict__ part, int tiles, int C,
                                                           double rcount, double* var, const double* mean,
                                                           const float* gamma, const float* beta, float eps,
                                                           float* mean32, float* scale32, float* beta32,
                                                           float* inv32) {
  griddep_launch();
  griddep_wait();
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  double s1, s2;
  reduce_two(part, tiles, C, c, s1, s2);
  if ((threadIdx.x >> 5) == 0 && c < C) {
    const double v = s1 * rcount;
    var[c] = v;
    if (gamma) {
      const double vv = v > 0.0 ? v : 0.0;
      const double inv = 1.0 / sqrt(vv + (double)eps);
      mean32[c] = (float)mean[c];
      scale32[c] = (float)((double)gamma[c] * inv);
      beta32[c] = beta[c];
      inv32[c] = (float)inv;
    }
  }
}
}  // namespace bnff

extern "C" int bnff_var_finalize(const double* part, int32_t tiles, int32_t c, int64_t count, double* var,
                                 void* stream) {
  launch(var_finalize_kernel, dim3((c + 31) / 32), dim3(512), 0, (cudaStream_t)stream, part, tiles, c,
         1.0 / (double)count, var, (const double*)nullptr, (const float*)nullptr, (const float*)nullptr, 0.f,
         (float*)nullptr, (float*)nullptr, (float*)nullptr, (float*)nullptr);
  return check_launch("var_finalize");
}

extern "C" int bnff_var_finalize_coeffs(const double* part, int32_t tiles, int32_t c, int64_t count, double* var,
                                        const double* mean, const float* gamma, const float* beta, float eps,
                                        float* mean32, float* scale32, float* beta32, float* inv32,
                                        void* stream) {
  if (!mean || !gamma || !beta || !mean32 || !scale32 || !beta32 || !inv32)
    return set_error(BNFF_ERR_STATE, "var_finalize_coeffs: null table");
  launch(var_finalize_kernel, dim3((c + 31) / 32), dim3(512), 0, (cudaStream_t)stream, part, tiles, c,
         1.0 / (double)count, var, mean, gamma, beta, eps, mean32, scale32, beta32, inv32);
  return check_launch("var_finalize_coeffs");
}

extern "C" int bnff_stats_finalize_coeffs(const double* part, int32_t tiles, int32_t c_new, int64_t count,
                                          double* sum, double* sumsq, double* mean, double* var,
                                          int32_t c_off, int32_t c_total, const double* mean_all,
                                          const double* var_all, const float* gamma, const float* beta,
                                          float eps, float* mean32, float* scale32, float* beta32,
                                          float* inv32, void* stream) {
  if (c_off < 0 || c_new < 0 || c_off + c_new > c_total) return set_error(BNFF_ERR_SHAPE, "finalize_coeffs: piece range");
  launch(finalize_coeffs_kernel, dim3((c_total + 31) / 32), dim3(512), 0, (cudaStream_t)stream, part, tiles, c_new,
         (long long)count, sum, sumsq, mean, var, c_off, c_total, mean_all, var_all, gamma, beta, eps, mean32,
         scale32, beta32, inv32);
  return check_launch("stats_finalize_coeffs");
}

extern "C" int bnff_bn_coeffs(int32_t c, const double* mean, const double* var, const float* gamma,
                              const float* beta, float eps, float* mean32, float* scale32, float* beta32,
                              float* inv32, void* stream) {
  launch(bn_coeffs_kernel, dim3((c + 127) / 128), dim3(128), 0, (cudaStream_t)stream, c, mean, var, gamma, beta, eps, mean32,
                                                                       scale32, beta32, inv32);
  return check_launch("bn_coeffs");
}

extern "C" int bnff_dx_coeffs(int32_t c, const double* part, int32_t tiles, int64_t count, const double* mean,
                              const double* var, const float* gamma, float eps, double* dgamma64,
                              double* dbeta64, float* k1, float* k2, float* g, float* mean32, float* inv32,
                              float* dgamma32, float* dbeta32, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  launch(dx_coeffs_fused_kernel, dim3((c + 31) / 32), dim3(512), 0, st, part, tiles, c, count, mean, var, gamma, eps, dgamma64,
                                                         dbeta64, k1, k2, g, mean32, inv32, dgamma32, dbeta32,
         (float*)nullptr, (float*)nullptr, 0);
  return check_launch("dx_coeffs");
}

extern "C" int bnff_dx_coeffs_acc(int32_t c, const double* part, int32_t tiles, int64_t count, const double* mean,
                                  const double* var, const float* gamma, float eps, double* dgamma64,
                                  double* dbeta64, float* k1, float* k2, float* g, float* mean32, float* inv32,
                                  float* dgamma32, float* dbeta32, float* acc_a, float* acc_b, int32_t acc_init,
                                  void* stream) {
  if (!acc_a || !acc_b) return set_error(BNFF_ERR_SHAPE, "dx_coeffs_acc: accumulators required");
  cudaStream_t st = (cudaStream_t)stream;
  launch(dx_coeffs_fused_kernel, dim3((c + 31) / 32), dim3(512), 0, st, part, tiles, c, count, mean, var, gamma, eps, dgamma64,
                                                         dbeta64, k1, k2, g, mean32, inv32, dgamma32, dbeta32, acc_a,
         acc_b, (int)acc_init);
  return check_launch("dx_coeffs_acc");
}

extern "C" int bnff_bn_apply(int32_t dtype, bnff_view x, bnff_view y, bnff_coef coef, int32_t relu,
                             void* stream) {
  int rc;
  if ((rc = check_view(dtype, x, "bn_apply x")) || (rc = check_view(dtype, y, "bn_apply y"))) return rc;
  if (!same_dims(x, y)) return set_error(BNFF_ERR_SHAPE, "bn_apply: x/y dims differ");
  if (!coef.a || !coef.b || !coef.c) return set_error(BNFF_ERR_STATE, "bn_apply: missing statistics");
  const long long pixels = x.n * x.h * x.w;
  BNFF_DISPATCH(dtype, bn_apply_kernel, rowchunk_grid(pixels, (int)x.c, dtype == BNFF_BF16 ? 8 : 4), 256, 0,
                (cudaStream_t)stream, vw(x), vw(y), pixels, (int)x.c, coef, relu);
  return check_launch("bn_apply");
}

extern "C" int bnff_grad_sum(int32_t dtype, bnff_view out, int32_t accumulate, const bnff_grad_term* terms,
                             int32_t nterms, void* stream) {
  int rc;
  if (nterms < 1 || nterms > 2) return set_error(BNFF_ERR_UNSUPPORTED, "grad_sum: 1..2 terms");
  if ((rc = check_view(dtype, out, "grad_sum out"))) return rc;
  TermDev td[2]{};
  for (int i = 0; i < nterms; ++i) {
    if ((rc = check_view(dtype, terms[i].g, "grad_sum term"))) return rc;
    if (!same_dims(terms[i].g, out)) return set_error(BNFF_ERR_SHAPE, "grad_sum: term %d dims differ", i);
    if (terms[i].deferred && (rc = check_view(dtype, terms[i].x, "grad_sum term x"))) return rc;
    td[i].g = vw(terms[i].g);
    td[i].x = vw(terms[i].x);
    td[i].deferred = terms[i].deferred;
    td[i].cf = terms[i].coef;
  }
  const long long pixels = out.n * out.h * out.w;
  if (dtype == BNFF_BF16) {
    const int grid = rowchunk_grid(pixels, (int)out.c, 8);
    if (nterms == 1)
      launch(grad_sum_bf16_kernel<4, 1>, dim3(grid), dim3(256), 0, (cudaStream_t)stream, vw(out), pixels, (int)out.c, accumulate,
                                                                      td[0], td[1], nterms);
    else
      launch(grad_sum_bf16_kernel<2, 2>, dim3(grid), dim3(256), 0, (cudaStream_t)stream, vw(out), pixels, (int)out.c, accumulate,
                                                                      td[0], td[1], nterms);
    return check_launch("grad_sum");
  }
  BNFF_DISPATCH(dtype, grad_sum_kernel, rowchunk_grid(pixels, (int)out.c, dtype == BNFF_BF16 ? 8 : 4), 256, 0,
                (cudaStream_t)stream, vw(out), pixels, (int)out.c, accumulate, td[0], td[1], nterms);
  return check_launch("grad_sum");
}

extern "C" int bnff_relu_fwd(int32_t dtype, bnff_view x, bnff_view y, void* stream) {
  int rc;
  if ((rc = check_view(dtype, x, "relu x")) || (rc = check_view(dtype, y, "relu y"))) return rc;
  const long long pixels = x.n * x.h * x.w;
  BNFF_DISPATCH(dtype, relu_kernel, rowchunk_grid(pixels, (int)x.c, dtype == BNFF_BF16 ? 8 : 4), 256, 0,
                (cudaStream_t)stream, vw(x), vw(x), vw(y), pixels, (int)x.c, 0);
  return check_launch("relu_fwd");
}

extern "C" int bnff_relu_bwd(int32_t dtype, bnff_view x, bnff_view dy, bnff_view dx, void* stream) {
  int rc;
  if ((rc = check_view(dtype, x, "relu_bwd x")) || (rc = check_view(dtype, dy, "relu_bwd dy")) ||
      (rc = check_view(dtype, dx, "relu_bwd dx")))
    return rc;
  if (!same_dims(x, dy)) return set_error(BNFF_ERR_SHAPE, "relu_bwd: shape mismatch");
  const long long pixels = x.n * x.h * x.w;
  BNFF_DISPATCH(dtype, relu_kernel, rowchunk_grid(pixels, (int)x.c, dtype == BNFF_BF16 ? 8 : 4), 256, 0,
                (cudaStream_t)stream, vw(x), vw(dy), vw(dx), pixels, (int)x.c, 1);
  return check_launch("relu_bwd");
}

extern "C" int bnff_avgpool_fwd(int32_t dtype, bnff_view x, bnff_view y, int32_t k, double* stat_part,
                                void* stream) {
  int rc;
  if ((rc = check_view(dtype, x, "avgpool x")) || (rc = check_view(dtype, y, "avgpool y"))) return rc;
  if (y.h != x.h / k || y.w != x.w / k || y.c != x.c || y.n != x.n || y.h < 1 || y.w < 1)
    return set_error(BNFF_ERR_SHAPE, "avgpool: bad output dims");
  const long long pixels = y.n * y.h * y.w;
  if (stat_part == nullptr && k * k > 4 && pixels <= 148 * 64) {
    BNFF_DISPATCH(dtype, avgpool_wide_kernel, (int)pixels, 256, 0, (cudaStream_t)stream, vw(x), vw(y), (int)x.h,
                  (int)x.w, (int)y.h, (int)y.w, (int)x.c, k);
    return check_launch("avgpool_fwd");
  }
  BNFF_DISPATCH(dtype, avgpool_fwd_kernel, sum_tiles(pixels), kSumThreads, 0, (cudaStream_t)stream, vw(x), vw(y),
                (int)x.n, (int)x.h, (int)x.w, (int)y.h, (int)y.w, (int)x.c, k, stat_part);
  return check_launch("avgpool_fwd");
}

extern "C" int bnff_norm_relu_pool_fwd(int32_t dtype, bnff_view x, bnff_view y, int32_t k, bnff_coef coef,
                                       double* stat_part, void* stream) {
  int rc;
  if ((rc = check_view(dtype, x, "norm_relu_pool x")) || (rc = check_view(dtype, y, "norm_relu_pool y"))) return rc;
  if (y.h != x.h / k || y.w != x.w / k || y.c != x.c || y.n != x.n || y.h < 1 || y.w < 1)
    return set_error(BNFF_ERR_SHAPE, "norm_relu_pool: bad output dims");
  if (!coef.a || !coef.b || !coef.c) return set_error(BNFF_ERR_STATE, "norm_relu_pool: missing statistics");
  const long long pixels = y.n * y.h * y.w;
  BNFF_DISPATCH(dtype, norm_relu_pool_fwd_kernel, sum_tiles(pixels), kSumThreads, 0, (cudaStream_t)stream, vw(x),
                vw(y), (int)x.n, (int)x.h, (int)x.w, (int)y.h, (int)y.w, (int)x.c, k, coef, stat_part);
  return check_launch("norm_relu_pool_fwd");
}

extern "C" int bnff_pool_relu_bn_bwd(int32_t dtype, bnff_view dy, bnff_view x, bnff_view dt1, int32_t k,
                                     bnff_coef coef, double* part, void* stream) {
  int rc;
  if ((rc = check_view(dtype, dy, "pool_relu_bn_bwd dy")) || (rc = check_view(dtype, x, "pool_relu_bn_bwd x")) ||
      (rc = check_view(dtype, dt1, "pool_relu_bn_bwd dt1")))
    return rc;
  if (dy.h != x.h / k || dy.w != x.w / k || dy.c != x.c || dt1.c != x.c || dt1.h != x.h || dt1.w != x.w)
    return set_error(BNFF_ERR_SHAPE, "pool_relu_bn_bwd: dims");
  if (!coef.a || !coef.b || !coef.c || !coef.d) return set_error(BNFF_ERR_STATE, "pool_relu_bn_bwd: missing tables");
  const long long pixels = x.n * x.h * x.w;
  BNFF_DISPATCH(dtype, pool_relu_bn_bwd_kernel, sum_tiles(pixels), kSumThreads, 0, (cudaStream_t)stream, vw(dy),
                vw(x), vw(dt1), (int)x.n, (int)x.h, (int)x.w, (int)dy.h, (int)dy.w, (int)x.c, k, coef, part);
  return check_launch("pool_relu_bn_bwd");
}

extern "C" int bnff_avgpool_bwd(int32_t dtype, bnff_view dy, bnff_view dx, int32_t k, void* stream) {
  int rc;
  if ((rc = check_view(dtype, dy, "avgpool_bwd dy")) || (rc = check_view(dtype, dx, "avgpool_bwd dx"))) return rc;
  const long long pixels = dx.n * dx.h * dx.w;
  BNFF_DISPATCH(dtype, avgpool_bwd_kernel, grid_for(pixels * dx.c / (dtype == BNFF_BF16 ? 8 : 4)), 256, 0,
                (cudaStream_t)stream, vw(dy), vw(dx), (int)dx.n, (int)dx.h, (int)dx.w, (int)dy.h, (int)dy.w,
                (int)dx.c, k);
  return check_launch("avgpool_bwd");
}

extern "C" int bnff_ews_fwd(int32_t dtype, bnff_view a, bnff_view b, bnff_view y, void* stream) {
  int rc;
  if ((rc = check_view(dtype, a, "ews a")) || (rc = check_view(dtype, b, "ews b")) ||
      (rc = check_view(dtype, y, "ews y")))
    return rc;
  if (b.c > a.c || a.n != b.n || a.h != b.h || a.w != b.w) return set_error(BNFF_ERR_SHAPE, "ews: bad dims");
  const long long pixels = a.n * a.h * a.w;
  BNFF_DISPATCH(dtype, ews_kernel, grid_for(pixels * a.c / (dtype == BNFF_BF16 ? 8 : 4)), 256, 0,
                (cudaStream_t)stream, vw(a), vw(b), vw(y), pixels, (int)a.c, (int)b.c);
  return check_launch("ews_fwd");
}

extern "C" int bnff_copy(int32_t dtype, bnff_view src, bnff_view dst, void* stream) {
  int rc;
  if ((rc = check_view(dtype, src, "copy src")) || (rc = check_view(dtype, dst, "copy dst"))) return rc;
  if (!same_dims(src, dst)) return set_error(BNFF_ERR_SHAPE, "copy: dims differ");
  const long long pixels = src.n * src.h * src.w;
  BNFF_DISPATCH(dtype, copy_kernel, grid_for(pixels * src.c / (dtype == BNFF_BF16 ? 8 : 4)), 256, 0,
                (cudaStream_t)stream, vw(src), vw(dst), pixels, (int)src.c);
  return check_launch("copy");
}

extern "C" int bnff_nchw_to_nhwc(int32_t dtype, const float* src, int64_t n, int64_t c, int64_t h, int64_t w,
                                 bnff_view dst, void* stream) {
  if (dst.c < c || dst.n != n || dst.h != h || dst.w != w) return set_error(BNFF_ERR_SHAPE, "nchw_to_nhwc dims");
  const int vec = dtype == BNFF_BF16 ? 8 : 4;
  if (dst.c == vec && dst.row_stride % vec == 0) {  // the channel-padded image: 16-byte pixels
    BNFF_DISPATCH(dtype, nchw_to_nhwc_px16_kernel, grid_for(n * h * w), 256, 0, (cudaStream_t)stream, src, n,
                  (int)c, h * w, vw(dst));
    return check_launch("nchw_to_nhwc");
  }
  BNFF_DISPATCH(dtype, nchw_to_nhwc_kernel, grid_for(n * h * w * dst.c), 256, 0, (cudaStream_t)stream, src, n,
                c, h, w, vw(dst), (int)dst.c);
  return check_launch("nchw_to_nhwc");
}

extern "C" int bnff_nhwc_to_nchw(int32_t dtype, bnff_view src, float* dst, void* stream) {
  BNFF_DISPATCH(dtype, nhwc_to_nchw_kernel, grid_for(src.n * src.c * src.h * src.w), 256, 0,
                (cudaStream_t)stream, vw(src), src.n, src.c, src.h, src.w, dst);
  return check_launch("nhwc_to_nchw");
}

extern "C" int bnff_sgd(float* w, const float* g, int64_t n, float lr, void* stream) {
  launch(sgd_kernel, dim3(grid_for(n)), dim3(256), 0, (cudaStream_t)stream, w, g, n, lr);
  return check_launch("sgd");
}

extern "C" int64_t bnff_pack_size(int32_t dtype, int32_t c_out, int32_t c_in_store, int32_t kh, int32_t kw) {
  const int kb = dtype == BNFF_BF16 ? 64 : 32;
  const long long k = (long long)kh * kw * c_in_store;
  return (long long)c_out * ((k + kb - 1) / kb * kb);
}

extern "C" int bnff_pack_weights(int32_t dtype, const float* w, int32_t c_out, int32_t c_in, int32_t c_in_store,
                                 int32_t kh, int32_t kw, void* wpack, void* wpack_t, void* stream) {
  const int kb = dtype == BNFF_BF16 ? 64 : 32;
  const int taps = kh * kw;
  const int kpad = (taps * c_in_store + kb - 1) / kb * kb;
  const int kpad_t = (taps * c_out + kb - 1) / kb * kb;
  const long long work = (long long)c_out * kpad + (long long)c_in_store * kpad_t;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == BNFF_BF16)
    launch(pack_weights_kernel<__nv_bfloat16>, dim3(grid_for(work)), dim3(256), 0, st, 
        w, c_out, c_in, c_in_store, taps, kpad, kpad_t, (__nv_bfloat16*)wpack, (__nv_bfloat16*)wpack_t);
  else
    launch(pack_weights_kernel<float>, dim3(grid_for(work)), dim3(256), 0, st, w, c_out, c_in, c_in_store, taps, kpad, kpad_t,
                                                               (float*)wpack, (float*)wpack_t);
  return check_launch("pack_weights");
}

// dbias = sum over pixels of dy (optionally BN_DX-transformed); scratch is the
// caller's partial buffer [tiles][2][C] placed after the wgrad workspace.
namespace bnff {
__global__ void parts_to_f32_kernel(const double* part, int tiles, int C, float* out) {
  griddep_launch();
  griddep_wait();
  // 256 threads per 32 channels; 8 warps split the tiles, combined in fixed order
  __shared__ double sh[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + tx;
  double acc = 0.0;
  if (c < C)
    for (int t = ty; t < tiles; t += 8) acc += (double)part[(long long)t * 2 * C + c];
  sh[ty][tx] = acc;
  __syncthreads();
  if (ty == 0 && c < C) {
    double s = 0.0;
    for (int k = 0; k < 8; ++k) s += sh[k][tx];
    out[c] = (float)s;
  }
}
}  // namespace bnff

extern "C" int bnff_dbias_scratch(int32_t dtype, bnff_view dy, bnff_view dy_x, int32_t dy_pro, bnff_coef coef,
                                  double* scratch, float* dbias, void* stream) {
  bnff_coef cf = coef;
  if (dy_pro != BNFF_PRO_BN_DX) cf.e = nullptr;
  int rc = bnff_channel_sums(dtype, 2, dy_x, dy, cf, scratch, stream);
  if (rc) return rc;
  const long long pixels = dy.n * dy.h * dy.w;
  launch(parts_to_f32_kernel, dim3((int)((dy.c + 31) / 32)), dim3(256), 0, (cudaStream_t)stream, scratch, sum_tiles(pixels),
                                                                                (int)dy.c, dbias);
  return check_launch("dbias");
}

// ---------------------------------------------------------------------------
// SyncBN helpers: finalize from (all-reduced) float64 sums
// ---------------------------------------------------------------------------
namespace bnff {
__global__ void dx_coeffs_from_sums_kernel(int C, long long count, const double* dbeta64,
                                           const double* dgamma64, const double* mean, const double* var,
                                           const float* gamma, float eps, float* k1, float* k2, float* g,
                                           float* mean32, float* inv32) {
  griddep_launch();
  griddep_wait();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const double v = var[c] > 0.0 ? var[c] : 0.0;
  const double inv = 1.0 / sqrt(v + (double)eps);
  k1[c] = (float)(dbeta64[c] / (double)count);
  k2[c] = (float)(dgamma64[c] / (double)count);
  g[c] = (float)((double)gamma[c] * inv);
  mean32[c] = (float)mean[c];
  inv32[c] = (float)inv;
}
__global__ void sums_to_f32_kernel(int C, const double* a, const double* b, float* a32, float* b32) {
  griddep_launch();
  griddep_wait();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  if (a32) a32[c] = (float)a[c];
  if (b32) b32[c] = (float)b[c];
}
}  // namespace bnff

extern "C" int bnff_stats_from_sums(int32_t c, int64_t count, const double* sum, const double* sumsq,
                                    double* mean, double* var, void* stream) {
  launch(stats_from_sums_kernel, dim3((c + 127) / 128), dim3(128), 0, (cudaStream_t)stream, c,
         (long long)count, sum, sumsq, mean, var);
  return check_launch("stats_from_sums");
}

extern "C" int bnff_dx_coeffs_from_sums(int32_t c, int64_t count, const double* dbeta64, const double* dgamma64,
                                        const double* mean, const double* var, const float* gamma, float eps,
                                        float* k1, float* k2, float* g, float* mean32, float* inv32,
                                        void* stream) {
  launch(dx_coeffs_from_sums_kernel, dim3((c + 127) / 128), dim3(128), 0, (cudaStream_t)stream, c,
         (long long)count, dbeta64, dgamma64, mean, var, gamma, eps, k1, k2, g, mean32, inv32);
  return check_launch("dx_coeffs_from_sums");
}

extern "C" int bnff_sums_to_f32(int32_t c, const double* a, const double* b, float* a32, float* b32,
                                void* stream) {
  launch(sums_to_f32_kernel, dim3((c + 127) / 128), dim3(128), 0, (cudaStream_t)stream, c, a, b, a32, b32);
  return check_launch("sums_to_f32");
}

// ncu node ledger (tools/ncu_node_ledger.py): an empty kernel launched before every engine
// launch so a profiler's launch list can be cut into per-launch (per graph node) groups
namespace bnff {
__global__ void mark_kernel(int) {}
}  // namespace bnff
extern "C" int bnff_debug_mark(int32_t id, void* stream) {
  bnff::mark_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(id);
  return check_launch("mark");
}
