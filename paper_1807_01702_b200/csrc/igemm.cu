// igemm.cu -- implicit-GEMM convolution kernels on tcgen05 / TMEM (sm_100a).
//
// One warp-specialised kernel template serves the three convolution passes of
// the restructured-BN training path:
//
//   FPROP  C[pix, co]   = sum_{tap,ci} pro(x)[pix+tap, ci] * W[co, tap, ci]
//          prologue: none | ReLU (RCF) | BN-normalize+ReLU (sub-BN2, fused.py:133-135)
//          epilogue: +bias, store at a channel offset of an NHWC block buffer
//                    (in-place concat), per-channel sum/sum^2 partials of the
//                    STORED values (sub-BN1 + MVF, fused.py:91-98)
//   DGRAD  C[pix, ci]   = sum_{tap,co} pro(dy)[pix-tap, co] * W[co, tap, ci]
//          prologue: none | deferred BN dx of the incoming package (sub-BN1', ops.py:283-298)
//          epilogue: plain | clip mask (x>0) | NRC: mask relu(bn(x))>0 recomputed
//                    from x, dt1 store, sum dt1 / sum dt1*xhat partials (fused.py:176-188)
//   WGRAD  C[tap*ci, co] = sum_{pix} pro(x)[pix+tap, ci] * pro(dy)[pix, co]
//          (split-K over pixels; MN-major operands; deterministic fixed-order reduce)
//
// CTA = 160 threads: warps 0-3 gather operands global->registers->transform->
// swizzled shared memory (they are also the epilogue: warp w owns TMEM lanes
// 32w..32w+31), warp 4 owns TMEM and one elected lane issues tcgen05.mma.
// Stage hand-off uses mbarriers (producers arrive; tcgen05.commit frees a slot).
// Layout/descriptor encodings validated on B200 by tools/umma_probe.cu.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "sm100.cuh"
#include "common.cuh"

namespace bnff {

enum { MODE_FPROP = 0, MODE_DGRAD = 1, MODE_WGRAD = 2 };

struct IgParams {
  int M, N;             // GEMM extents
  int nkb;              // total k-blocks
  int kpt;              // k-blocks per tile (WGRAD: per split)
  int mtiles, ntiles, splits, ntiles_total;
  // geometry (conv input h,w; output oh,ow)
  int n, h, w, cin, oh, ow, cout, kh, kw, stride, pad, taps;
  int kred;             // reduction channel count of the K index (fprop: cin, dgrad: cout)
  FastDiv fd_kred, fd_kw, fd_ohow, fd_ow, fd_hw, fd_w, fd_cin;
  // A operand source
  const void* a_ptr; long long a_rs;
  const void* a_xptr; long long a_xrs;
  int a_pro; bnff_coef a_coef;
  // B operand source
  const void* b_ptr; long long b_rs;
  const void* b_xptr; long long b_xrs;
  int b_pro; bnff_coef b_coef;
  // epilogue
  void* c_ptr; long long c_rs;
  const float* bias;
  int epi;
  const void* e_xptr; long long e_xrs;
  bnff_coef e_coef;
  double* stat_part;
  int stat_ld;
  int tf32_mode;  // fp32: 0 = hi*hi + hi*lo + lo*hi, 1 = + lo*lo, 2 = cross terms first (BNFF_TF32_MODE)
};

// ---------------------------------------------------------------------------
// 16-byte chunk: 8 bf16 or 4 f32, as floats
// ---------------------------------------------------------------------------
template <typename T> struct Chunk;
template <> struct Chunk<__nv_bfloat16> {
  static constexpr int V = 8;
  uint4 raw;
  __device__ __forceinline__ void load(const void* p) { raw = __ldg(reinterpret_cast<const uint4*>(p)); }
  __device__ __forceinline__ void zero() { raw = make_uint4(0, 0, 0, 0); }
  __device__ __forceinline__ void to_float(float (&f)[8]) const {
    f[0] = bf16lo(raw.x); f[1] = bf16hi(raw.x); f[2] = bf16lo(raw.y); f[3] = bf16hi(raw.y);
    f[4] = bf16lo(raw.z); f[5] = bf16hi(raw.z); f[6] = bf16lo(raw.w); f[7] = bf16hi(raw.w);
  }
};
template <> struct Chunk<float> {
  static constexpr int V = 4;
  float4 raw;
  __device__ __forceinline__ void load(const void* p) { raw = __ldg(reinterpret_cast<const float4*>(p)); }
  __device__ __forceinline__ void zero() { raw = make_float4(0.f, 0.f, 0.f, 0.f); }
  __device__ __forceinline__ void to_float(float (&f)[4]) const {
    f[0] = raw.x; f[1] = raw.y; f[2] = raw.z; f[3] = raw.w;
  }
};

// operand prologue transforms (exact fp32 op order of the reference, no FMA contraction)
// per-channel coefficients of a V-channel chunk as vector loads (c0 is a multiple of V;
// every coefficient array is 16-byte aligned at such offsets)
template <int V>
__device__ __forceinline__ void ldv(const float* p, int c0, float (&o)[V]) {
#pragma unroll
  for (int i = 0; i < V; i += 4) {
    const float4 t = __ldg(reinterpret_cast<const float4*>(p + c0 + i));
    o[i] = t.x; o[i + 1] = t.y; o[i + 2] = t.z; o[i + 3] = t.w;
  }
}

// the per-channel coefficients of one V-channel chunk, loaded once per stage by a thread
// whose chunk column is fixed for the whole stage
template <int V>
struct ProCoef {
  float a[V], b[V], c[V], d[V], e[V];
  __device__ __forceinline__ void load(int pro, int c0, const bnff_coef& cf) {
    if (pro == BNFF_PRO_BN_RELU || pro == BNFF_PRO_BN_DX) {
      ldv<V>(cf.a, c0, a);
      ldv<V>(cf.b, c0, b);
      ldv<V>(cf.c, c0, c);
    }
    if (pro == BNFF_PRO_BN_DX) {
      ldv<V>(cf.d, c0, d);
      ldv<V>(cf.e, c0, e);
    }
  }
  __device__ __forceinline__ void apply(int pro, float (&f)[V], const float (&xf)[V]) const {
    if (pro == BNFF_PRO_RELU) {
#pragma unroll
      for (int i = 0; i < V; ++i) f[i] = fmaxf(f[i], 0.f);
    } else if (pro == BNFF_PRO_BN_RELU) {
#pragma unroll
      for (int i = 0; i < V; ++i) f[i] = fmaxf(__fadd_rn(__fmul_rn(__fsub_rn(f[i], a[i]), b[i]), c[i]), 0.f);
    } else if (pro == BNFF_PRO_BN_DX) {
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const float xh = __fmul_rn(__fsub_rn(xf[i], a[i]), b[i]);
        f[i] = __fmul_rn(e[i], __fsub_rn(__fsub_rn(f[i], c[i]), __fmul_rn(xh, d[i])));
      }
    }
  }
};

template <int V>
__device__ __forceinline__ void apply_pro(int pro, float (&f)[V], const float (&xf)[V], int c0,
                                          const bnff_coef& cf) {
  if (pro == BNFF_PRO_RELU) {
#pragma unroll
    for (int i = 0; i < V; ++i) f[i] = fmaxf(f[i], 0.f);
  } else if (pro == BNFF_PRO_BN_RELU) {
    float a[V], b[V], c[V];
    ldv<V>(cf.a, c0, a);
    ldv<V>(cf.b, c0, b);
    ldv<V>(cf.c, c0, c);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      float t = __fmul_rn(__fsub_rn(f[i], a[i]), b[i]);
      f[i] = fmaxf(__fadd_rn(t, c[i]), 0.f);
    }
  } else if (pro == BNFF_PRO_BN_DX) {
    float a[V], b[V], c[V], d[V], e[V];
    ldv<V>(cf.a, c0, a);
    ldv<V>(cf.b, c0, b);
    ldv<V>(cf.c, c0, c);
    ldv<V>(cf.d, c0, d);
    ldv<V>(cf.e, c0, e);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      float xh = __fmul_rn(__fsub_rn(xf[i], a[i]), b[i]);
      float t = __fsub_rn(__fsub_rn(f[i], c[i]), __fmul_rn(xh, d[i]));
      f[i] = __fmul_rn(e[i], t);
    }
  }
}

// write one transformed chunk (V floats) into the operand tile: bf16 -> one plane;
// f32 -> 3xTF32 split: hi plane (tf32-exact) and lo plane (residual)
template <typename T, int V>
__device__ __forceinline__ void st_chunk(uint8_t* plane0, uint8_t* plane1, uint32_t off,
                                         const float (&f)[V]) {
  if constexpr (sizeof(T) == 2) {
    uint4 o;
    o.x = pack_bf16(f[0], f[1]); o.y = pack_bf16(f[2], f[3]);
    o.z = pack_bf16(f[4], f[5]); o.w = pack_bf16(f[6], f[7]);
    *reinterpret_cast<uint4*>(plane0 + off) = o;
  } else {
    float4 hi, lo;
    hi.x = tf32_hi(f[0]); hi.y = tf32_hi(f[1]); hi.z = tf32_hi(f[2]); hi.w = tf32_hi(f[3]);
    lo.x = tf32_rn(f[0] - hi.x); lo.y = tf32_rn(f[1] - hi.y);
    lo.z = tf32_rn(f[2] - hi.z); lo.w = tf32_rn(f[3] - hi.w);
    *reinterpret_cast<float4*>(plane0 + off) = hi;
    *reinterpret_cast<float4*>(plane1 + off) = lo;
  }
}

// byte offset of a 16B chunk in an MN-major operand tile with `krows` K rows
// and MN extent `mn_ext` elements (see sm100.cuh for the validated layouts)
template <typename T, int MN_EXT, int KROWS>
__device__ __forceinline__ uint32_t mn_off(int krow, int mn_elem) {
  const uint32_t mnbyte = mn_elem * sizeof(T);
  if constexpr (sizeof(T) == 2 && MN_EXT * 2 < 128) {  // SW64, 64B rows
    uint32_t off = krow * 64 + mnbyte;
    return off ^ (((off >> 7) & 3u) << 4);
  } else if constexpr (sizeof(T) == 2) {  // SW128
    uint32_t off = (mnbyte >> 7) * (KROWS * 128) + krow * 128 + (mnbyte & 127);
    return off ^ (((off >> 7) & 7u) << 4);
  } else {  // 128B_BASE32B (tf32 MN-major)
    uint32_t off = (mnbyte >> 7) * (KROWS * 128) + krow * 128 + (mnbyte & 127);
    return off ^ (((off >> 7) & 3u) << 5);
  }
}

template <typename T, int MN_EXT, int KROWS>
__device__ __forceinline__ uint64_t mn_desc(uint32_t base, int kk) {
  if constexpr (sizeof(T) == 2 && MN_EXT * 2 < 128) {
    return make_sdesc(base + kk * 16 * 64, KROWS * 64, 512, kLayoutSW64);
  } else if constexpr (sizeof(T) == 2) {
    return make_sdesc(base + kk * 16 * 128, KROWS * 128, 1024, kLayoutSW128);
  } else {
    return make_sdesc(base + kk * 8 * 128, KROWS * 128, 512, kLayoutSW128Base32);
  }
}

__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// butterfly transpose-reduce of 16 per-row values over a warp: afterwards even
// lane l holds the 32-row total of column l/2 (fixed order => deterministic)
template <typename A>
__device__ __forceinline__ void warp_colsum16(A (&v)[16], int lane) {
#pragma unroll
  for (int w = 8; w >= 1; w >>= 1) {
    const int off = w * 2;  // 16, 8, 4, 2
    const bool upper = lane & off;
#pragma unroll
    for (int i = 0; i < w; ++i) {
      A keep = upper ? v[i + w] : v[i];
      A send = upper ? v[i] : v[i + w];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
}

template <int MODE, int BN, typename T, bool HASX>
struct IgCfg {
  static constexpr int ESZ = sizeof(T);
  static constexpr int V = 16 / ESZ;           // elements per 16-byte chunk
  static constexpr int KB = 128 / ESZ;         // K elements per stage
  static constexpr bool F32 = ESZ == 4;
  static constexpr int PLANES = F32 ? 2 : 1;   // 3xTF32: hi / lo planes
  static constexpr int A_BYTES = 128 * 128;
  static constexpr int B_BYTES = BN * 128;
  static constexpr int X_BYTES = HASX ? (MODE == MODE_WGRAD ? B_BYTES : A_BYTES) : 0;
  static constexpr int STAGE_BYTES = PLANES * (A_BYTES + B_BYTES) + X_BYTES;
  static constexpr int BUDGET = 176 * 1024;
  static constexpr int STAGES_RAW = BUDGET / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW < 2 ? 2 : (STAGES_RAW > 8 ? 8 : STAGES_RAW);
  static constexpr int LAG = STAGES >= 4 ? STAGES - 2 : STAGES - 1;  // cp.async groups in flight
  static constexpr int TCOLS = 2 * BN;         // double-buffered fp32 accumulators
  static constexpr int B_PER = BN / 16;        // B chunks per producer thread per stage
  static constexpr int META_BYTES = 2 * STAGES * 128 * 4;
  static constexpr int SMEM_FIXED = STAGES * STAGE_BYTES + META_BYTES + 1024;
  static constexpr int THREADS = 288;          // 4 producer, 1 MMA, 4 epilogue warps
};

template <int MODE, int BN, typename T, bool HASX>
__global__ void __launch_bounds__(288, 1) igemm_kernel(const IgParams p) {
  griddep_launch();
  griddep_wait();
  using C = IgCfg<MODE, BN, T, HASX>;
  constexpr int V = C::V, KB = C::KB, STAGES = C::STAGES, LAG = C::LAG;
  extern __shared__ uint8_t dsmem_raw[];
  // offset (not integer-cast) the shared array so the compiler keeps the shared state space
  uint8_t* smem = dsmem_raw + ((1024u - (smem_u32(dsmem_raw) & 1023u)) & 1023u);
  uint32_t* meta_a = reinterpret_cast<uint32_t*>(smem + STAGES * C::STAGE_BYTES);
  uint32_t* meta_b = meta_a + STAGES * 128;
  double* sacc = reinterpret_cast<double*>(meta_b + STAGES * 128);  // [2][stat_ld], f64 across tiles
  __shared__ uint64_t full_bar[STAGES], empty_bar[STAGES], accf_bar[2], acce_bar[2];
  __shared__ uint32_t tmem_sh;
  // per-tile column sums: fp32 data in float64 (ops.py:231-237), bf16 data in fp32
  using SAcc = typename std::conditional<sizeof(T) == 4, double, float>::type;
  __shared__ SAcc red[4][2][BN];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ntl = (p.ntiles_total - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  const bool do_stats = MODE != MODE_WGRAD && p.stat_part != nullptr;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full_bar[s], 128); mbar_init(&empty_bar[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&accf_bar[s], 1); mbar_init(&acce_bar[s], 128); }
    fence_mbar_init();
  }
  if (do_stats)
    for (int i = tid; i < 2 * p.stat_ld; i += blockDim.x) sacc[i] = 0.0;
  if (warp == 4) tmem_alloc<C::TCOLS>(&tmem_sh);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_sh;

  auto stage_a = [&](int s, int plane) { return smem + s * C::STAGE_BYTES + plane * C::A_BYTES; };
  auto stage_b = [&](int s, int plane) {
    return smem + s * C::STAGE_BYTES + C::PLANES * C::A_BYTES + plane * C::B_BYTES;
  };
  auto stage_x = [&](int s) { return smem + s * C::STAGE_BYTES + C::PLANES * (C::A_BYTES + C::B_BYTES); };

  // tile index -> (m0, n0, kb0)
  auto tile_of = [&](int lt, int& m0, int& n0, int& kb0) {
    const int t = (int)blockIdx.x + lt * (int)gridDim.x;
    const int mt = t % p.mtiles;
    const int r = t / p.mtiles;
    m0 = mt * 128;
    if (MODE == MODE_WGRAD) {
      n0 = (r % p.ntiles) * BN;
      kb0 = (r / p.ntiles) * p.kpt;
    } else {
      n0 = r * BN;
      kb0 = 0;
    }
  };

  if (warp < 4) {
    // ======================= producers (cp.async) =======================
    const int G = ntl * p.kpt;
    // per-tile state
    int pbase[8], ph[8], pw[8];
    int cur_lt = -1, m0 = 0, n0 = 0, kb0 = 0;
    // WGRAD fixed per-tile operand columns
    constexpr int CPR_A = 128 / V, RSTEP_A = 128 / CPR_A;
    constexpr int CPR_B = BN / V, RSTEP_B = 128 / CPR_B;
    const int ja = tid % CPR_A, ra0 = tid / CPR_A;
    const int jb = tid % CPR_B, rb0 = tid / CPR_B;
    int a_ci = 0, a_ty = 0, a_tx = 0;
    bool a_mval = false;
    const int j = tid & 7, r0 = tid >> 3;  // K-major mapping (FPROP/DGRAD A, B weights)
    const uint32_t npix = (uint32_t)(p.n * p.oh * p.ow);
    const bool xa = HASX && MODE == MODE_DGRAD && p.a_pro == BNFF_PRO_BN_DX;
    const bool xb = HASX && MODE == MODE_WGRAD && p.b_pro == BNFF_PRO_BN_DX;
    const bool need_ta = C::F32 || p.a_pro != BNFF_PRO_NONE;
    const bool need_tb = C::F32 || (MODE == MODE_WGRAD && p.b_pro != BNFF_PRO_NONE);

    for (int g = 0; g < G + LAG; ++g) {
      if (g < G) {
        const int lt = g / p.kpt, kk = g - lt * p.kpt;
        const int s = g % STAGES;
        if (lt != cur_lt) {
          cur_lt = lt;
          tile_of(lt, m0, n0, kb0);
          if constexpr (MODE != MODE_WGRAD) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int m = m0 + r0 + 16 * i;
              if (m < p.M) {
                if constexpr (MODE == MODE_FPROP) {
                  const uint32_t img = fdiv(m, p.fd_ohow), rem = m - img * (p.oh * p.ow);
                  const uint32_t oy = fdiv(rem, p.fd_ow), ox = rem - oy * p.ow;
                  pbase[i] = img * p.h * p.w;
                  ph[i] = oy * p.stride - p.pad;
                  pw[i] = ox * p.stride - p.pad;
                } else {
                  const uint32_t img = fdiv(m, p.fd_hw), rem = m - img * (p.h * p.w);
                  const uint32_t y = fdiv(rem, p.fd_w), x = rem - y * p.w;
                  pbase[i] = img * p.oh * p.ow;
                  ph[i] = y + p.pad;
                  pw[i] = x + p.pad;
                }
              } else {
                pbase[i] = -1; ph[i] = 0; pw[i] = 0;
              }
            }
          } else {
            const int midx = m0 + ja * V;
            a_mval = midx < p.M;
            const int tap = fdiv(midx, p.fd_cin);
            a_ci = midx - tap * p.cin;
            a_ty = fdiv(tap, p.fd_kw);
            a_tx = tap - a_ty * p.kw;
          }
        }
        if (g >= STAGES) mbar_wait(&empty_bar[s], ((g / STAGES) - 1) & 1);
        const int kb = kb0 + kk;
        const uint32_t abase = smem_u32(stage_a(s, 0)), bbase = smem_u32(stage_b(s, 0));
        const uint32_t xbase = smem_u32(stage_x(s));
        if constexpr (MODE != MODE_WGRAD) {
          const int kidx = kb * KB + j * V;
          const int tap = fdiv(kidx, p.fd_kred), cc = kidx - tap * p.kred;
          const int ty = fdiv(tap, p.fd_kw), tx = tap - ty * p.kw;
          const bool kval = tap < p.taps;
          uint32_t mask = 0;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            bool ok = kval && pbase[i] >= 0;
            long long pix = 0;
            if constexpr (MODE == MODE_FPROP) {
              const int iy = ph[i] + ty, ix = pw[i] + tx;
              ok = ok && iy >= 0 && iy < p.h && ix >= 0 && ix < p.w;
              pix = (long long)pbase[i] + (long long)iy * p.w + ix;
            } else {
              int ay = ph[i] - ty, ax = pw[i] - tx;
              if (p.stride > 1) {
                ok = ok && ay >= 0 && ax >= 0 && (ay % p.stride) == 0 && (ax % p.stride) == 0;
                ay /= p.stride;
                ax /= p.stride;
              }
              ok = ok && ay >= 0 && ay < p.oh && ax >= 0 && ax < p.ow;
              pix = (long long)pbase[i] + (long long)ay * p.ow + ax;
            }
            const uint32_t off = kmajor_sw128_off(r0 + 16 * i, j * 16);
            const T* src = reinterpret_cast<const T*>(p.a_ptr) + (ok ? pix * p.a_rs + cc : 0);
            cp_async16(abase + off, src, ok ? 16u : 0u);
            if (xa) {
              const T* xs = reinterpret_cast<const T*>(p.a_xptr) + (ok ? pix * p.a_xrs + cc : 0);
              cp_async16(xbase + off, xs, ok ? 16u : 0u);
            }
            mask |= (ok ? 1u : 0u) << i;
          }
          meta_a[s * 128 + tid] = ((uint32_t)cc << 8) | mask;
#pragma unroll
          for (int i = 0; i < C::B_PER; ++i) {
            const int row = n0 + r0 + 16 * i;
            const bool ok = row < p.N;
            const T* src = reinterpret_cast<const T*>(p.b_ptr) +
                           (ok ? (long long)row * p.b_rs + kb * KB + j * V : 0);
            cp_async16(bbase + kmajor_sw128_off(r0 + 16 * i, j * 16), src, ok ? 16u : 0u);
          }
        } else {
          uint32_t mask = 0;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint32_t pix = (uint32_t)(kb * KB + ra0 + RSTEP_A * i);
            bool ok = a_mval && pix < npix && kb < p.nkb;
            long long src = 0;
            if (ok) {
              const uint32_t img = fdiv(pix, p.fd_ohow), rem = pix - img * (p.oh * p.ow);
              const uint32_t oy = fdiv(rem, p.fd_ow), ox = rem - oy * p.ow;
              const int iy = (int)oy * p.stride - p.pad + a_ty, ix = (int)ox * p.stride - p.pad + a_tx;
              ok = iy >= 0 && iy < p.h && ix >= 0 && ix < p.w;
              src = ((long long)img * p.h + iy) * p.w + ix;
            }
            const T* sp = reinterpret_cast<const T*>(p.a_ptr) + (ok ? src * p.a_rs + a_ci : 0);
            cp_async16(abase + mn_off<T, 128, KB>(ra0 + RSTEP_A * i, ja * V), sp, ok ? 16u : 0u);
            mask |= (ok ? 1u : 0u) << i;
          }
          meta_a[s * 128 + tid] = ((uint32_t)a_ci << 8) | mask;
          const int co = n0 + jb * V;
          uint32_t maskb = 0;
#pragma unroll
          for (int i = 0; i < C::B_PER; ++i) {
            const uint32_t pix = (uint32_t)(kb * KB + rb0 + RSTEP_B * i);
            const bool ok = co < p.N && pix < npix && kb < p.nkb;
            const uint32_t off = mn_off<T, BN, KB>(rb0 + RSTEP_B * i, jb * V);
            const T* sp = reinterpret_cast<const T*>(p.b_ptr) + (ok ? (long long)pix * p.b_rs + co : 0);
            cp_async16(bbase + off, sp, ok ? 16u : 0u);
            if (xb) {
              const T* xs = reinterpret_cast<const T*>(p.b_xptr) + (ok ? (long long)pix * p.b_xrs + co : 0);
              cp_async16(xbase + off, xs, ok ? 16u : 0u);
            }
            maskb |= (ok ? 1u : 0u) << i;
          }
          meta_b[s * 128 + tid] = ((uint32_t)co << 16) | maskb;  // mask: B_PER <= 16 bits
        }
      }
      cp_async_commit();
      if (g >= LAG) {
        const int gg = g - LAG;
        const int s2 = gg % STAGES;
        cp_async_wait<LAG>();
        if (need_ta) {
          const uint32_t ma = meta_a[s2 * 128 + tid];
          const int cc = (int)(ma >> 8);
          uint8_t* a0 = stage_a(s2, 0);
          uint8_t* a1 = stage_a(s2, 1);
          uint8_t* xs = stage_x(s2);
          ProCoef<V> pca;
          if (ma & 0xFFu) pca.load(p.a_pro, cc, p.a_coef);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            uint32_t off;
            if constexpr (MODE == MODE_WGRAD) off = mn_off<T, 128, KB>(ra0 + RSTEP_A * i, ja * V);
            else off = kmajor_sw128_off(r0 + 16 * i, j * 16);
            Chunk<T> ch, cx;
            ch.raw = *reinterpret_cast<const decltype(ch.raw)*>(a0 + off);
            float f[V], xf[V];
            ch.to_float(f);
            if (xa) {
              cx.raw = *reinterpret_cast<const decltype(cx.raw)*>(xs + off);
              cx.to_float(xf);
            }
            if ((ma >> i) & 1u) pca.apply(p.a_pro, f, xf);
            st_chunk<T, V>(a0, a1, off, f);
          }
        }
        if (need_tb) {
          uint8_t* b0 = stage_b(s2, 0);
          uint8_t* b1 = stage_b(s2, 1);
          uint8_t* xs = stage_x(s2);
          const uint32_t mb = MODE == MODE_WGRAD ? meta_b[s2 * 128 + tid] : 0u;
          const int co = (int)(mb >> 16);
          ProCoef<V> pcb;
          if (MODE == MODE_WGRAD && (mb & 0xFFFFu)) pcb.load(p.b_pro, co, p.b_coef);
#pragma unroll
          for (int i = 0; i < C::B_PER; ++i) {
            uint32_t off;
            if constexpr (MODE == MODE_WGRAD) off = mn_off<T, BN, KB>(rb0 + RSTEP_B * i, jb * V);
            else off = kmajor_sw128_off(r0 + 16 * i, j * 16);
            Chunk<T> ch, cx;
            ch.raw = *reinterpret_cast<const decltype(ch.raw)*>(b0 + off);
            float f[V], xf[V];
            ch.to_float(f);
            if (MODE == MODE_WGRAD && ((mb >> i) & 1u)) {
              if (xb) {
                cx.raw = *reinterpret_cast<const decltype(cx.raw)*>(xs + off);
                cx.to_float(xf);
              }
              pcb.apply(p.b_pro, f, xf);
            }
            st_chunk<T, V>(b0, b1, off, f);
          }
        }
        fence_proxy_async_smem();
        mbar_arrive(&full_bar[s2]);
      }
    }
  } else if (warp == 4) {
    // ======================= MMA issuer =======================
    if (lane == 0) {
      constexpr uint32_t fmt = C::F32 ? kFmtTF32 : kFmtBF16;
      constexpr uint32_t mn = MODE == MODE_WGRAD ? 1u : 0u;
      constexpr uint32_t idesc = make_idesc(128, BN, fmt, mn, mn);
      int g = 0;
      for (int lt = 0; lt < ntl; ++lt) {
        const int slot = lt & 1;
        if (lt >= 2) mbar_wait(&acce_bar[slot], ((lt >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t dt = tmem + slot * BN;
        for (int kk = 0; kk < p.kpt; ++kk, ++g) {
          const int s = g % STAGES;
          mbar_wait(&full_bar[s], (g / STAGES) & 1);
          tc_fence_after();
          const uint32_t a0 = smem_u32(stage_a(s, 0)), b0 = smem_u32(stage_b(s, 0));
          const uint32_t a1 = smem_u32(stage_a(s, 1)), b1 = smem_u32(stage_b(s, 1));
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint64_t ad0, bd0, ad1, bd1;
            if constexpr (MODE == MODE_WGRAD) {
              ad0 = mn_desc<T, 128, KB>(a0, q);
              bd0 = mn_desc<T, BN, KB>(b0, q);
              ad1 = mn_desc<T, 128, KB>(a1, q);
              bd1 = mn_desc<T, BN, KB>(b1, q);
            } else {
              ad0 = make_sdesc(a0 + q * 32, 16, 1024, kLayoutSW128);
              bd0 = make_sdesc(b0 + q * 32, 16, 1024, kLayoutSW128);
              ad1 = make_sdesc(a1 + q * 32, 16, 1024, kLayoutSW128);
              bd1 = make_sdesc(b1 + q * 32, 16, 1024, kLayoutSW128);
            }
            const uint32_t acc = (kk > 0 || q > 0) ? 1u : 0u;
            if constexpr (C::F32) {
              if (p.tf32_mode == 2) {  // the two cross terms first, then hi*hi
                umma_tf32(dt, ad0, bd1, idesc, acc);
                umma_tf32(dt, ad1, bd0, idesc, 1u);
                umma_tf32(dt, ad0, bd0, idesc, 1u);
              } else {
                umma_tf32(dt, ad0, bd0, idesc, acc);
                umma_tf32(dt, ad0, bd1, idesc, 1u);
                umma_tf32(dt, ad1, bd0, idesc, 1u);
                if (p.tf32_mode == 1) umma_tf32(dt, ad1, bd1, idesc, 1u);  // + lo*lo
              }
            } else {
              umma_f16(dt, ad0, bd0, idesc, acc);
            }
          }
          umma_commit(&empty_bar[s]);
        }
        umma_commit(&accf_bar[slot]);
      }
    }
    __syncwarp();
  } else {
    // ======================= epilogue (warps 5-8) =======================
    const int ew = warp - 5;          // epilogue warp index 0..3
    const int quad = warp & 3;        // TMEM lane quadrant this warp may access
    const int et = tid - 160;         // 0..127
    for (int lt = 0; lt < ntl; ++lt) {
      const int slot = lt & 1;
      int m0, n0, kb0;
      tile_of(lt, m0, n0, kb0);
      mbar_wait(&accf_bar[slot], (lt >> 1) & 1);
      tc_fence_after();
      const int row = quad * 32 + lane;
      const int gm = m0 + row;
      const bool rval = gm < p.M;
      const uint32_t tbase = tmem + slot * BN + ((uint32_t)(quad * 32) << 16);
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        float v[16];
        tmem_ld16(tbase + c0, v);
        tmem_ld_wait();
        const int gc0 = n0 + c0;
        if constexpr (MODE == MODE_WGRAD) {
          if (rval) {
            const int split = kb0 / p.kpt;
            float* dst = reinterpret_cast<float*>(p.c_ptr) +
                         ((long long)split * p.M + gm) * (long long)p.c_rs + gc0;
#pragma unroll
            for (int q = 0; q < 16; q += 4)
              if (gc0 + q < p.N)
                *reinterpret_cast<float4*>(dst + q) = make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
          }
        } else {
          SAcc s1[16], s2[16];
          float xv[16];
          const bool need_x = MODE == MODE_DGRAD && p.epi != BNFF_DG_PLAIN;
          if (need_x) {
#pragma unroll
            for (int q = 0; q < 16; q += V) {
              Chunk<T> ch;
              if (rval && gc0 + q < p.N)
                ch.load(reinterpret_cast<const T*>(p.e_xptr) + (long long)gm * p.e_xrs + gc0 + q);
              else
                ch.zero();
              float f[V];
              ch.to_float(f);
#pragma unroll
              for (int u = 0; u < V; ++u) xv[q + u] = f[u];
            }
          }
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const int gc = gc0 + q;
            const bool cval = gc < p.N;
            float val = v[q];
            if constexpr (MODE == MODE_FPROP) {
              if (p.bias != nullptr && cval) val = __fadd_rn(val, __ldg(p.bias + gc));
            } else {
              if (p.epi == BNFF_DG_CLIP) {
                val = xv[q] > 0.f ? val : 0.f;
              } else if (p.epi == BNFF_DG_NRC && cval) {
                float t = __fmul_rn(__fsub_rn(xv[q], __ldg(p.e_coef.a + gc)), __ldg(p.e_coef.b + gc));
                t = __fadd_rn(t, __ldg(p.e_coef.c + gc));
                val = t > 0.f ? val : 0.f;
              }
            }
            float r;
            if constexpr (sizeof(T) == 2) r = __bfloat162float(__float2bfloat16_rn(val));
            else r = val;
            v[q] = r;
            const bool sv = rval && cval;
            if constexpr (MODE == MODE_FPROP) {
              s1[q] = sv ? (SAcc)r : SAcc(0);
              s2[q] = sv ? (SAcc)r * (SAcc)r : SAcc(0);
            } else {
              float xh = 0.f;
              if (p.epi == BNFF_DG_NRC && cval)
                xh = __fmul_rn(__fsub_rn(xv[q], __ldg(p.e_coef.a + gc)), __ldg(p.e_coef.d + gc));
              s1[q] = sv ? (SAcc)r : SAcc(0);
              s2[q] = sv ? (SAcc)r * (SAcc)xh : SAcc(0);
            }
          }
          if (rval) {
            T* dst = reinterpret_cast<T*>(p.c_ptr) + (long long)gm * p.c_rs + gc0;
#pragma unroll
            for (int q = 0; q < 16; q += V) {
              if (gc0 + q < p.N) {
                if constexpr (sizeof(T) == 2) {
                  uint4 o;
                  o.x = pack_bf16(v[q], v[q + 1]); o.y = pack_bf16(v[q + 2], v[q + 3]);
                  o.z = pack_bf16(v[q + 4], v[q + 5]); o.w = pack_bf16(v[q + 6], v[q + 7]);
                  *reinterpret_cast<uint4*>(dst + q) = o;
                } else {
                  *reinterpret_cast<float4*>(dst + q) = make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
                }
              }
            }
          }
          if (do_stats) {
            warp_colsum16(s1, lane);
            warp_colsum16(s2, lane);
            if ((lane & 1) == 0) {
              red[ew][0][c0 + (lane >> 1)] = s1[0];
              red[ew][1][c0 + (lane >> 1)] = s2[0];
            }
          }
        }
      }
      // accumulator slot drained -> MMA may reuse it
      tc_fence_before();
      mbar_arrive(&acce_bar[slot]);
      if (do_stats) {
        named_bar(1, 128);
        for (int c = et; c < BN; c += 128) {
          const int gc = n0 + c;
          if (gc < p.N) {
            sacc[gc] += (double)red[0][0][c] + (double)red[1][0][c] + (double)red[2][0][c] + (double)red[3][0][c];
            sacc[p.stat_ld + gc] += (double)red[0][1][c] + (double)red[1][1][c] + (double)red[2][1][c] + (double)red[3][1][c];
          }
        }
        named_bar(2, 128);
      }
    }
    if (do_stats) {
      // one partial row per CTA (fixed tile->CTA assignment => deterministic)
      for (int c = et; c < p.stat_ld; c += 128) {
        p.stat_part[((long long)blockIdx.x * 2 + 0) * p.stat_ld + c] = sacc[c];
        p.stat_part[((long long)blockIdx.x * 2 + 1) * p.stat_ld + c] = sacc[p.stat_ld + c];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) tmem_dealloc<C::TCOLS>(tmem);
}

// ---------------------------------------------------------------------------
// launch helpers
// ---------------------------------------------------------------------------
static int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
  }
  return n;
}

template <int MODE, int BN, typename T, bool HASX>
static int launch_ig(IgParams p, cudaStream_t st) {
  using C = IgCfg<MODE, BN, T, HASX>;
  auto kern = igemm_kernel<MODE, BN, T, HASX>;
  const int smem = C::SMEM_FIXED + (MODE != MODE_WGRAD && p.stat_part ? 2 * p.stat_ld * 8 : 0);
  static int attr_smem = 0;  // per instantiation
  if (smem > attr_smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(igemm)");
    attr_smem = smem;
  }
  p.mtiles = (p.M + 127) / 128;
  p.ntiles = (p.N + BN - 1) / BN;
  p.ntiles_total = p.mtiles * p.ntiles * p.splits;
  p.fd_kred = make_fastdiv(p.kred > 0 ? p.kred : 1);
  p.fd_kw = make_fastdiv(p.kw);
  p.fd_ohow = make_fastdiv(p.oh * p.ow);
  p.fd_ow = make_fastdiv(p.ow);
  p.fd_hw = make_fastdiv(p.h * p.w);
  p.fd_w = make_fastdiv(p.w);
  p.fd_cin = make_fastdiv(p.cin);
  p.taps = p.kh * p.kw;
  static int tf32_mode = -1;
  if (tf32_mode < 0) {
    const char* e = getenv("BNFF_TF32_MODE");
    tf32_mode = e ? atoi(e) : 0;
  }
  p.tf32_mode = tf32_mode;
  const int grid = p.ntiles_total < num_sms() ? p.ntiles_total : num_sms();
  launch(kern, dim3(grid), dim3(C::THREADS), smem, st, p);
  return check_launch("igemm");
}

template <int MODE, typename T, bool HASX>
static int dispatch_bn(const IgParams& p, int bn, cudaStream_t st) {
  switch (bn) {
    case 32: return launch_ig<MODE, 32, T, HASX>(p, st);
    case 64: return launch_ig<MODE, 64, T, HASX>(p, st);
    case 128: return launch_ig<MODE, 128, T, HASX>(p, st);
    default: return launch_ig<MODE, 256, T, HASX>(p, st);
  }
}

template <int MODE>
static int dispatch(int dtype, const IgParams& p, int bn, bool hasx, cudaStream_t st) {
  // fp32: hi/lo operand planes, float64 statistics -- a 256-wide N tile does not fit two stages
  if (dtype != BNFF_BF16 && bn > 128) bn = 128;
  if (dtype == BNFF_BF16) {
    if (MODE != MODE_FPROP && hasx) return dispatch_bn<MODE, __nv_bfloat16, true>(p, bn, st);
    return dispatch_bn<MODE, __nv_bfloat16, false>(p, bn, st);
  }
  // 3xTF32 stages carry hi/lo planes: a 256-wide B tile plus the x tile of a deferred-dx
  // prologue would not fit two stages in shared memory, so those run as 128-wide N tiles
  if (MODE != MODE_FPROP && hasx) return dispatch_bn<MODE, float, true>(p, bn > 128 ? 128 : bn, st);
  return dispatch_bn<MODE, float, false>(p, bn, st);
}

static int pick_bn(int n) {
  if (n <= 32) return 32;
  if (n <= 64) return 64;
  if (n <= 128) return 128;
  return 256;
}

}  // namespace bnff

using namespace bnff;

// K index padding for packed weights: multiple of one stage (64 bf16 / 32 f32)
static inline int kpad_elems(int dtype, int k) {
  const int kb = dtype == BNFF_BF16 ? 64 : 32;
  return (k + kb - 1) / kb * kb;
}

static constexpr int kWindowNoFitAbi = -100;  // wconv.cu: shape does not fit its smem plan

static int check_common(int dtype, const bnff_view& v, const char* what) {
  const int vec = dtype == BNFF_BF16 ? 8 : 4;
  if (dtype != BNFF_BF16 && dtype != BNFF_F32) return set_error(BNFF_ERR_UNSUPPORTED, "dtype %d", dtype);
  if (v.ptr == nullptr) return set_error(BNFF_ERR_STATE, "%s: null pointer", what);
  if (v.c % vec != 0 || v.row_stride % vec != 0)
    return set_error(BNFF_ERR_UNSUPPORTED, "%s: channels (%lld) and row stride (%lld) must be multiples of %d",
                     what, (long long)v.c, (long long)v.row_stride, vec);
  if ((reinterpret_cast<uintptr_t>(v.ptr) & 15) != 0)
    return set_error(BNFF_ERR_UNSUPPORTED, "%s: base pointer not 16B aligned", what);
  return BNFF_OK;
}

extern "C" int bnff_conv_fprop(const bnff_fprop_args* a, void* stream) {
  int rc;
  if ((rc = check_common(a->dtype, a->x, "fprop x"))) return rc;
  if ((rc = check_common(a->dtype, a->y, "fprop y"))) return rc;
  IgParams p{};
  p.n = (int)a->x.n; p.h = (int)a->x.h; p.w = (int)a->x.w; p.cin = (int)a->x.c;
  p.kh = a->kh; p.kw = a->kw; p.stride = a->stride; p.pad = a->pad;
  p.oh = (p.h + 2 * p.pad - p.kh) / p.stride + 1;
  p.ow = (p.w + 2 * p.pad - p.kw) / p.stride + 1;
  p.cout = (int)a->y.c;
  if (a->y.n != a->x.n || a->y.h != p.oh || a->y.w != p.ow)
    return set_error(BNFF_ERR_SHAPE, "fprop: y dims (%lld,%lld,%lld) != (%d,%d,%d)", (long long)a->y.n,
                     (long long)a->y.h, (long long)a->y.w, p.n, p.oh, p.ow);
  if (a->x_pro == BNFF_PRO_BN_DX) return set_error(BNFF_ERR_UNSUPPORTED, "fprop: BN_DX prologue");
  if (a->x_pro == BNFF_PRO_BN_RELU && (!a->x_coef.a || !a->x_coef.b || !a->x_coef.c))
    return set_error(BNFF_ERR_STATE, "fprop: missing statistics for the normalize prologue");
  if (a->wwin && bnff_window_ok_ex(a->dtype, (int)a->x.c, p.cout, p.kh, p.kw, p.stride, p.pad, p.h, p.w,
                                    a->x_pro != BNFF_PRO_NONE ? BNFF_WT_FPROP_PRO : 0)) {
    bnff_view none{};
    const int wrc = bnff_window_conv(a->dtype, 0, p.kh, p.pad, a->x, none, a->x_pro, a->x_coef, a->y, a->wwin,
                                     a->bias, 0, none, bnff_coef{}, a->stat_part, stream);
    if (wrc != kWindowNoFitAbi) return wrc;
  }
  p.M = p.n * p.oh * p.ow;
  p.N = p.cout;
  p.kred = p.cin;
  const int K = p.kh * p.kw * p.cin;
  const int kb = a->dtype == BNFF_BF16 ? 64 : 32;
  p.nkb = (K + kb - 1) / kb;
  p.kpt = p.nkb;
  p.splits = 1;
  p.a_ptr = a->x.ptr; p.a_rs = a->x.row_stride; p.a_pro = a->x_pro; p.a_coef = a->x_coef;
  if (!a->wpack)  // window-only weights and the window plan rejected the launch: never run stale packs
    return set_error(BNFF_ERR_STATE, "fprop: window kernel not eligible and no generic packed weights");
  p.b_ptr = a->wpack; p.b_rs = kpad_elems(a->dtype, K);
  p.c_ptr = a->y.ptr; p.c_rs = a->y.row_stride;
  p.bias = a->bias;
  p.stat_part = a->stat_part;
  p.stat_ld = p.cout;
  return dispatch<MODE_FPROP>(a->dtype, p, pick_bn(p.N), false, (cudaStream_t)stream);
}

extern "C" int bnff_conv_dgrad(const bnff_dgrad_args* a, void* stream) {
  int rc;
  if ((rc = check_common(a->dtype, a->dy, "dgrad dy"))) return rc;
  if ((rc = check_common(a->dtype, a->dx, "dgrad dx"))) return rc;
  IgParams p{};
  p.n = (int)a->dx.n; p.h = (int)a->dx.h; p.w = (int)a->dx.w; p.cin = (int)a->dx.c;
  p.kh = a->kh; p.kw = a->kw; p.stride = a->stride; p.pad = a->pad;
  p.oh = (int)a->dy.h; p.ow = (int)a->dy.w; p.cout = (int)a->dy.c;
  if ((p.h + 2 * p.pad - p.kh) / p.stride + 1 != p.oh || (p.w + 2 * p.pad - p.kw) / p.stride + 1 != p.ow)
    return set_error(BNFF_ERR_SHAPE, "dgrad: dy spatial dims inconsistent with dx");
  if (a->dy_pro == BNFF_PRO_BN_DX && (rc = check_common(a->dtype, a->dy_x, "dgrad dy_x"))) return rc;
  if (a->epi != BNFF_DG_PLAIN && (rc = check_common(a->dtype, a->x, "dgrad x"))) return rc;
  const bool fold = a->epi == BNFF_DG_NRC_ACC || a->epi == BNFF_DG_NRC_SET;
  if (a->epi < BNFF_DG_PLAIN || a->epi > BNFF_DG_NRC_SET) return set_error(BNFF_ERR_SHAPE, "dgrad: bad epilogue");
  if (a->wwin && bnff_window_ok_ex(a->dtype, p.cin, p.cout, p.kh, p.kw, p.stride, p.pad, p.h, p.w,
                                    (a->dy_pro != BNFF_PRO_NONE ? BNFF_WT_DGRAD_PRO : 0) |
                                        (a->epi >= BNFF_DG_NRC ? BNFF_WT_DGRAD_NRC : 0))) {
    if (a->dy_pro == BNFF_PRO_BN_DX && (!a->dy_coef.a || !a->dy_coef.e))
      return set_error(BNFF_ERR_STATE, "dgrad: missing deferred-gradient coefficients");
    const int wrc = bnff_window_conv(a->dtype, 1, p.kh, p.pad, a->dy, a->dy_x, a->dy_pro, a->dy_coef, a->dx,
                                     a->wwin, nullptr, a->epi, a->x, a->x_coef,
                                     a->epi >= BNFF_DG_NRC ? a->stat_part : nullptr, stream);
    if (wrc != kWindowNoFitAbi) return wrc;
  }
  if (fold) return set_error(BNFF_ERR_UNSUPPORTED, "dgrad: the block-gradient fold needs the window kernel");
  p.M = p.n * p.h * p.w;
  p.N = p.cin;
  p.kred = p.cout;
  const int K = p.kh * p.kw * p.cout;
  const int kb = a->dtype == BNFF_BF16 ? 64 : 32;
  p.nkb = (K + kb - 1) / kb;
  p.kpt = p.nkb;
  p.splits = 1;
  p.a_ptr = a->dy.ptr; p.a_rs = a->dy.row_stride; p.a_pro = a->dy_pro; p.a_coef = a->dy_coef;
  p.a_xptr = a->dy_x.ptr; p.a_xrs = a->dy_x.row_stride;
  if (!a->wpack_t)
    return set_error(BNFF_ERR_STATE, "dgrad: window kernel not eligible and no generic packed weights");
  p.b_ptr = a->wpack_t; p.b_rs = kpad_elems(a->dtype, K);
  p.c_ptr = a->dx.ptr; p.c_rs = a->dx.row_stride;
  p.epi = a->epi;
  p.e_xptr = a->x.ptr; p.e_xrs = a->x.row_stride; p.e_coef = a->x_coef;
  p.stat_part = a->epi == BNFF_DG_NRC ? a->stat_part : nullptr;
  p.stat_ld = p.cin;
  return dispatch<MODE_DGRAD>(a->dtype, p, pick_bn(p.N), a->dy_pro == BNFF_PRO_BN_DX,
                              (cudaStream_t)stream);
}

extern "C" int32_t bnff_stat_rows(void) { return num_sms(); }

extern "C" int32_t bnff_wgrad_default_splits(int32_t n, int32_t oh, int32_t ow, int32_t kh,
                                             int32_t kw, int32_t c_in, int32_t c_out) {
  const long long npix = (long long)n * oh * ow;
  const int nkb = (int)((npix + 63) / 64);
  const int tiles = ((kh * kw * c_in + 127) / 128) * ((c_out + pick_bn(c_out) - 1) / pick_bn(c_out));
  int splits = (num_sms() + tiles - 1) / tiles;
  const int max_splits = nkb / 8 > 0 ? nkb / 8 : 1;  // >= 8 k-blocks per split
  if (splits > max_splits) splits = max_splits;
  if (splits < 1) splits = 1;
  return splits;
}

extern "C" int64_t bnff_wgrad_workspace(int32_t n, int32_t oh, int32_t ow, int32_t kh, int32_t kw,
                                        int32_t c_in, int32_t c_out, int32_t splits) {
  if (splits <= 0) splits = bnff_wgrad_default_splits(n, oh, ow, kh, kw, c_in, c_out);
  const long long npix = (long long)n * oh * ow;
  // split-K partial tiles + dbias channel partials [tiles][2][c_out]
  long long part = (long long)splits * kh * kw * c_in * c_out;
  if (kh == kw && (kh == 1 || kh == 3)) {  // the window kernels may plan more splits (stride 1: oh = h)
    const long long wwin = bnff_window_wgrad_ws(n, oh, ow, kh, c_in, c_out);
    if (wwin > part) part = wwin;
    const long long w32 = bnff_wgrad_f32_ws(n, oh, ow, kh, c_in, c_out);
    if (w32 > part) part = w32;
  }
  // + 1: the dbias partials are float64, 8-byte aligned after the split-K partials
  return (int64_t)part + 1 + (int64_t)bnff_sum_tiles(npix) * 2 * c_out * 2;
}

namespace bnff {
// dW[co][ci][ky][kx] = sum_s ws[s][(tap*cin + ci)][co]   (fixed split order)
__global__ void wgrad_reduce_kernel(const float* __restrict__ ws, int splits, int M, int N, int cin,
                                    int cin_real, int taps, float* __restrict__ dw) {
  griddep_launch();
  griddep_wait();
  const long long total = (long long)M * N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int co = (int)(i % N);
    const int m = (int)(i / N);
    float acc = 0.f;
    for (int s = 0; s < splits; ++s) acc += ws[((long long)s * M + m) * N + co];
    const int tap = m / cin, ci = m - tap * cin;
    if (ci < cin_real) dw[((long long)co * cin_real + ci) * taps + tap] = acc;
  }
}
}  // namespace bnff

extern "C" int bnff_conv_wgrad(const bnff_wgrad_args* a, void* stream) {
  int rc;
  if ((rc = check_common(a->dtype, a->x, "wgrad x"))) return rc;
  if ((rc = check_common(a->dtype, a->dy, "wgrad dy"))) return rc;
  if (a->dy_pro == BNFF_PRO_BN_DX && (rc = check_common(a->dtype, a->dy_x, "wgrad dy_x"))) return rc;
  if (a->workspace == nullptr || a->dw == nullptr) return set_error(BNFF_ERR_STATE, "wgrad: null output");
  IgParams p{};
  p.n = (int)a->x.n; p.h = (int)a->x.h; p.w = (int)a->x.w; p.cin = (int)a->x.c;
  p.kh = a->kh; p.kw = a->kw; p.stride = a->stride; p.pad = a->pad;
  p.oh = (int)a->dy.h; p.ow = (int)a->dy.w; p.cout = (int)a->dy.c;
  if ((p.h + 2 * p.pad - p.kh) / p.stride + 1 != p.oh || (p.w + 2 * p.pad - p.kw) / p.stride + 1 != p.ow)
    return set_error(BNFF_ERR_SHAPE, "wgrad: dy spatial dims inconsistent with x");
  // (the window wgrad plans its own shared memory and reports a no-fit: shape class only)
  if (a->splits >= 0 && a->dtype == BNFF_BF16 &&
      bnff_window_ok_ex(a->dtype, p.cin, p.cout, p.kh, p.kw, p.stride, p.pad, p.h, p.w, 0)) {
    // window-shift kernel (splits < 0 forces the generic path)
    int rc2 = bnff_window_wgrad(a->x, a->x_pro, a->x_coef, a->dy, a->dy_x, a->dy_pro, a->dy_coef, p.kh,
                                a->workspace, a->dw, a->dw_cin, a->dbias, stream);
    if (rc2 == kWindowNoFitAbi) goto generic;
    return rc2;
  }
  if (a->splits >= 0 && a->dtype == BNFF_F32 && p.stride == 1 && p.kh == p.kw && (p.kh == 1 || p.kh == 3) &&
      p.pad == p.kh / 2) {
    // fp32: TMA tap-box wgrad (wgrad32.cu), then the fixed-order split reduction
    int splits = 0;
    const int rc3 = bnff_wgrad_f32_partials(a->x, a->x_pro, a->x_coef, a->dy, a->dy_x, a->dy_pro, a->dy_coef, p.kh,
                                            a->workspace, a->dbias != nullptr, &splits, stream);
    if (rc3 != kWindowNoFitAbi) {
      if (rc3) return rc3;
      const float* wsb = a->workspace + (long long)splits * p.kh * p.kw * p.cin * p.cout;
      return bnff_wgrad_reduce(a->workspace, splits, p.kh * p.kw, p.cin, p.cout, a->dw_cin, a->dw,
                               a->dbias ? wsb : nullptr, a->dbias, stream);
    }
  }
generic:
  const int taps = p.kh * p.kw;
  p.M = taps * p.cin;
  p.N = p.cout;
  const int kb = a->dtype == BNFF_BF16 ? 64 : 32;
  const long long npix = (long long)p.n * p.oh * p.ow;
  p.nkb = (int)((npix + kb - 1) / kb);
  int splits = a->splits > 0 ? a->splits
                             : bnff_wgrad_default_splits(p.n, p.oh, p.ow, p.kh, p.kw, p.cin, p.cout);
  if (splits > p.nkb) splits = p.nkb;
  p.kpt = (p.nkb + splits - 1) / splits;
  splits = (p.nkb + p.kpt - 1) / p.kpt;  // no empty splits (the last may be partial)
  p.splits = splits;
  p.a_ptr = a->x.ptr; p.a_rs = a->x.row_stride; p.a_pro = a->x_pro; p.a_coef = a->x_coef;
  p.b_ptr = a->dy.ptr; p.b_rs = a->dy.row_stride; p.b_pro = a->dy_pro; p.b_coef = a->dy_coef;
  p.b_xptr = a->dy_x.ptr; p.b_xrs = a->dy_x.row_stride;
  p.c_ptr = a->workspace; p.c_rs = p.N;
  cudaStream_t st = (cudaStream_t)stream;
  rc = dispatch<MODE_WGRAD>(a->dtype, p, pick_bn(p.N), a->dy_pro == BNFF_PRO_BN_DX, st);
  if (rc) return rc;
  const long long total = (long long)p.M * p.N;
  const int blocks = (int)((total + 255) / 256 < 148 * 8 ? (total + 255) / 256 : 148 * 8);
  const int cin_real = a->dw_cin > 0 ? a->dw_cin : p.cin;
  launch(wgrad_reduce_kernel, dim3(blocks), dim3(256), 0, st, a->workspace, splits, p.M, p.N, p.cin, cin_real, taps,
                                               a->dw);
  rc = check_launch("wgrad_reduce");
  if (rc) return rc;
  if (a->dbias != nullptr) {
    double* scratch = reinterpret_cast<double*>(a->workspace + (((long long)splits * p.M * p.N + 1) & ~1LL));
    return bnff_dbias_scratch(a->dtype, a->dy, a->dy_x, a->dy_pro, a->dy_coef, scratch, a->dbias, stream);
  }
  return BNFF_OK;
}
