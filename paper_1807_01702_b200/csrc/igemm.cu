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
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "sm100.cuh"
#include "common.cuh"

namespace bnff {

enum { MODE_FPROP = 0, MODE_DGRAD = 1, MODE_WGRAD = 2 };

struct IgParams {
  int M, N;             // GEMM extents
  int nkb;              // total k-blocks
  int kb_per_split;     // k-blocks per split (blockIdx.z)
  // geometry (conv input h,w; output oh,ow)
  int n, h, w, cin, oh, ow, cout, kh, kw, stride, pad;
  int kred;             // reduction channel count for the K index (fprop: cin, dgrad: cout)
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
  float* stat_part;
  int stat_ld;
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
template <int V>
__device__ __forceinline__ void apply_pro(int pro, float (&f)[V], const float (&xf)[V], int c0,
                                          const bnff_coef& cf) {
  if (pro == BNFF_PRO_RELU) {
#pragma unroll
    for (int i = 0; i < V; ++i) f[i] = fmaxf(f[i], 0.f);
  } else if (pro == BNFF_PRO_BN_RELU) {
#pragma unroll
    for (int i = 0; i < V; ++i) {
      float t = __fmul_rn(__fsub_rn(f[i], __ldg(cf.a + c0 + i)), __ldg(cf.b + c0 + i));
      f[i] = fmaxf(__fadd_rn(t, __ldg(cf.c + c0 + i)), 0.f);
    }
  } else if (pro == BNFF_PRO_BN_DX) {
#pragma unroll
    for (int i = 0; i < V; ++i) {
      float xh = __fmul_rn(__fsub_rn(xf[i], __ldg(cf.a + c0 + i)), __ldg(cf.b + c0 + i));
      float t = __fsub_rn(__fsub_rn(f[i], __ldg(cf.c + c0 + i)), __fmul_rn(xh, __ldg(cf.d + c0 + i)));
      f[i] = __fmul_rn(__ldg(cf.e + c0 + i), t);
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
    lo.x = f[0] - hi.x; lo.y = f[1] - hi.y; lo.z = f[2] - hi.z; lo.w = f[3] - hi.w;
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
__device__ __forceinline__ void warp_colsum16(float (&v)[16], int lane) {
#pragma unroll
  for (int w = 8; w >= 1; w >>= 1) {
    const int off = w * 2;  // 16, 8, 4, 2
    const bool upper = lane & off;
#pragma unroll
    for (int i = 0; i < w; ++i) {
      float keep = upper ? v[i + w] : v[i];
      float send = upper ? v[i] : v[i + w];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
}

template <int MODE, int BN, typename T>
struct IgCfg {
  static constexpr int ESZ = sizeof(T);
  static constexpr int V = 16 / ESZ;           // elements per chunk
  static constexpr int KB = 128 / ESZ;         // K elements per stage
  static constexpr bool F32 = ESZ == 4;
  static constexpr int PLANES = F32 ? 2 : 1;
  static constexpr int A_BYTES = 128 * 128;
  static constexpr int B_BYTES = BN * 128;
  static constexpr int STAGE_BYTES = PLANES * (A_BYTES + B_BYTES);
  static constexpr int BUDGET = (F32 ? 200 : 100) * 1024;
  static constexpr int STAGES_RAW = BUDGET / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW < 2 ? 2 : (STAGES_RAW > 4 ? 4 : STAGES_RAW);
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024;
  static constexpr int TCOLS = BN < 32 ? 32 : BN;
  static constexpr int B_PER = BN / 16;        // B chunks per producer thread
};

template <int MODE, int BN, typename T>
__global__ void __launch_bounds__(160, 1) igemm_kernel(const IgParams p) {
  using C = IgCfg<MODE, BN, T>;
  constexpr int V = C::V, KB = C::KB, STAGES = C::STAGES;
  extern __shared__ uint8_t dsmem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsmem_raw) + 1023) &
                                             ~uintptr_t(1023));
  __shared__ uint64_t full_bar[STAGES], empty_bar[STAGES], acc_bar;
  __shared__ uint32_t tmem_sh;
  __shared__ float red[4][2][BN];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.x * 128, n0 = blockIdx.y * BN;
  const int kb0 = blockIdx.z * p.kb_per_split;
  const int kb1 = min(p.nkb, kb0 + p.kb_per_split);
  const int nk = kb1 - kb0;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full_bar[s], 128); mbar_init(&empty_bar[s], 1); }
    mbar_init(&acc_bar, 1);
    fence_mbar_init();
  }
  if (warp == 4) tmem_alloc<C::TCOLS>(&tmem_sh);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_sh;

  auto stage_a = [&](int s, int plane) { return smem + s * C::STAGE_BYTES + plane * C::A_BYTES; };
  auto stage_b = [&](int s, int plane) {
    return smem + s * C::STAGE_BYTES + C::PLANES * C::A_BYTES + plane * C::B_BYTES;
  };

  if (warp < 4) {
    // ===================== producers =====================
    const int taps = p.kh * p.kw;
    if constexpr (MODE != MODE_WGRAD) {
      // A: K-major [128 rows][128B]; thread -> chunk column j, rows r0 + 16*i
      const int j = tid & 7, r0 = tid >> 3;
      int pbase[8], ph[8], pw[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int m = m0 + r0 + 16 * i;
        if (m < p.M) {
          if constexpr (MODE == MODE_FPROP) {
            const int img = m / (p.oh * p.ow), rem = m - img * (p.oh * p.ow);
            const int oy = rem / p.ow, ox = rem - oy * p.ow;
            pbase[i] = img * p.h * p.w;
            ph[i] = oy * p.stride - p.pad;
            pw[i] = ox * p.stride - p.pad;
          } else {
            const int img = m / (p.h * p.w), rem = m - img * (p.h * p.w);
            const int y = rem / p.w, x = rem - y * p.w;
            pbase[i] = img * p.oh * p.ow;
            ph[i] = y + p.pad;
            pw[i] = x + p.pad;
          }
        } else {
          pbase[i] = -1; ph[i] = 0; pw[i] = 0;
        }
      }
      const int bj = tid & 7, br0 = tid >> 3;
      for (int it = 0; it < nk; ++it) {
        const int kb = kb0 + it, s = it % STAGES;
        // ---- gather A ----
        const int kidx = kb * KB + j * V;
        const int tap = kidx / p.kred, cc = kidx - tap * p.kred;
        const int ty = tap / p.kw, tx = tap - ty * p.kw;
        const bool kval = tap < taps;
        Chunk<T> ra[8], rx[8];
        unsigned okmask = 0;
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
          if (ok) {
            ra[i].load(reinterpret_cast<const T*>(p.a_ptr) + pix * p.a_rs + cc);
            if (p.a_pro == BNFF_PRO_BN_DX)
              rx[i].load(reinterpret_cast<const T*>(p.a_xptr) + pix * p.a_xrs + cc);
          } else {
            ra[i].zero();
            rx[i].raw = ra[i].raw;
          }
          okmask |= (ok ? 1u : 0u) << i;
        }
        // ---- gather B (packed weights, K-major rows of b_rs elements) ----
        Chunk<T> rb[C::B_PER];
#pragma unroll
        for (int i = 0; i < C::B_PER; ++i) {
          const int row = n0 + br0 + 16 * i;
          if (row < p.N)
            rb[i].load(reinterpret_cast<const T*>(p.b_ptr) + (long long)row * p.b_rs + kb * KB + bj * V);
          else
            rb[i].zero();
        }
        if (it >= STAGES) mbar_wait(&empty_bar[s], ((it / STAGES) - 1) & 1);
        uint8_t* a0 = stage_a(s, 0);
        uint8_t* a1 = stage_a(s, 1);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float f[V], xf[V];
          ra[i].to_float(f);
          if (p.a_pro == BNFF_PRO_BN_DX) rx[i].to_float(xf);
          if ((okmask >> i) & 1u) {
            apply_pro<V>(p.a_pro, f, xf, cc, p.a_coef);
          } else {
#pragma unroll
            for (int q = 0; q < V; ++q) f[q] = 0.f;
          }
          st_chunk<T, V>(a0, a1, kmajor_sw128_off(r0 + 16 * i, j * 16), f);
        }
        uint8_t* b0 = stage_b(s, 0);
        uint8_t* b1 = stage_b(s, 1);
#pragma unroll
        for (int i = 0; i < C::B_PER; ++i) {
          float f[V];
          rb[i].to_float(f);
          st_chunk<T, V>(b0, b1, kmajor_sw128_off(br0 + 16 * i, bj * 16), f);
        }
        fence_proxy_async_smem();
        mbar_arrive(&full_bar[s]);
      }
    } else {
      // ===================== WGRAD producers (MN-major) =====================
      // A: KB pixel rows x 128 (tap,ci) elements; thread -> M chunk column ja
      constexpr int CPR_A = 128 / V;            // chunks per K-row (16 bf16 / 32 f32)
      constexpr int RSTEP_A = 128 / CPR_A;      // 8 / 4
      const int ja = tid % CPR_A, ra0 = tid / CPR_A;
      const int midx = m0 + ja * V;
      const int a_tap = midx / p.cin, a_ci = midx - a_tap * p.cin;
      const int a_ty = a_tap / p.kw, a_tx = a_tap - a_ty * p.kw;
      const bool a_mval = midx < p.M;
      constexpr int CPR_B = BN / V;
      constexpr int RSTEP_B = 128 / CPR_B;
      const int jb = tid % CPR_B, rb0 = tid / CPR_B;
      const int co = n0 + jb * V;
      const bool b_nval = co < p.N;
      const int npix = p.n * p.oh * p.ow;
      for (int it = 0; it < nk; ++it) {
        const int kb = kb0 + it, s = it % STAGES;
        Chunk<T> ra[8];
        unsigned okmask = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int pix = kb * KB + ra0 + RSTEP_A * i;
          bool ok = a_mval && pix < npix;
          long long src = 0;
          if (ok) {
            const int img = pix / (p.oh * p.ow), rem = pix - img * (p.oh * p.ow);
            const int oy = rem / p.ow, ox = rem - oy * p.ow;
            const int iy = oy * p.stride - p.pad + a_ty, ix = ox * p.stride - p.pad + a_tx;
            ok = iy >= 0 && iy < p.h && ix >= 0 && ix < p.w;
            src = ((long long)img * p.h + iy) * p.w + ix;
          }
          if (ok) ra[i].load(reinterpret_cast<const T*>(p.a_ptr) + src * p.a_rs + a_ci);
          else ra[i].zero();
          okmask |= (ok ? 1u : 0u) << i;
        }
        Chunk<T> rb[C::B_PER], rbx[C::B_PER];
#pragma unroll
        for (int i = 0; i < C::B_PER; ++i) {
          const int pix = kb * KB + rb0 + RSTEP_B * i;
          if (b_nval && pix < npix) {
            rb[i].load(reinterpret_cast<const T*>(p.b_ptr) + (long long)pix * p.b_rs + co);
            if (p.b_pro == BNFF_PRO_BN_DX)
              rbx[i].load(reinterpret_cast<const T*>(p.b_xptr) + (long long)pix * p.b_xrs + co);
          } else {
            rb[i].zero();
            rbx[i].raw = rb[i].raw;
          }
        }
        if (it >= STAGES) mbar_wait(&empty_bar[s], ((it / STAGES) - 1) & 1);
        uint8_t* a0 = stage_a(s, 0);
        uint8_t* a1 = stage_a(s, 1);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float f[V], xf[V];
          ra[i].to_float(f);
          if ((okmask >> i) & 1u) {
            apply_pro<V>(p.a_pro, f, xf, a_ci, p.a_coef);
          } else {
#pragma unroll
            for (int q = 0; q < V; ++q) f[q] = 0.f;
          }
          st_chunk<T, V>(a0, a1, mn_off<T, 128, KB>(ra0 + RSTEP_A * i, ja * V), f);
        }
        uint8_t* b0 = stage_b(s, 0);
        uint8_t* b1 = stage_b(s, 1);
#pragma unroll
        for (int i = 0; i < C::B_PER; ++i) {
          const int pix = kb * KB + rb0 + RSTEP_B * i;
          float f[V], xf[V];
          rb[i].to_float(f);
          if (p.b_pro == BNFF_PRO_BN_DX) rbx[i].to_float(xf);
          if (b_nval && pix < npix) {
            apply_pro<V>(p.b_pro, f, xf, co, p.b_coef);
          } else {
#pragma unroll
            for (int q = 0; q < V; ++q) f[q] = 0.f;
          }
          st_chunk<T, V>(b0, b1, mn_off<T, BN, KB>(rb0 + RSTEP_B * i, jb * V), f);
        }
        fence_proxy_async_smem();
        mbar_arrive(&full_bar[s]);
      }
    }
  } else if (lane == 0) {
    // ===================== MMA issuer =====================
    constexpr uint32_t fmt = C::F32 ? kFmtTF32 : kFmtBF16;
    constexpr uint32_t mn = MODE == MODE_WGRAD ? 1u : 0u;
    constexpr uint32_t idesc = make_idesc(128, BN, fmt, mn, mn);
    for (int it = 0; it < nk; ++it) {
      const int s = it % STAGES;
      mbar_wait(&full_bar[s], (it / STAGES) & 1);
      tc_fence_after();
      const uint32_t abase0 = smem_u32(stage_a(s, 0)), bbase0 = smem_u32(stage_b(s, 0));
      const uint32_t abase1 = smem_u32(stage_a(s, 1)), bbase1 = smem_u32(stage_b(s, 1));
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t ad0, bd0, ad1, bd1;
        if constexpr (MODE == MODE_WGRAD) {
          ad0 = mn_desc<T, 128, KB>(abase0, kk);
          bd0 = mn_desc<T, BN, KB>(bbase0, kk);
          ad1 = mn_desc<T, 128, KB>(abase1, kk);
          bd1 = mn_desc<T, BN, KB>(bbase1, kk);
        } else {
          ad0 = make_sdesc(abase0 + kk * 32, 16, 1024, kLayoutSW128);
          bd0 = make_sdesc(bbase0 + kk * 32, 16, 1024, kLayoutSW128);
          ad1 = make_sdesc(abase1 + kk * 32, 16, 1024, kLayoutSW128);
          bd1 = make_sdesc(bbase1 + kk * 32, 16, 1024, kLayoutSW128);
        }
        const uint32_t acc = (it > 0 || kk > 0) ? 1u : 0u;
        if constexpr (C::F32) {
          umma_tf32(tmem, ad0, bd0, idesc, acc);  // hi*hi
          umma_tf32(tmem, ad0, bd1, idesc, 1u);   // hi*lo
          umma_tf32(tmem, ad1, bd0, idesc, 1u);   // lo*hi
        } else {
          umma_f16(tmem, ad0, bd0, idesc, acc);
        }
      }
      umma_commit(&empty_bar[s]);
    }
    umma_commit(&acc_bar);
  }
  __syncwarp();

  // ===================== epilogue (warps 0-3) =====================
  if (warp < 4) {
    mbar_wait(&acc_bar, 0);
    tc_fence_after();
    const int row = warp * 32 + lane;
    const int gm = m0 + row;
    const bool rval = gm < p.M;
    const bool do_stats = p.stat_part != nullptr;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
      float v[16];
      tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
      tmem_ld_wait();
      const int gc0 = n0 + c0;
      if constexpr (MODE == MODE_WGRAD) {
        if (rval) {
          float* dst = reinterpret_cast<float*>(p.c_ptr) +
                       ((long long)blockIdx.z * p.M + gm) * (long long)p.c_rs + gc0;
#pragma unroll
          for (int q = 0; q < 16; q += 4) {
            if (gc0 + q < p.N)
              *reinterpret_cast<float4*>(dst + q) = make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
          }
        }
      } else {
        float s1[16], s2[16];
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
          // round to storage precision; statistics use the stored value
          float r;
          if constexpr (sizeof(T) == 2) r = __bfloat162float(__float2bfloat16_rn(val));
          else r = val;
          v[q] = r;
          const bool sv = rval && cval;
          if constexpr (MODE == MODE_FPROP) {
            s1[q] = sv ? r : 0.f;
            s2[q] = sv ? r * r : 0.f;
          } else {
            float xh = 0.f;
            if (p.epi == BNFF_DG_NRC && cval)
              xh = __fmul_rn(__fsub_rn(xv[q], __ldg(p.e_coef.a + gc)), __ldg(p.e_coef.d + gc));
            s1[q] = sv ? r : 0.f;
            s2[q] = sv ? r * xh : 0.f;
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
            red[warp][0][c0 + (lane >> 1)] = s1[0];
            red[warp][1][c0 + (lane >> 1)] = s2[0];
          }
        }
      }
    }
    if (MODE != MODE_WGRAD && do_stats) {
      named_bar(1, 128);
      for (int c = tid; c < BN; c += 128) {
        const int gc = n0 + c;
        if (gc < p.N) {
          const float a = ((red[0][0][c] + red[1][0][c]) + red[2][0][c]) + red[3][0][c];
          const float b = ((red[0][1][c] + red[1][1][c]) + red[2][1][c]) + red[3][1][c];
          p.stat_part[((long long)blockIdx.x * 2 + 0) * p.stat_ld + gc] = a;
          p.stat_part[((long long)blockIdx.x * 2 + 1) * p.stat_ld + gc] = b;
        }
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
template <int MODE, int BN, typename T>
static int launch_ig(const IgParams& p, int splits, cudaStream_t st) {
  using C = IgCfg<MODE, BN, T>;
  auto kern = igemm_kernel<MODE, BN, T>;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(igemm)");
    attr_set = true;
  }
  dim3 grid((p.M + 127) / 128, (p.N + BN - 1) / BN, splits);
  kern<<<grid, 160, C::SMEM, st>>>(p);
  return check_launch("igemm");
}

template <int MODE, typename T>
static int dispatch_bn(const IgParams& p, int bn, int splits, cudaStream_t st) {
  switch (bn) {
    case 32: return launch_ig<MODE, 32, T>(p, splits, st);
    case 64: return launch_ig<MODE, 64, T>(p, splits, st);
    case 128: return launch_ig<MODE, 128, T>(p, splits, st);
    default: return launch_ig<MODE, 256, T>(p, splits, st);
  }
}

template <int MODE>
static int dispatch(int dtype, const IgParams& p, int bn, int splits, cudaStream_t st) {
  if (dtype == BNFF_BF16) return dispatch_bn<MODE, __nv_bfloat16>(p, bn, splits, st);
  return dispatch_bn<MODE, float>(p, bn, splits, st);
}

static int pick_bn(int n) {
  if (n <= 32) return 32;
  if (n <= 64) return 64;
  if (n <= 128) return 128;
  return 256;
}

static inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace bnff

using namespace bnff;

// K index padding for packed weights: multiple of one stage (64 bf16 / 32 f32)
static inline int kpad_elems(int dtype, int k) {
  const int kb = dtype == BNFF_BF16 ? 64 : 32;
  return (k + kb - 1) / kb * kb;
}

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
  p.M = p.n * p.oh * p.ow;
  p.N = p.cout;
  p.kred = p.cin;
  const int K = p.kh * p.kw * p.cin;
  const int kb = a->dtype == BNFF_BF16 ? 64 : 32;
  p.nkb = (K + kb - 1) / kb;
  p.kb_per_split = p.nkb;
  p.a_ptr = a->x.ptr; p.a_rs = a->x.row_stride; p.a_pro = a->x_pro; p.a_coef = a->x_coef;
  p.b_ptr = a->wpack; p.b_rs = kpad_elems(a->dtype, K);
  p.c_ptr = a->y.ptr; p.c_rs = a->y.row_stride;
  p.bias = a->bias;
  p.stat_part = a->stat_part;
  p.stat_ld = p.cout;
  return dispatch<MODE_FPROP>(a->dtype, p, pick_bn(p.N), 1, (cudaStream_t)stream);
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
  p.M = p.n * p.h * p.w;
  p.N = p.cin;
  p.kred = p.cout;
  const int K = p.kh * p.kw * p.cout;
  const int kb = a->dtype == BNFF_BF16 ? 64 : 32;
  p.nkb = (K + kb - 1) / kb;
  p.kb_per_split = p.nkb;
  p.a_ptr = a->dy.ptr; p.a_rs = a->dy.row_stride; p.a_pro = a->dy_pro; p.a_coef = a->dy_coef;
  p.a_xptr = a->dy_x.ptr; p.a_xrs = a->dy_x.row_stride;
  p.b_ptr = a->wpack_t; p.b_rs = kpad_elems(a->dtype, K);
  p.c_ptr = a->dx.ptr; p.c_rs = a->dx.row_stride;
  p.epi = a->epi;
  p.e_xptr = a->x.ptr; p.e_xrs = a->x.row_stride; p.e_coef = a->x_coef;
  p.stat_part = a->epi == BNFF_DG_NRC ? a->stat_part : nullptr;
  p.stat_ld = p.cin;
  return dispatch<MODE_DGRAD>(a->dtype, p, pick_bn(p.N), 1, (cudaStream_t)stream);
}

extern "C" int32_t bnff_wgrad_default_splits(int32_t n, int32_t oh, int32_t ow, int32_t kh,
                                             int32_t kw, int32_t c_in, int32_t c_out) {
  const long long npix = (long long)n * oh * ow;
  const int nkb = (int)((npix + 63) / 64);
  const int tiles = ((kh * kw * c_in + 127) / 128) * ((c_out + pick_bn(c_out) - 1) / pick_bn(c_out));
  int splits = (2 * 148 + tiles - 1) / tiles;
  const int max_splits = nkb / 4 > 0 ? nkb / 4 : 1;  // >= 4 k-blocks per split
  if (splits > max_splits) splits = max_splits;
  if (splits < 1) splits = 1;
  return splits;
}

extern "C" int64_t bnff_wgrad_workspace(int32_t n, int32_t oh, int32_t ow, int32_t kh, int32_t kw,
                                        int32_t c_in, int32_t c_out, int32_t splits) {
  if (splits <= 0) splits = bnff_wgrad_default_splits(n, oh, ow, kh, kw, c_in, c_out);
  const long long npix = (long long)n * oh * ow;
  // split-K partial tiles + dbias channel partials [tiles][2][c_out]
  return (int64_t)splits * kh * kw * c_in * c_out + (int64_t)bnff_sum_tiles(npix) * 2 * c_out;
}

namespace bnff {
// dW[co][ci][ky][kx] = sum_s ws[s][(tap*cin + ci)][co]   (fixed split order)
__global__ void wgrad_reduce_kernel(const float* __restrict__ ws, int splits, int M, int N, int cin,
                                    int cin_real, int taps, float* __restrict__ dw) {
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
  const int taps = p.kh * p.kw;
  p.M = taps * p.cin;
  p.N = p.cout;
  const int kb = a->dtype == BNFF_BF16 ? 64 : 32;
  const long long npix = (long long)p.n * p.oh * p.ow;
  p.nkb = (int)((npix + kb - 1) / kb);
  int splits = a->splits > 0 ? a->splits
                             : bnff_wgrad_default_splits(p.n, p.oh, p.ow, p.kh, p.kw, p.cin, p.cout);
  if (splits > p.nkb) splits = p.nkb;
  p.kb_per_split = (p.nkb + splits - 1) / splits;
  splits = (p.nkb + p.kb_per_split - 1) / p.kb_per_split;  // no empty splits
  p.a_ptr = a->x.ptr; p.a_rs = a->x.row_stride; p.a_pro = a->x_pro; p.a_coef = a->x_coef;
  p.b_ptr = a->dy.ptr; p.b_rs = a->dy.row_stride; p.b_pro = a->dy_pro; p.b_coef = a->dy_coef;
  p.b_xptr = a->dy_x.ptr; p.b_xrs = a->dy_x.row_stride;
  p.c_ptr = a->workspace; p.c_rs = p.N;
  cudaStream_t st = (cudaStream_t)stream;
  rc = dispatch<MODE_WGRAD>(a->dtype, p, pick_bn(p.N), splits, st);
  if (rc) return rc;
  const long long total = (long long)p.M * p.N;
  const int blocks = (int)((total + 255) / 256 < 148 * 8 ? (total + 255) / 256 : 148 * 8);
  const int cin_real = a->dw_cin > 0 ? a->dw_cin : p.cin;
  wgrad_reduce_kernel<<<blocks, 256, 0, st>>>(a->workspace, splits, p.M, p.N, p.cin, cin_real, taps,
                                               a->dw);
  rc = check_launch("wgrad_reduce");
  if (rc) return rc;
  if (a->dbias != nullptr) {
    float* scratch = a->workspace + (long long)splits * p.M * p.N;
    return bnff_dbias_scratch(a->dtype, a->dy, a->dy_x, a->dy_pro, a->dy_coef, scratch, a->dbias, stream);
  }
  return BNFF_OK;
}
