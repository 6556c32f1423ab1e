// wconv.cu -- window-shift implicit-GEMM convolutions on tcgen05 / TMEM (sm_100a, bf16).
//
// Stride-1 "same" convolutions (1x1 pad 0, 3x3 pad 1) are run on a PADDED GRID of
// output positions q = (img, py, px), py < h+2p, px < w+2p.  With the normalized
// input laid out on the same grid (zero border), every filter tap (ty, tx) of output
// q reads grid row q + ty*wp + tx: a pure row shift.  A CTA therefore loads and
// transforms each input element ONCE per tile into a shared-memory window of
// 128 + 2*wp + 2 rows (K-major, 128B/64B swizzled rows) and the MMA warp issues all
// 9 taps as UMMAs whose A descriptors start at shifted rows of that window
// (row-shifted swizzled descriptors validated by tools/umma_probe.cu).  Positions in
// the padding columns/rows are computed and discarded (7% at 56x56).
//
// FPROP  y[q, co] = sum_tap,ci  pro(x)[q + s_tap, ci] * W[co, ci, tap]
//        pro: NONE | RELU | BN_RELU (sub-BN2 + ReLU, fused.py:133-135)
//        epilogue: +bias, bf16 store into a channel-offset NHWC view (in-place concat),
//                  per-channel sum / sum^2 of the STORED values (sub-BN1 + MVF)
// DGRAD  dx[q, ci] = sum_tap,co pro(dy)[q + s_tap, co] * W[co, ci, flip(tap)]
//        pro: NONE | BN_DX (deferred sub-BN1' dx, ops.py:283-298)
//        epilogue: PLAIN | CLIP (x>0) | NRC (mask relu(bn(x))>0, sum dt1, sum dt1*xhat,
//                  fused.py:176-188)
//
// CTA = 13 warps: 8 loader warps (LDG -> transform in fp32 -> packed bf16 -> swizzled
// STS), 1 MMA warp (TMEM owner, one elected lane issues tcgen05.mma), 4 epilogue warps
// (TMEM -> registers -> smem staging -> coalesced stores; column statistics from the
// staged tile).  Persistent grid, double-buffered TMEM accumulators, mbarrier rings.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "sm100.cuh"
#include <type_traits>
#include "common.cuh"

namespace bnff {
namespace wc {

enum { M_FPROP = 0, M_DGRAD = 1 };
constexpr int NLW = 8;                  // loader warps
constexpr int LT = NLW * 32;            // loader threads
constexpr int THREADS = (NLW + 1 + 4) * 32;      // wgrad kernel: 4 epilogue warps
constexpr int NEW = 8;                           // wconv: epilogue warps (2 groups of 4)
constexpr int WC_THREADS = (NLW + 1 + NEW + 1) * 32;  // + one TMA producer warp
constexpr int PRODUCER = NLW + 1 + NEW;
constexpr int RMAX = 384;               // max window rows (wp <= 127 for 3x3)
constexpr int SMEM_BUDGET = 225 * 1024;
constexpr int kWindowNoFit = -100;      // internal: shape does not fit, use the generic kernel

struct WcParams {
  // TMA boxes of the window operand (and of the BN_DX x operand): rank 2 {c, pixels}
  // box {slab, 128} for 1x1; rank 4 {c, w, h, n} box {slab, wp, BR, BI} for 3x3
  CUtensorMap tma_a, tma_x;
  CUtensorMap tma_out;
  CUtensorMap tma_ex;   // tstore + dgrad mask: the x tile of the output channels, same box as tma_out  // tstore: the output written by TMA stores from the swizzled staging tile
  // 3x3 tiling: tmode 1 = kt output rows of one image (window rows oy-1 .. oy+kt),
  // tmode 2 = kt whole images per tile (small maps); WPI = window rows per image block,
  // tpi = tiles per image (tmode 1), Rld = rows the TMA writes per stage
  int tmode, kt, BR, BI, WPI, tpi, Rld, P;
  int n, h, w, hp, wp, pad, Q, mtiles, ntiles, tiles, R, stages;
  FastDiv fd_hpwp, fd_wp;
  int ci, nslab, N, npad;
  int pro;
  bnff_coef pcoef;
  const uint8_t* wpk;
  void* out; long long out_rs;      // bf16 or fp32 elements (the kernel's ES)
  const float* bias;
  int epi;
  const void* ex; long long ex_rs;
  bnff_coef ecoef;
  double* stat_part;
  int tstore;                  // 1: staging in 128B-swizzled rows, stored by cp.async.bulk.tensor
  unsigned long long* trace;  // debug: per-event %globaltimer stamps of CTA 0 (bnff_debug_trace)
};

// small-M 1x1 fprop tile target (default 0 = off: at 120 the D121 step measured 0.5% (fp32) and
// 1.4% (bf16) slower -- the re-read A tile and its prologue cost more than the idle SMs)
inline int smallm_tiles() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BNFF_SMALLM");
    v = e ? atoi(e) : 0;
  }
  return v;
}


// event stamps of CTA 0 into p.trace[ev * 1024 + i]: compiled in only with -DBNFF_WC_TRACE=1
// (tools/ab_defines.sh builds such a library for tools/trace_conv.py)
#ifndef BNFF_WC_TRACE
#define BNFF_WC_TRACE 0
#endif
__device__ __forceinline__ void trace_ev(unsigned long long* tr, int ev, int i) {
  if (BNFF_WC_TRACE && tr != nullptr && blockIdx.x == 0 && i < 1024) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[ev * 1024 + i] = t;
  }
}

// BNFF_WRES3=0: stream the fp32 3x3 dgrad weights per stage (A/B timing)
inline bool wres3_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BNFF_WRES3");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v != 0;
}

__host__ __device__ constexpr int align_up(int v, int a) { return (v + a - 1) / a * a; }

// GEMM N tile for an output-channel count
__host__ __device__ inline int pick_bn(int N) { return N <= 32 ? 32 : (N <= 64 ? 64 : (N <= 128 ? 128 : 256)); }
__host__ __device__ inline int pick_rb(int CI) { return CI <= 32 ? 64 : 128; }

struct Geo {
  int taps, RB, BN, ntiles, npad, nslab, sw;
};
// dgrad N tiles are capped at 128 columns: the NRC epilogue keeps a whole x tile in flight.
// 3x3 weights stay resident in shared memory when they fit (<= 96 KB, one N tile); wider
// 3x3 convs (ResNet's 128..512 channels) stream the 9 taps of each slab with the stage
// (sw = 1), in 64-column N tiles.
__host__ __device__ inline Geo geo(int CI, int N, int kh, int kw, int dgrad, int es = 2) {
  Geo g{};
  g.taps = kh * kw;
  if (es == 4) {
    // fp32 (3xTF32): every operand element takes 8 bytes of shared memory (hi + lo planes).
    // 1x1: 128-byte slabs (32 channels), N tiles <= 128 (fprop) / 64 (dgrad: x tile + 2
    // staging buffers per group); 3x3: 64-byte slabs (16 channels), weights streamed with
    // the stage, N tiles of 32 / 64
    // 1x1 dgrad: 64-byte slabs too, so two stages, the x tile, the staging rows and the ICF
    // fold's block-gradient tile fit beside a 1024-column epilogue table
    g.RB = (g.taps == 9 || CI <= 16 || dgrad) ? 64 : 128;
    g.BN = pick_bn(N);
    const int cap = g.taps == 9 ? (dgrad ? 32 : 64) : (dgrad ? 64 : (g.RB == 64 ? 32 : 128));
    if (g.BN > cap) g.BN = cap;
    g.nslab = (CI + g.RB / 4 - 1) / (g.RB / 4);
    // 3x3 dgrad over few output channels (DenseNet's growth k = 32: 2 slabs): the CTA's N tile
    // of the packed weights (9 taps x hi/lo, 72 KB) stays resident instead of streaming with
    // every stage of every tile
#ifdef __CUDA_ARCH__
    const bool w3 = true;
#else
    const bool w3 = wres3_enabled();
#endif
    g.sw = g.taps == 9 && !(dgrad && g.BN == 32 && g.nslab * 9 * 32 * 64 * 2 <= 80 * 1024 && w3) ? 1 : 0;
    g.ntiles = (N + g.BN - 1) / g.BN;
    g.npad = g.ntiles * g.BN;
    return g;
  }
  // 3x3: 64-byte slabs (32 channels) -> small window stages, deep prefetch beside the
  // resident weights
  g.RB = (CI <= 32 || g.taps == 9) ? 64 : pick_rb(CI);
  g.BN = pick_bn(N);
  if (dgrad && g.BN > 128) g.BN = 128;
  g.nslab = (CI + g.RB / 2 - 1) / (g.RB / 2);
  g.ntiles = (N + g.BN - 1) / g.BN;
  if (g.taps == 9 && (g.ntiles > 1 || g.nslab * 9 * g.BN * g.RB > 96 * 1024)) {
    g.sw = 1;
    g.BN = 64;
    g.ntiles = (N + g.BN - 1) / g.BN;
  }
  g.npad = g.ntiles * g.BN;
  return g;
}


template <int BN, int RB, int TAPS, int MODE, bool SW = false, int ES = 2>
struct Layout {
  static constexpr bool F32 = ES == 4;               // fp32 storage, 3xTF32 MMAs
  static constexpr int PL = F32 ? 2 : 1;             // operand planes (hi, lo)
  static constexpr int SLABW = RB / ES;              // channels per slab row
  static constexpr int CPR = RB / 16;                // 16B chunks per row
  static constexpr int RS = LT / CPR;                // loader row step
  static constexpr int UR = (TAPS == 1 ? 128 : RMAX) / RS;  // rows per loader thread (max)
  // weights resident in smem (else streamed per stage): 3x3 unless streamed (SW); 1x1 fprop
  // when SW is set (the CTA's fixed N tile of every slab, loaded once by the producer)
  static constexpr bool WRES = (TAPS == 9 && !SW) || (TAPS == 1 && SW && MODE == M_FPROP);
  static constexpr bool XOP = MODE == M_DGRAD;       // second window operand (BN_DX x)
  // epilogue column chunk: two groups of 4 warps take alternate chunks
  static constexpr int CW = F32 ? (BN <= 32 ? 16 : 32) : (BN <= 32 ? 16 : (BN == 64 ? 32 : 64));
  static constexpr int NCH = BN / CW;                // chunks per tile (>= 2)
  static constexpr int MYCH = (NCH + 1) / 2;         // chunks per epilogue group
  // staging row pitch (bytes): 64-column chunks use dense 128-byte rows with the 128B swizzle
  // (the TMA box layout); narrower chunks pad each row by 16 bytes against bank conflicts
  static constexpr bool TST = CW * ES == 128;       // 128-byte staging rows stored by TMA
  static constexpr int SROWB = TST ? 128 : CW * ES + 16;
  static constexpr int STG = 128 * SROWB;
  // per group: out staging (+ dgrad: one x buffer per owned chunk = a whole-tile lookahead)
  static constexpr int NSTG = MODE == M_DGRAD ? 1 + MYCH : 1;
  // 3xTF32 with a stacked B operand: A_hi x [B_hi | B_lo] is ONE N = 2*BN MMA into [D | D'] and
  // A_lo x B_hi accumulates into D', the epilogue adds the halves (two MMAs per K step, not three)
  static constexpr int ACOLS = F32 && BNFF_TF32_STACK ? 2 * BN : BN;  // TMEM columns per accumulator
  static constexpr int TCOLS = 2 * ACOLS < 32 ? 32 : 2 * ACOLS;
  static constexpr uint32_t LAY = RB == 128 ? kLayoutSW128 : kLayoutSW64;
  static constexpr uint32_t SBO = 8 * RB;
};

// byte offsets of the dynamic shared memory carve-up (identical on host and device)
struct Carve {
  int wres, stage0, stage_bytes, a_bytes, stg, gbuf, ptab, etab, sacc, red, rowtab, rowpix, meta, total;
};

template <int BN, int RB, int TAPS, int MODE, bool SW = false, int ES = 2>
// tf: tables the launch needs -- bit 0: operand-prologue table (pro != NONE), bit 1: the NRC
// epilogue's four columns (dgrad, epi >= NRC); plain launches (patch-matrix GEMMs) carve neither
__host__ __device__ inline Carve carve(int R, int nslab, int npad, int stages, bool xop, bool gb = false,
                                       int tf = 3) {
  using L = Layout<BN, RB, TAPS, MODE, SW, ES>;
  Carve c{};
  int off = 0;
  c.wres = off;
  if (L::WRES) off += align_up(nslab * TAPS * BN * RB * L::PL, 1024);
  c.a_bytes = align_up(R * RB, 1024);
  // stage: A planes (hi[, lo]) | x operand (BN_DX; fp32: inside the lo plane) | B planes (streamed weights)
  c.stage_bytes = c.a_bytes * (L::PL + (xop && !L::F32 ? 1 : 0)) + (L::WRES ? 0 : TAPS * BN * RB * L::PL);
  c.stage0 = off;
  off += stages * c.stage_bytes;
  c.stg = off;
  off += 2 * L::NSTG * L::STG;
  c.gbuf = off;  // block-gradient fold by TMA: one 128B-swizzled G tile per owned chunk
  if (gb) off += 2 * L::MYCH * 128 * 128;
  c.ptab = off;
  if (tf & 1) off += 3 * nslab * L::SLABW * 4;
  c.etab = off;
  off += (MODE == M_DGRAD && (tf & 2) ? 4 : 1) * npad * 4;  // bias | NRC (scale, shift, inv, -mean*inv)
  c.sacc = off;
  off += 2 * BN * (L::F32 ? 8 : 4);  // per-CTA sums (fp32 data: float64)
  c.red = off;
  off += 2 * 4 * 128 * (L::F32 ? 8 : 4);
  c.rowtab = off;
  off += 2 * RMAX * 4;
  c.rowpix = off;
  off += 2 * 128 * 4;
  c.meta = off;  // (unused by the TMA loader)
  c.total = off + 1024;  // + alignment slack
  return c;
}

template <int MODE>
__host__ __device__ inline int wtables(const WcParams& p) {
  return (p.pro != BNFF_PRO_NONE ? 1 : 0) | (MODE == M_DGRAD && p.epi >= BNFF_DG_NRC ? 2 : 0);
}

// the 1x1 block-gradient fold runs through TMA (G tile loaded, folded in smem, stored back)
template <int BN, int RB, int TAPS, int MODE, bool SW, int ES = 2>
__host__ __device__ inline bool fold_tma(const WcParams& p) {
  return TAPS == 1 && MODE == M_DGRAD && Layout<BN, RB, TAPS, MODE, SW, ES>::TST && p.epi >= BNFF_DG_NRC_ACC;
}

__device__ __forceinline__ void unpack8(const uint4& r, float* f) {
  f[0] = bf16lo(r.x); f[1] = bf16hi(r.x); f[2] = bf16lo(r.y); f[3] = bf16hi(r.y);
  f[4] = bf16lo(r.z); f[5] = bf16hi(r.z); f[6] = bf16lo(r.w); f[7] = bf16hi(r.w);
}
__device__ __forceinline__ uint4 pack8(const float* f, bool relu) {
  uint4 o;
  if (relu) {
    o.x = pack_bf16_relu(f[0], f[1]); o.y = pack_bf16_relu(f[2], f[3]);
    o.z = pack_bf16_relu(f[4], f[5]); o.w = pack_bf16_relu(f[6], f[7]);
  } else {
    o.x = pack_bf16_rn(f[0], f[1]); o.y = pack_bf16_rn(f[2], f[3]);
    o.z = pack_bf16_rn(f[4], f[5]); o.w = pack_bf16_rn(f[6], f[7]);
  }
  return o;
}
__device__ __forceinline__ void ld4f(const float* p, float* v) {  // 4 floats, 16B aligned
  const float4 a = *reinterpret_cast<const float4*>(p);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
}
__device__ __forceinline__ void ld8f(const float* p, float* v) {  // 8 floats, 16B aligned
  const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void ld16f(const float* p, float* v) {  // 16 floats, 16B aligned
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float4 t = reinterpret_cast<const float4*>(p)[i];
    v[4 * i] = t.x; v[4 * i + 1] = t.y; v[4 * i + 2] = t.z; v[4 * i + 3] = t.w;
  }
}
__device__ __forceinline__ void cp_async_wait_dyn(int n) {
  switch (n) {
    case 0: cp_async_wait<0>(); break;
    case 1: cp_async_wait<1>(); break;
    case 2: cp_async_wait<2>(); break;
    case 3: cp_async_wait<3>(); break;
    case 4: cp_async_wait<4>(); break;
    case 5: cp_async_wait<5>(); break;
    case 6: cp_async_wait<6>(); break;
    default: cp_async_wait<7>(); break;
  }
}

template <int BN, int RB, int TAPS, int MODE, bool SW = false, int ES = 2>
__global__ void __launch_bounds__(WC_THREADS, 1) wconv_kernel(const __grid_constant__ WcParams p) {
  griddep_launch();
  if (threadIdx.x == 0) trace_ev(p.trace, 8, 0);
  using L = Layout<BN, RB, TAPS, MODE, SW, ES>;
  constexpr bool F32 = L::F32;
  constexpr int PL = L::PL;
  using E = typename std::conditional<F32, float, __nv_bfloat16>::type;  // storage element
  using SA = typename std::conditional<F32, double, float>::type;        // statistics accumulator
  constexpr int CPR = L::CPR, RS = L::RS, UR = L::UR, SLABW = L::SLABW, CW = L::CW;
  extern __shared__ uint8_t dsm_raw[];
  // offset (not integer-cast) the shared array so the compiler keeps the shared state space
  uint8_t* smem = dsm_raw + ((1024u - (smem_u32(dsm_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full_bar[8], empty_bar[8], ld_bar[8], accf_bar[2], acce_bar[2], w_bar, g_bar[4], x_bar[4];
  __shared__ uint32_t tmem_sh;
  const bool xop_s = L::XOP && p.pro == BNFF_PRO_BN_DX;
  const bool gb_s = fold_tma<BN, RB, TAPS, MODE, SW, ES>(p);
  const int tf_s = wtables<MODE>(p);
  const Carve cv = carve<BN, RB, TAPS, MODE, SW, ES>(p.R, p.nslab, p.npad, p.stages, xop_s, gb_s, tf_s);
  const int ST = p.stages;
  float* ptab = reinterpret_cast<float*>(smem + cv.ptab);
  float* etab = reinterpret_cast<float*>(smem + cv.etab);
  SA* sacc = reinterpret_cast<SA*>(smem + cv.sacc);
  SA* red = reinterpret_cast<SA*>(smem + cv.red);
  int* rowtab = reinterpret_cast<int*>(smem + cv.rowtab);
  int* rowpix = reinterpret_cast<int*>(smem + cv.rowpix);
  uint32_t* meta = reinterpret_cast<uint32_t*>(smem + cv.meta);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ntl = (p.tiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  const bool do_stats = p.stat_part != nullptr;
  const int kpad = p.nslab * SLABW;

  // ---- setup: barriers, TMEM, coefficient tables
  if (tid == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full_bar[s], LT + (L::WRES ? 0 : 1));
      mbar_init(&empty_bar[s], 1);
      mbar_init(&ld_bar[s], 1);
    }
    tma_prefetch_desc(&p.tma_a);
    if (xop_s) tma_prefetch_desc(&p.tma_x);
    for (int s = 0; s < 2; ++s) { mbar_init(&accf_bar[s], 1); mbar_init(&acce_bar[s], NEW * 32); }
    mbar_init(&w_bar, 1);
    for (int s = 0; s < 4; ++s) { mbar_init(&g_bar[s], 1); mbar_init(&x_bar[s], 1); }
    if (p.tstore) tma_prefetch_desc(&p.tma_out);
    if (p.tstore && MODE == M_DGRAD && p.epi != BNFF_DG_PLAIN) tma_prefetch_desc(&p.tma_ex);
    fence_mbar_init();
    if (L::WRES && TAPS == 9) {
      // resident weights: packed after the previous optimizer step, i.e. at least two
      // launches back, so they may be fetched before this grid's dependency wait
      const uint32_t wb = p.nslab * TAPS * BN * RB * PL;
      mbar_arrive_expect_tx(&w_bar, wb);
      if (p.ntiles == 1) {
        bulk_g2s(smem_u32(smem + cv.wres), p.wpk, wb, &w_bar);
      } else {  // this CTA's N tile ([slab][tap][plane][npad][RB] rows n0 .. n0 + BN of each)
        const int n0r = ((int)blockIdx.x % p.ntiles) * BN;
        for (int c = 0; c < p.nslab * TAPS * PL; ++c)
          bulk_g2s(smem_u32(smem + cv.wres) + c * BN * RB, p.wpk + ((long long)c * p.npad + n0r) * RB, BN * RB,
                   &w_bar);
      }
    }
  }
  if (warp == NLW) tmem_alloc<L::TCOLS>(&tmem_sh);
  __syncthreads();  // barrier initialisation visible to every role (no data dependency yet)
  griddep_wait();   // everything below reads data of the preceding launches
  // the producer warp (the last warp) starts streaming the first stages at once; the other
  // warps build the coefficient tables meanwhile and meet on a named barrier
  constexpr int ST_THREADS = WC_THREADS - 32;
  static_assert(PRODUCER * 32 == ST_THREADS, "producer is the last warp");
  if (warp != PRODUCER) {
  // window-operand tables: BN_RELU: (scale, beta - mean*scale); BN_DX: (g, -g*k2*inv, g*(k2*inv*mean-k1))
  for (int c = tid; (tf_s & 1) && c < kpad; c += ST_THREADS) {
    float t0 = 1.f, t1 = 0.f, t2 = 0.f;
    if (c < p.ci) {
      if (p.pro == BNFF_PRO_BN_RELU) {
        const float m = p.pcoef.a[c], s = p.pcoef.b[c], b = p.pcoef.c[c];
        t0 = s;
        t1 = b - m * s;
      } else if (p.pro == BNFF_PRO_BN_DX) {
        const float m = p.pcoef.a[c], inv = p.pcoef.b[c], k1 = p.pcoef.c[c], k2 = p.pcoef.d[c],
                    g = p.pcoef.e[c];
        t0 = g;
        t1 = -g * k2 * inv;
        t2 = g * (k2 * inv * m - k1);
      }
    }
    ptab[c] = t0;
    ptab[kpad + c] = t1;
    ptab[2 * kpad + c] = t2;
  }
  // epilogue tables: FPROP: bias; DGRAD NRC: (scale, beta-mean*scale, inv, -mean*inv)
  for (int c = tid; c < p.npad; c += ST_THREADS) {
    float t0 = 0.f, t1 = 0.f, t2 = 0.f, t3 = 0.f;
    if (c < p.N) {
      if (MODE == M_FPROP) {
        t0 = p.bias ? p.bias[c] : 0.f;
      } else if (p.epi >= BNFF_DG_NRC) {
        const float m = p.ecoef.a[c], s = p.ecoef.b[c], b = p.ecoef.c[c], inv = p.ecoef.d[c];
        t0 = s;
        t1 = b - m * s;
        t2 = inv;
        t3 = -m * inv;
      }
    }
    etab[c] = t0;
    if (MODE == M_DGRAD && (tf_s & 2)) {
      etab[p.npad + c] = t1;
      etab[2 * p.npad + c] = t2;
      etab[3 * p.npad + c] = t3;
    }
  }
  for (int c = tid; c < BN; c += ST_THREADS) {
    sacc[c] = SA(0);
    sacc[BN + c] = SA(0);
  }
  if (TAPS == 9) {  // window row -> (image block, padded row, padded column), same every tile
    for (int r = tid; r < p.Rld; r += ST_THREADS) {
      const int i = r / p.WPI, rem = r - i * p.WPI;
      const int ry = rem / p.wp, rx = rem - ry * p.wp;
      rowtab[r] = (i << 20) | (ry << 10) | rx;
    }
  }
  if (p.stat_part != nullptr && p.ntiles > 1)  // this CTA's partial row accumulates in place
    for (int c = tid; c < 2 * p.N; c += ST_THREADS) p.stat_part[(long long)blockIdx.x * 2 * p.N + c] = 0.f;
  tc_fence_before();
  asm volatile("bar.sync 1, %0;" ::"n"(ST_THREADS) : "memory");
  tc_fence_after();
  }
  if (threadIdx.x == 0) trace_ev(p.trace, 9, 0);
  const uint32_t tmem = tmem_sh;

  // stage: A hi [| A lo] [| x] | B (tap-major [tap][plane][BN][RB])
  auto stage_a = [&](int s) { return smem + cv.stage0 + s * cv.stage_bytes; };
  // fp32: the BN_DX x operand lands in the lo plane -- each element is read by the thread that
  // then writes its lo value there, so it needs no plane of its own
  auto stage_x = [&](int s) { return smem + cv.stage0 + s * cv.stage_bytes + cv.a_bytes * (F32 ? 1 : PL); };
  auto stage_b = [&](int s) {
    return smem + cv.stage0 + s * cv.stage_bytes + cv.a_bytes * (PL + (xop_s && !F32 ? 1 : 0));
  };
  auto tile_of = [&](int it, int& mt, int& n0) {
    const int t = (int)blockIdx.x + it * (int)gridDim.x;
    mt = t / p.ntiles;
    n0 = (t % p.ntiles) * BN;
  };
  // 3x3 tile origin: first image and the padded-input row the window starts at
  auto tile_org = [&](int mt, int& img0, int& y0) {
    if (p.tmode == 1) {
      img0 = mt / p.tpi;
      y0 = (mt - img0 * p.tpi) * p.kt - 1;
    } else {
      img0 = mt * p.kt;
      y0 = -1;
    }
  };

  if (warp < NLW) {
    // =============================== transform warps ===============================
    // wait for a stage's TMA box, apply the operand prologue in place (halo / border
    // positions stay zero: padding applies after normalize/ReLU), arrive on full_bar.
    // the operand prologue kind is a compile-time constant inside the loop (one copy per kind)
    auto transform = [&](auto pro_c) {
    constexpr int PRO = decltype(pro_c)::value;
    const int j = tid % CPR, r0 = tid / CPR;
    const bool need_t = PRO != BNFF_PRO_NONE;
    int st = 0;
    uint32_t ph = 0;
    for (int it = 0; it < ntl; ++it) {
      int img0 = 0, y0 = 0;
      if (TAPS == 9) {
        int mt, n0;
        tile_of(it, mt, n0);
        tile_org(mt, img0, y0);
      }
      for (int s = 0; s < p.nslab; ++s) {
        mbar_wait(&ld_bar[st], ph);
        if (tid == 0) trace_ev(p.trace, 2, it * p.nslab + s);
        const int cs = min(SLABW, p.ci - s * SLABW);
        if constexpr (F32) {
          // prologue in fp32, then the 3xTF32 split: hi (round-to-nearest TF32) in place,
          // lo = f - hi (exact; the MMA truncates it to TF32) into the second plane; halo /
          // border positions keep the TMA's zero fill in hi and get a zero lo
          uint8_t* A = stage_a(st);
          uint8_t* AL = A + cv.a_bytes;
          const uint8_t* X = stage_x(st);
          const bool live = j * 4 < cs;
          const int c0 = s * SLABW + j * 4;
          float t0[4] = {1.f, 1.f, 1.f, 1.f}, t1[4] = {0.f, 0.f, 0.f, 0.f}, t2[4] = {0.f, 0.f, 0.f, 0.f};
          if (need_t && live) {
            ld4f(ptab + c0, t0);
            ld4f(ptab + kpad + c0, t1);
            ld4f(ptab + 2 * kpad + c0, t2);
          }
#pragma unroll
          for (int u = 0; u < UR; ++u) {
            const int r = r0 + u * RS;
            if (r >= p.Rld) continue;
            uint32_t off;
            if constexpr (RB == 128) off = r * 128 + ((j ^ (r & 7)) << 4);
            else off = r * 64 + ((j ^ ((r >> 1) & 3)) << 4);
            bool dead = !live;
            if (TAPS == 9) {
              const int wr = rowtab[r];
              const int y = y0 + ((wr >> 10) & 1023), rx = wr & 1023;
              dead = dead || (unsigned)y >= (unsigned)p.h || rx < 1 || rx > p.w || img0 + (wr >> 20) >= p.n;
            }
            if (dead) {
              *reinterpret_cast<uint4*>(AL + off) = make_uint4(0, 0, 0, 0);
              continue;
            }
            const float4 a4 = *reinterpret_cast<const float4*>(A + off);
            float f[4] = {a4.x, a4.y, a4.z, a4.w};
            if (PRO == BNFF_PRO_RELU) {
#pragma unroll
              for (int i = 0; i < 4; ++i) f[i] = fmaxf(f[i], 0.f);
            } else if (PRO == BNFF_PRO_BN_RELU) {
#pragma unroll
              for (int i = 0; i < 4; ++i) f[i] = fmaxf(fmaf(f[i], t0[i], t1[i]), 0.f);
            } else if (PRO == BNFF_PRO_BN_DX) {
              const float4 x4 = *reinterpret_cast<const float4*>(X + off);
              const float xf[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
              for (int i = 0; i < 4; ++i) f[i] = fmaf(f[i], t0[i], fmaf(xf[i], t1[i], t2[i]));
            }
            float4 hi, lo;
            hi.x = tf32_rn(f[0]); hi.y = tf32_rn(f[1]); hi.z = tf32_rn(f[2]); hi.w = tf32_rn(f[3]);
            lo.x = f[0] - hi.x; lo.y = f[1] - hi.y;
            lo.z = f[2] - hi.z; lo.w = f[3] - hi.w;
            *reinterpret_cast<float4*>(A + off) = hi;
            *reinterpret_cast<float4*>(AL + off) = lo;
          }
          fence_proxy_async_smem();
        } else if (need_t && j * 8 < cs) {
          const int c0 = s * SLABW + j * 8;
          float t0[8], t1[8], t2[8];
          ld8f(ptab + c0, t0);
          ld8f(ptab + kpad + c0, t1);
          ld8f(ptab + 2 * kpad + c0, t2);
          uint8_t* A = stage_a(st);
          uint8_t* X = stage_x(st);
#pragma unroll
          for (int u = 0; u < UR; ++u) {
            const int r = r0 + u * RS;
            if (r >= p.Rld) continue;
            if (TAPS == 9) {
              const int wr = rowtab[r];
              const int y = y0 + ((wr >> 10) & 1023), rx = wr & 1023;
              if ((unsigned)y >= (unsigned)p.h || rx < 1 || rx > p.w || img0 + (wr >> 20) >= p.n) continue;
            }
            uint32_t off;
            if constexpr (RB == 128) off = r * 128 + ((j ^ (r & 7)) << 4);
            else off = r * 64 + ((j ^ ((r >> 1) & 3)) << 4);
            float f[8];
            unpack8(*reinterpret_cast<const uint4*>(A + off), f);
            uint4 o;
            if (PRO == BNFF_PRO_RELU) {
              o = pack8(f, true);
            } else if (PRO == BNFF_PRO_BN_RELU) {  // paired FFMA2: same RN fp32 FMAs, half the issues
#pragma unroll
              for (int i = 0; i < 8; i += 2) {
                const float2 r2 = __ffma2_rn(make_float2(f[i], f[i + 1]), make_float2(t0[i], t0[i + 1]),
                                             make_float2(t1[i], t1[i + 1]));
                f[i] = r2.x;
                f[i + 1] = r2.y;
              }
              o = pack8(f, true);
            } else {
              float xf[8];
              unpack8(*reinterpret_cast<const uint4*>(X + off), xf);
#pragma unroll
              for (int i = 0; i < 8; i += 2) {
                const float2 in2 = __ffma2_rn(make_float2(xf[i], xf[i + 1]), make_float2(t1[i], t1[i + 1]),
                                              make_float2(t2[i], t2[i + 1]));
                const float2 r2 = __ffma2_rn(make_float2(f[i], f[i + 1]), make_float2(t0[i], t0[i + 1]), in2);
                f[i] = r2.x;
                f[i + 1] = r2.y;
              }
              o = pack8(f, false);
            }
            *reinterpret_cast<uint4*>(A + off) = o;
          }
          fence_proxy_async_smem();
        }
        mbar_arrive(&full_bar[st]);
        if (tid == 0) trace_ev(p.trace, 3, it * p.nslab + s);
        if (++st == ST) { st = 0; ph ^= 1u; }
      }
    }
    };
    switch (p.pro) {
      case BNFF_PRO_RELU: transform(std::integral_constant<int, BNFF_PRO_RELU>{}); break;
      case BNFF_PRO_BN_RELU: transform(std::integral_constant<int, BNFF_PRO_BN_RELU>{}); break;
      case BNFF_PRO_BN_DX: transform(std::integral_constant<int, BNFF_PRO_BN_DX>{}); break;
      default: transform(std::integral_constant<int, BNFF_PRO_NONE>{}); break;
    }
  } else if (warp == PRODUCER) {
    // =============================== TMA producer ===============================
    // the producer warp streams window boxes into the stage ring as fast as the MMA frees stages
    // (zero-filled outside the map: the 3x3 halo and image borders come for free)
    {  // converged warp; one elected lane issues the copies
      if (TAPS == 1 && L::WRES && elect_one()) {  // this CTA's N tile of every slab, once
        const int n0r = ((int)blockIdx.x % p.ntiles) * BN;
        mbar_arrive_expect_tx(&w_bar, (uint32_t)(p.nslab * BN * RB * PL));
        for (int s = 0; s < p.nslab * PL; ++s)  // [slab][plane] rows of the pack
          bulk_g2s(smem_u32(smem + cv.wres) + s * BN * RB, p.wpk + ((long long)s * p.npad + n0r) * RB, BN * RB,
                   &w_bar);
      }
      __syncwarp();
      const bool xop = L::XOP && p.pro == BNFF_PRO_BN_DX;
      const uint32_t tx_bytes = (uint32_t)p.Rld * RB * (xop ? 2u : 1u);
      int st = 0, round = 0;
      for (int it = 0; it < ntl; ++it) {
        int mt, n0;
        tile_of(it, mt, n0);
        int img0 = 0, y0 = 0;
        if (TAPS == 9) tile_org(mt, img0, y0);
        for (int s = 0; s < p.nslab; ++s) {
          trace_ev(p.trace, 0, it * p.nslab + s);
          if (round > 0) mbar_wait(&empty_bar[st], (round - 1) & 1);
          trace_ev(p.trace, 1, it * p.nslab + s);
          if (elect_one()) {
            if (!L::WRES) {  // this slab's weights for the N tile, every tap ([slab][tap][plane][npad][RB])
              mbar_arrive_expect_tx(&full_bar[st], TAPS * BN * RB * PL);
#pragma unroll 1
              for (int u = 0; u < TAPS * PL; ++u)
                bulk_g2s(smem_u32(stage_b(st)) + u * BN * RB,
                         p.wpk + ((long long)(s * TAPS * PL + u) * p.npad + n0) * RB, BN * RB, &full_bar[st]);
            }
            mbar_arrive_expect_tx(&ld_bar[st], tx_bytes);
            const int c = s * SLABW;
            if (TAPS == 9) {
              tma_load_4d(smem_u32(stage_a(st)), &p.tma_a, c, -1, y0, img0, &ld_bar[st]);
              if (xop) tma_load_4d(smem_u32(stage_x(st)), &p.tma_x, c, -1, y0, img0, &ld_bar[st]);
            } else {
              tma_load_2d(smem_u32(stage_a(st)), &p.tma_a, c, mt * 128, &ld_bar[st]);
              if (xop) tma_load_2d(smem_u32(stage_x(st)), &p.tma_x, c, mt * 128, &ld_bar[st]);
            }
          }
          __syncwarp();
          if (++st == ST) { st = 0; ++round; }
        }
      }
    }
    __syncwarp();
  } else if (warp == NLW) {
    // =============================== MMA issuer ===============================
    // the whole warp runs the loop (converged, warp-uniform operands); one elected lane issues
    {
      if (L::WRES) mbar_wait(&w_bar, 0);
      constexpr uint32_t idesc = make_idesc(128, BN, F32 ? kFmtTF32 : kFmtBF16, 0, 0);
      constexpr int KE = F32 ? 8 : 16;  // K elements per MMA (32 bytes either way)
      const uint32_t wres = smem_u32(smem + cv.wres);
      int st = 0;
      uint32_t ph = 0;
      for (int it = 0; it < ntl; ++it) {
        const int buf = it & 1;
        if (it >= 2) mbar_wait(&acce_bar[buf], ((it >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + buf * L::ACOLS;
        uint32_t acc = 0;
        for (int s = 0; s < p.nslab; ++s) {
          mbar_wait(&full_bar[st], ph);
          trace_ev(p.trace, 4, it * p.nslab + s);
          tc_fence_after();
          const uint32_t abase = smem_u32(stage_a(st));
          const uint32_t bbase = L::WRES ? wres + s * TAPS * BN * RB * PL : smem_u32(stage_b(st));
          const int ks = min(SLABW, p.ci - s * SLABW) / KE;
          // descriptors advance by adding (byte offset >> 4) to the start-address field
          const uint64_t a0 = make_sdesc(abase, 16, L::SBO, L::LAY);
          const uint64_t b0 = make_sdesc(bbase, 16, L::SBO, L::LAY);
#pragma unroll
          for (int u = 0; u < TAPS; ++u) {
            const uint32_t ash = TAPS == 9 ? (uint32_t)(((u / 3) * p.wp + (u % 3)) * RB) >> 4 : 0u;
            const uint32_t bsh = (uint32_t)(u * PL * BN * RB) >> 4;
#pragma unroll
            for (int kk = 0; kk < SLABW / KE; ++kk) {
              if (kk < ks) {
                if constexpr (F32) {  // 3xTF32: hi*hi + hi*lo + lo*hi
                  constexpr uint32_t blo = (uint32_t)(BN * RB) >> 4;
                  const uint32_t alo = (uint32_t)cv.a_bytes >> 4;
#if BNFF_TF32_STACK
                  // the lo plane of B follows the hi plane as rows BN..2BN-1 of one K-major
                  // operand (same SBO), so [B_hi | B_lo] is a single N = 2*BN descriptor
                  constexpr uint32_t idesc2 = make_idesc(128, 2 * BN, kFmtTF32, 0, 0);
                  umma_tf32_elect(d, a0 + ash + kk * 2, b0 + bsh + kk * 2, idesc2, acc);
                  umma_tf32_elect(d + BN, a0 + alo + ash + kk * 2, b0 + bsh + kk * 2, idesc, 1u);
                  (void)blo;
#else
                  umma_tf32_elect(d, a0 + ash + kk * 2, b0 + bsh + kk * 2, idesc, acc);
                  umma_tf32_elect(d, a0 + ash + kk * 2, b0 + bsh + blo + kk * 2, idesc, 1u);
                  umma_tf32_elect(d, a0 + alo + ash + kk * 2, b0 + bsh + kk * 2, idesc, 1u);
#endif
                } else {
                  umma_f16_elect(d, a0 + ash + kk * 2, b0 + bsh + kk * 2, idesc, acc);
                }
                acc = 1;
              }
            }
          }
          umma_commit_elect(&empty_bar[st]);
          trace_ev(p.trace, 5, it * p.nslab + s);
          if (++st == ST) { st = 0; ph ^= 1u; }
        }
        umma_commit_elect(&accf_bar[buf]);
      }
    }
    __syncwarp();
  } else {
    // =============================== epilogue ===============================
    // 8 warps = 2 groups x 4 (one warp per TMEM lane quadrant in each group); group h
    // drains column chunks h, h+2, ...  Per chunk: row pass (TMEM -> fp32 epilogue math
    // -> bf16 staging, thread = row), column pass (per-channel sums of the STAGED values,
    // thread = column pair, accumulated in registers), store pass (coalesced 16B stores
    // into the NHWC view).  Dgrad: the x tile for the NRC/CLIP mask is fetched one tile
    // ahead, chunk buffer by chunk buffer.
    // the dgrad epilogue kind is a compile-time constant inside the tile loop (one copy per kind)
    auto epilogue = [&](auto epi_c) {
    constexpr int EPI = decltype(epi_c)::value;
    const int quad = warp & 3;
    const int et = tid - (NLW + 1) * 32;     // 0..255
    const int grp = et >> 7;                 // 0 / 1
    const int gt = et & 127;
    const int row = quad * 32 + lane;
    const int bar_id = 2 + grp;
    uint8_t* stg = smem + cv.stg + grp * L::NSTG * L::STG;
    uint8_t* xs0 = stg + L::STG;             // dgrad: x buffers, one per owned chunk
    SA* gred = red + grp * 512;
    int* gpix = rowpix + grp * 128;
    const int hpwp = p.hp * p.wp;
    constexpr int CW = L::CW, NCH = L::NCH, MYCH = L::MYCH;
    constexpr int HALF = CW / 2;             // column pairs per chunk
    constexpr int RG = 128 / HALF;           // row groups in the column pass
    const int cp = gt % HALF, rg = gt / HALF;
    const bool need_x = MODE == M_DGRAD && EPI != BNFF_DG_PLAIN;
    const bool nrc = MODE == M_DGRAD && EPI >= BNFF_DG_NRC;
    // out (+)= scale * dt1: the ICF fold exists for 1x1 dgrads only (the host rejects it for 3x3),
    // so the 3x3 instantiations carry no fold code
    const bool fold = MODE == M_DGRAD && TAPS == 1 && EPI >= BNFF_DG_NRC_ACC && (!F32 || L::TST);
    const bool fold_acc = MODE == M_DGRAD && TAPS == 1 && EPI == BNFF_DG_NRC_ACC && (!F32 || L::TST);
    E* const outp = reinterpret_cast<E*>(p.out);
    const E* const exq = reinterpret_cast<const E*>(p.ex);
    constexpr int EPC = 16 / ES;             // elements per 16-byte chunk
    // TMA-store epilogue (64-column chunks): the staged chunk leaves by one bulk tensor store;
    // the 1x1 fold also loads the old block-gradient tile by TMA one tile ahead, folds it in
    // place in shared memory during the row pass and stores it back
    // 64-column chunks always take the TMA path (the host encodes the descriptors or declines the
    // window kernel), so the register-store / register-fold variants exist for narrow chunks only
    const bool tfold = L::TST && fold;  // == gb_s (fold_tma)
    constexpr bool tst = L::TST;
    uint8_t* gb0 = smem + cv.gbuf + grp * MYCH * 128 * 128;
    const bool tx = tst && need_x;  // x tiles by TMA into 128B-swizzled rows
    // 3x3 boxes cover kt*wp (or kt*hp*wp) rows; the rows below never receive data: zero once
    const int xrows = TAPS == 1 ? 128 : p.wp * (p.tmode == 2 ? p.hp * p.kt : p.kt);
    if (tx && TAPS == 9 && row >= xrows) {
#pragma unroll
      for (int k = 0; k < MYCH; ++k)
#pragma unroll
        for (int i = 0; i < 8; ++i)
          *reinterpret_cast<uint4*>(xs0 + k * L::STG + row * 128 + i * 16) = make_uint4(0, 0, 0, 0);
    }
    const bool stats = do_stats && (MODE == M_FPROP || nrc);
    const bool persist = true;  // grid % ntiles == 0: a CTA's columns never change, sums stay in registers
    struct D2 { double x, y; };
    using P2 = typename std::conditional<F32, D2, float2>::type;  // a column pair's running sums
    P2 acc1[MYCH], acc2[MYCH];
#pragma unroll
    for (int k = 0; k < MYCH; ++k) { acc1[k] = P2{SA(0), SA(0)}; acc2[k] = P2{SA(0), SA(0)}; }
    auto out_pix = [&](int mt, int m) {
      // output row m of m-tile mt -> output pixel (or -1: a padding column / row past the map)
      if (TAPS == 1) {
        const int q = mt * 128 + m;
        return q < p.P ? q : -1;
      }
      int img0, y0;
      tile_org(mt, img0, y0);
      int i = 0, rem = m;
      if (p.tmode == 2) {
        i = (int)fdiv((uint32_t)m, p.fd_hpwp);
        rem = m - i * hpwp;
      }
      const int yo = (int)fdiv((uint32_t)rem, p.fd_wp);
      const int x = rem - yo * p.wp;
      const int y = y0 + 1 + yo;
      const bool ok = x < p.w && y < p.h && (p.tmode == 2 ? (i < p.kt && img0 + i < p.n) : yo < p.kt);
      return ok ? ((img0 + i) * p.h + y) * p.w + x : -1;
    };
    // one commit group per (tile, owned chunk), issued in order; empty groups keep the count
    auto fetch_x = [&](int it2, int k) {
      if (tx) {
        if (gt == 0 && it2 < ntl && grp + 2 * k < NCH) {
          int mtb, n0b;
          tile_of(it2, mtb, n0b);
          const int col = n0b + (grp + 2 * k) * CW;
          const uint32_t dst = smem_u32(xs0 + k * L::STG);
          mbar_arrive_expect_tx(&x_bar[grp * 2 + k], xrows * 128);
          if (TAPS == 1) {
            tma_load_2d(dst, &p.tma_ex, col, mtb * 128, &x_bar[grp * 2 + k]);
          } else {
            int img0, y0;
            tile_org(mtb, img0, y0);
            tma_load_4d(dst, &p.tma_ex, col, 0, p.tmode == 2 ? 0 : y0 + 1, img0, &x_bar[grp * 2 + k]);
          }
        }
        return;
      }
      if (need_x && it2 < ntl && grp + 2 * k < NCH) {
        int mtb, n0b;
        tile_of(it2, mtb, n0b);
        const int pix = out_pix(mtb, row);
        const uint32_t dst = smem_u32(xs0 + k * L::STG + row * L::SROWB);
        const int col = n0b + (grp + 2 * k) * CW;
        const bool ok = pix >= 0 && col < p.N;
#pragma unroll
        for (int i = 0; i < CW / EPC; ++i)
          cp_async16(dst + i * 16, exq + (ok ? (long long)pix * p.ex_rs + col + i * EPC : 0), ok ? 16u : 0u);
      }
      cp_async_commit();
    };
    // fixed-order combine of one chunk's register sums: into sacc (one N tile) or into
    // this CTA's global partial row (several N tiles; only this thread touches the column)
    auto flush = [&](int k, int n0, int cc) {
      gred[(rg * 4 + 0) * HALF + cp] = acc1[k].x;
      gred[(rg * 4 + 1) * HALF + cp] = acc1[k].y;
      gred[(rg * 4 + 2) * HALF + cp] = acc2[k].x;
      gred[(rg * 4 + 3) * HALF + cp] = acc2[k].y;
      acc1[k] = P2{SA(0), SA(0)};
      acc2[k] = P2{SA(0), SA(0)};
      named_bar_sync(bar_id, 128);
      if (gt < CW) {
        const int c = gt, pc = c >> 1, odd = c & 1;
        SA s1 = SA(0), s2 = SA(0);
        for (int q = 0; q < RG; ++q) {
          s1 += gred[(q * 4 + odd) * HALF + pc];
          s2 += gred[(q * 4 + 2 + odd) * HALF + pc];
        }
        const int gcol = n0 + cc + c;
        if (gcol < p.N) {
          if (persist) {
            sacc[cc + c] += s1;
            sacc[BN + cc + c] += s2;
          } else {
            double* rowp = p.stat_part + (long long)blockIdx.x * 2 * p.N;
            rowp[gcol] += s1;
            rowp[p.N + gcol] += s2;
          }
        }
      }
      named_bar_sync(bar_id, 128);
    };
    auto fetch_g = [&](int it2, int k) {  // one thread of the group; the buffer is free
      if (tfold && fold_acc && it2 < ntl && grp + 2 * k < NCH) {
        int mtb, n0b;
        tile_of(it2, mtb, n0b);
        mbar_arrive_expect_tx(&g_bar[grp * 2 + k], 128 * 128);
        tma_load_2d(smem_u32(gb0 + k * 128 * 128), &p.tma_out, n0b + (grp + 2 * k) * CW, mtb * 128,
                    &g_bar[grp * 2 + k]);
      }
    };
#pragma unroll
    for (int k = 0; k < MYCH; ++k) {
      fetch_x(0, k);
      if (gt == 0) fetch_g(0, k);
    }
    for (int it = 0; it < ntl; ++it) {
      const int buf = it & 1;
      int mt, n0;
      tile_of(it, mt, n0);
      gpix[row] = out_pix(mt, row);
      if (MODE == M_DGRAD && fold_acc && !tfold) named_bar_sync(bar_id, 128);  // gpix of every row for the prefetch
      const int pix = gpix[row];
      mbar_wait(&accf_bar[buf], (it >> 1) & 1);
      if (et == 0) trace_ev(p.trace, 6, it);
      tc_fence_after();
#pragma unroll
      for (int k = 0; k < MYCH; ++k) {
        const int ci = grp + 2 * k;
        if (ci >= NCH) break;
        const int cc = ci * CW;
        uint4 gold[CW / 8];
        if (MODE == M_DGRAD && fold_acc && !tfold) {  // prefetch the old block-gradient chunks this thread stores
          constexpr int CPO = CW / 8;
#pragma unroll
          for (int i = 0; i < CPO; ++i) {
            const int kk = gt + 128 * i;
            const int r = kk / CPO, ch = kk - r * CPO;
            const int px = gpix[r];
            const int col = n0 + cc + ch * 8;
            gold[i] = (px >= 0 && col < p.N)
                          ? *reinterpret_cast<const uint4*>(outp + (long long)px * p.out_rs + col)
                          : make_uint4(0, 0, 0, 0);
          }
        } else {
#pragma unroll
          for (int i = 0; i < CW / 8; ++i) gold[i] = make_uint4(0, 0, 0, 0);
        }
        if (tx) mbar_wait(&x_bar[grp * 2 + k], it & 1);
        else if (need_x) cp_async_wait<MYCH - 1>();
        if (tfold && fold_acc) mbar_wait(&g_bar[grp * 2 + k], it & 1);
        const uint8_t* xrow = xs0 + k * L::STG + row * L::SROWB;
        if (et == 0) trace_ev(p.trace, 10, it * 4 + k);
        // ---- row pass
#pragma unroll
        for (int c16 = 0; c16 < CW; c16 += 16) {
          float v[16];
          tmem_ld16(tmem + buf * L::ACOLS + cc + c16 + ((uint32_t)(quad * 32) << 16), v);
          if constexpr (F32 && BNFF_TF32_STACK) {  // + the cross-term half (hi*lo + lo*hi)
            float v2[16];
            tmem_ld16(tmem + buf * L::ACOLS + BN + cc + c16 + ((uint32_t)(quad * 32) << 16), v2);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] += v2[i];
          } else {
            tmem_ld_wait();
          }
          const int gc = n0 + cc + c16;
          if (MODE == M_FPROP) {
            float bv[16];
            ld16f(etab + gc, bv);
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = pix >= 0 ? v[i] + bv[i] : 0.f;
          } else {
            if (need_x) {
              float xv[16];
              if constexpr (F32) {  // 16 fp32 = four 16-byte chunks
                const uint8_t* xb = xs0 + k * L::STG + row * (tx ? 128 : L::SROWB);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  const int j = (c16 >> 2) + q;
                  const float4 t = *reinterpret_cast<const float4*>(xb + (tx ? ((j ^ (row & 7)) << 4) : j * 16));
                  xv[4 * q] = t.x; xv[4 * q + 1] = t.y; xv[4 * q + 2] = t.z; xv[4 * q + 3] = t.w;
                }
              } else if (tx) {
                const uint8_t* xb = xs0 + k * L::STG + row * 128;
                const int j = c16 >> 3;
                unpack8(*reinterpret_cast<const uint4*>(xb + ((j ^ (row & 7)) << 4)), xv);
                unpack8(*reinterpret_cast<const uint4*>(xb + (((j + 1) ^ (row & 7)) << 4)), xv + 8);
              } else {
                unpack8(*reinterpret_cast<const uint4*>(xrow + c16 * 2), xv);
                unpack8(*reinterpret_cast<const uint4*>(xrow + c16 * 2 + 16), xv + 8);
              }
              if (EPI == BNFF_DG_CLIP) {
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] = xv[i] > 0.f ? v[i] : 0.f;
              } else {
                float e0[16], e1[16];
                ld16f(etab + gc, e0);
                ld16f(etab + p.npad + gc, e1);
#pragma unroll
                for (int i = 0; i < 16; i += 2) {
                  const float2 z = __ffma2_rn(make_float2(xv[i], xv[i + 1]), make_float2(e0[i], e0[i + 1]),
                                              make_float2(e1[i], e1[i + 1]));
                  v[i] = z.x > 0.f ? v[i] : 0.f;
                  v[i + 1] = z.y > 0.f ? v[i + 1] : 0.f;
                }
              }
            }
            if (pix < 0) {
#pragma unroll
              for (int i = 0; i < 16; ++i) v[i] = 0.f;
            }
          }
          if constexpr (F32) {  // fp32 staging: 16 values = four 16-byte chunks
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int j = (c16 >> 2) + q;
              const uint32_t o = tst ? row * 128 + ((j ^ (row & 7)) << 4) : row * L::SROWB + j * 16;
              const float4 vv = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
              *reinterpret_cast<float4*>(stg + o) = vv;
              if (MODE == M_DGRAD && tfold) {  // G = (acc ? G : 0) + scale * dt1, in the TMA G tile
                uint8_t* gt0 = gb0 + k * 128 * 128;
                const float* sc = etab + gc + 4 * q;
                float4 d;
                if (fold_acc) {
                  const float4 old = *reinterpret_cast<const float4*>(gt0 + o);
                  d = make_float4(fmaf(sc[0], vv.x, old.x), fmaf(sc[1], vv.y, old.y), fmaf(sc[2], vv.z, old.z),
                                  fmaf(sc[3], vv.w, old.w));
                } else {
                  d = make_float4(sc[0] * vv.x, sc[1] * vv.y, sc[2] * vv.z, sc[3] * vv.w);
                }
                *reinterpret_cast<float4*>(gt0 + o) = d;
              }
            }
          } else if (tst) {  // dense 128-byte rows, 128B swizzle (the TMA store's box layout)
            const int j = c16 >> 3;
            const int o0 = row * 128 + ((j ^ (row & 7)) << 4), o1 = row * 128 + (((j + 1) ^ (row & 7)) << 4);
            *reinterpret_cast<uint4*>(stg + o0) = pack8(v, false);
            *reinterpret_cast<uint4*>(stg + o1) = pack8(v + 8, false);
            if (MODE == M_DGRAD && tfold) {  // G = (acc ? G : 0) + scale * dt1 (dt1 rounded like the store)
              uint8_t* gt0 = gb0 + k * 128 * 128;
              float sc[16], d[16];
              ld16f(etab + gc, sc);
              const uint4 r0 = pack8(v, false), r1 = pack8(v + 8, false);
              unpack8(r0, d);
              unpack8(r1, d + 8);
              if (fold_acc) {
                float o[16];
                unpack8(*reinterpret_cast<const uint4*>(gt0 + o0), o);
                unpack8(*reinterpret_cast<const uint4*>(gt0 + o1), o + 8);
#pragma unroll
                for (int i = 0; i < 16; i += 2) {
                  const float2 z = __ffma2_rn(make_float2(sc[i], sc[i + 1]), make_float2(d[i], d[i + 1]),
                                              make_float2(o[i], o[i + 1]));
                  d[i] = z.x;
                  d[i + 1] = z.y;
                }
              } else {
#pragma unroll
                for (int i = 0; i < 16; ++i) d[i] = sc[i] * d[i];
              }
              *reinterpret_cast<uint4*>(gt0 + o0) = pack8(d, false);
              *reinterpret_cast<uint4*>(gt0 + o1) = pack8(d + 8, false);
            }
          } else {
            uint4* sp = reinterpret_cast<uint4*>(stg + row * L::SROWB + c16 * 2);
            sp[0] = pack8(v, false);
            sp[1] = pack8(v + 8, false);
          }
        }
        if (ci + 2 >= NCH) {
          tc_fence_before();
          mbar_arrive(&acce_bar[buf]);  // this group is done with the accumulator slot
          if (et == 0) trace_ev(p.trace, 7, it);
        }
        if (tst) fence_proxy_async_smem();  // staged rows -> visible to the TMA engine
        named_bar_sync(bar_id, 128);
        if (tst && gt == 0) {  // one thread stores the whole staged chunk, asynchronously
          if (TAPS == 1) {
            tma_store_2d(&p.tma_out, n0 + cc, mt * 128, smem_u32(tfold ? gb0 + k * 128 * 128 : stg));
          } else {
            int img0, y0;
            tile_org(mt, img0, y0);
            tma_store_4d(&p.tma_out, n0 + cc, 0, p.tmode == 2 ? 0 : y0 + 1, img0, smem_u32(stg));
          }
          bulk_commit();
        }
        if (et == 0) trace_ev(p.trace, 11, it * 4 + k);
        // ---- column pass: sums of the stored values (FPROP: y, y^2; NRC: dt1, dt1*xhat)
        if (stats && F32) {  // fp32 staging: a column pair is 8 bytes; float64 sums
          const float* sf = reinterpret_cast<const float*>(stg);
          const float* xf = reinterpret_cast<const float*>(xs0 + k * L::STG);
          SA a0 = acc1[k].x, a1 = acc1[k].y, b0 = acc2[k].x, b1 = acc2[k].y;
          const int gc = n0 + cc + 2 * cp;
          float hinv0 = 0.f, hinv1 = 0.f, hsh0 = 0.f, hsh1 = 0.f;
          if (MODE == M_DGRAD) {
            hinv0 = etab[2 * p.npad + gc]; hinv1 = etab[2 * p.npad + gc + 1];
            hsh0 = etab[3 * p.npad + gc]; hsh1 = etab[3 * p.npad + gc + 1];
          }
#pragma unroll 16
          for (int r = rg; r < 128; r += RG) {
            const int w = tst ? r * 32 + ((((cp >> 1) ^ (r & 7)) << 2) | ((2 * cp) & 3)) : r * (L::SROWB / 4) + 2 * cp;
            const float f0 = sf[w], f1 = sf[w + 1];
            a0 += (SA)f0;
            a1 += (SA)f1;
            if (MODE == M_FPROP) {
              b0 += (SA)f0 * (SA)f0;
              b1 += (SA)f1 * (SA)f1;
            } else {
              const int wx = tx ? r * 32 + ((((cp >> 1) ^ (r & 7)) << 2) | ((2 * cp) & 3)) : r * (L::SROWB / 4) + 2 * cp;
              b0 += (SA)f0 * (SA)fmaf(xf[wx], hinv0, hsh0);
              b1 += (SA)f1 * (SA)fmaf(xf[wx + 1], hinv1, hsh1);
            }
          }
          acc1[k] = P2{a0, a1};
          acc2[k] = P2{b0, b1};
        } else if (stats) {
          const uint32_t* s32 = reinterpret_cast<const uint32_t*>(stg);
          float2 a = make_float2((float)acc1[k].x, (float)acc1[k].y);
          float2 b = make_float2((float)acc2[k].x, (float)acc2[k].y);
          if (MODE == M_FPROP) {
#pragma unroll 32
            for (int r = rg; r < 128; r += RG) {
              const uint32_t wv = tst ? s32[r * 32 + ((((cp >> 2) ^ (r & 7)) << 2) | (cp & 3))]
                                      : s32[r * (L::SROWB / 4) + cp];
              const float2 f = make_float2(bf16lo(wv), bf16hi(wv));
              a = __fadd2_rn(a, f);
              b = __ffma2_rn(f, f, b);
            }
          } else {
            const uint32_t* x32 = reinterpret_cast<const uint32_t*>(xs0 + k * L::STG);
            const int gc = n0 + cc + 2 * cp;
            const float2 hinv = make_float2(etab[2 * p.npad + gc], etab[2 * p.npad + gc + 1]);
            const float2 hsh = make_float2(etab[3 * p.npad + gc], etab[3 * p.npad + gc + 1]);
#pragma unroll 32
            for (int r = rg; r < 128; r += RG) {
              const uint32_t wv = tst ? s32[r * 32 + ((((cp >> 2) ^ (r & 7)) << 2) | (cp & 3))]
                                      : s32[r * (L::SROWB / 4) + cp];
              const uint32_t xw = tx ? x32[r * 32 + ((((cp >> 2) ^ (r & 7)) << 2) | (cp & 3))]
                                     : x32[r * (L::SROWB / 4) + cp];
              const float2 f = make_float2(bf16lo(wv), bf16hi(wv));
              const float2 xh = __ffma2_rn(make_float2(bf16lo(xw), bf16hi(xw)), hinv, hsh);
              a = __fadd2_rn(a, f);
              b = __ffma2_rn(f, xh, b);
            }
          }
          acc1[k] = P2{a.x, a.y};
          acc2[k] = P2{b.x, b.y};
        }
        if (et == 0) trace_ev(p.trace, 12, it * 4 + k);
        // ---- store pass
        constexpr int CPO = CW / 8;  // 16B chunks per staged row
        if (MODE == M_DGRAD && fold && !tfold) {
          // block-gradient fold: out = (acc ? out : 0) + scale * dt1; the old block-gradient
          // chunks were fetched into registers before the row pass (their latency hides there)
#pragma unroll
          for (int i = 0; i < CPO; ++i) {
            const int kk = gt + 128 * i;
            const int r = kk / CPO, ch = kk - r * CPO;
            const int px = gpix[r];
            const int col = n0 + cc + ch * 8;
            if (px >= 0 && col < p.N) {
              float d[8], sc[8], o[8];
              unpack8(*reinterpret_cast<const uint4*>(stg + r * L::SROWB + ch * 16), d);
              ld8f(etab + col, sc);
              unpack8(gold[i], o);
#pragma unroll
              for (int e = 0; e < 8; ++e) d[e] = fold_acc ? fmaf(sc[e], d[e], o[e]) : sc[e] * d[e];
              *reinterpret_cast<uint4*>(outp + (long long)px * p.out_rs + col) = pack8(d, false);
            }
          }
        } else if (tst) {
          if (gt == 0) {
            bulk_wait_read0();  // the staging tile is read before it is rewritten
            fetch_g(it + 1, k); // the fold tile is free: fetch the next tile's old block gradient
          }
        } else {
          constexpr int CPS = CW * ES / 16;  // 16-byte chunks per staged row
#pragma unroll 2
          for (int kk = gt; kk < 128 * CPS; kk += 128) {
            const int r = kk / CPS, ch = kk - r * CPS;
            const int px = gpix[r];
            const int col = n0 + cc + ch * EPC;
            if (px >= 0 && col < p.N) {
              const uint4 vv = *reinterpret_cast<const uint4*>(stg + r * L::SROWB + ch * 16);
              *reinterpret_cast<uint4*>(outp + (long long)px * p.out_rs + col) = vv;
            }
          }
        }
        named_bar_sync(bar_id, 128);  // staging, x buffer k and gpix free
        if (et == 0) trace_ev(p.trace, 13, it * 4 + k);
        fetch_x(it + 1, k);            // recycle x buffer k for the next tile
        if (stats && !persist) flush(k, n0, cc);
      }
    }
    cp_async_wait<0>();
    if (tst && gt == 0) bulk_wait_all0();  // outstanding TMA stores complete before exit
    if (stats && persist) {
#pragma unroll
      for (int k = 0; k < MYCH; ++k)
        if (grp + 2 * k < NCH) flush(k, 0, (grp + 2 * k) * CW);
    }
    // both groups' sums are in sacc; write this CTA's partial row (one N tile)
    asm volatile("bar.sync 4, %0;" ::"n"(NEW * 32) : "memory");
    if (do_stats && persist && ntl > 0) {
      int mt0, n00;
      tile_of(0, mt0, n00);
      for (int c = et; c < BN; c += NEW * 32) {
        if (n00 + c >= p.N) continue;
        p.stat_part[((long long)blockIdx.x * 2 + 0) * p.N + n00 + c] = sacc[c];
        p.stat_part[((long long)blockIdx.x * 2 + 1) * p.N + n00 + c] = sacc[BN + c];
      }
    }
    };
    if (MODE == M_FPROP) {
      epilogue(std::integral_constant<int, BNFF_DG_PLAIN>{});
    } else {
      switch (p.epi) {
        case BNFF_DG_CLIP: epilogue(std::integral_constant<int, BNFF_DG_CLIP>{}); break;
        case BNFF_DG_NRC: epilogue(std::integral_constant<int, BNFF_DG_NRC>{}); break;
        case BNFF_DG_NRC_ACC:
          if constexpr (TAPS == 1) epilogue(std::integral_constant<int, BNFF_DG_NRC_ACC>{});
          break;
        case BNFF_DG_NRC_SET:
          if constexpr (TAPS == 1) epilogue(std::integral_constant<int, BNFF_DG_NRC_SET>{});
          break;
        default: epilogue(std::integral_constant<int, BNFF_DG_PLAIN>{}); break;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == NLW) tmem_dealloc<L::TCOLS>(tmem);
}

// ===========================================================================
// WGRAD:  dW[tap][ci][co] = sum_m  P_x[m + s_tap, ci] * G[m, co]
// K runs over the output positions of a k-block -- the same row/image-aligned tiles as
// the forward window kernel (3x3: kt padded output rows of one image, or kt whole
// images; 1x1: 128 pixels).  A = P_x, the TMA window of the tile with its zero halo
// (MN-major: 128-byte rows of 64 input channels per atom; all 9 taps read it through
// K-shifted descriptors), B = G = pro(dy) at the tile's output positions (MN-major,
// zero outside the map).  A CTA owns one work unit (m-group of MT*128 input channels,
// N tile, K split) at a time and keeps TAPS*MT accumulators of BN columns in TMEM;
// fp32 partials go to a workspace reduced in fixed split order (deterministic).
// Warp roles: 8 transform warps (prologues in place, dbias), 1 MMA warp, 4 epilogue
// warps, 1 TMA producer warp.
// ===========================================================================
int num_sms_wc();

constexpr int WG_THREADS = (NLW + 1 + 4 + 1) * 32;
constexpr int WG_PRODUCER = NLW + 1 + 4;

struct WgParams {
  CUtensorMap tma_x, tma_dy, tma_dyx;
  int tmode, kt, BR, BI, WPI, tpi, Rld, Kr, P;
  int n, h, w, hp, wp, pad, Q;
  FastDiv fd_hpwp, fd_wp;
  int cin, cout, KB, RA, nkb, kpt, splits, MG, NT, units, stages;
  int x_pro;
  bnff_coef x_coef;
  int dy_pro;
  bnff_coef dy_coef;
  float* ws;
  float* wsb;  // nullable: dbias partials [splits][cout] (m-group 0 units)
};

template <int BN, int MT, int TAPS, int KB>
struct WgL {
  static constexpr int BRB = BN * 2 >= 128 ? 128 : BN * 2;  // B row bytes per atom
  static constexpr int NBA = BN * 2 / BRB;                   // B atoms
  static constexpr int BCPR = BRB / 16;                      // B chunks per row per atom
  static constexpr int BCH = NBA * BCPR;                     // B chunks per row
  static constexpr int RAMAX = TAPS == 9 ? RMAX : KB;        // A rows (allocated, max)
  static constexpr int AAT = 2 * MT;                         // A atoms
  static constexpr int UAR = RAMAX / 32;                     // A rows per thread per atom
  static constexpr int UB = KB * BCH / LT;                   // B chunks per thread
  static constexpr uint32_t BLAY = BRB == 128 ? kLayoutSW128 : kLayoutSW64;
  static constexpr int NACC = TAPS * MT;
  static constexpr int TCOLS = NACC * BN <= 32 ? 32 : (NACC * BN <= 64 ? 64 : (NACC * BN <= 128 ? 128 : (NACC * BN <= 256 ? 256 : 512)));
  static_assert(NACC * BN <= 512, "TMEM");
  static_assert(KB * BCH % LT == 0, "B mapping");
};

struct WgCarve {
  int stage_bytes, a_bytes, b_bytes, ptab, qtab, rowx, rowg, meta, bred, total;
};
template <int BN, int MT, int TAPS, int KB>
__host__ __device__ inline WgCarve wg_carve(int RA, int cin_pad, int npad, int stages, bool xop) {
  using L = WgL<BN, MT, TAPS, KB>;
  WgCarve c{};
  c.a_bytes = L::AAT * RA * 128;
  c.b_bytes = L::NBA * KB * L::BRB;
  c.stage_bytes = align_up(c.a_bytes + (xop ? 2 : 1) * c.b_bytes, 1024);  // A | B | X(dy_x)
  int off = stages * c.stage_bytes;
  c.ptab = off;
  off += 2 * cin_pad * 4;
  c.qtab = off;
  off += 3 * npad * 4;
  c.rowx = off;  // window row -> (image block, padded row, padded column)
  off += RMAX * 4;
  c.rowg = off;  // k-block row -> (image block, output row, column)
  off += KB * 4;
  c.meta = off;
  c.bred = off;
  off += 8 * LT * 4;
  c.total = off + 1024;
  return c;
}

template <int BN, int MT, int TAPS, int KB>
__global__ void __launch_bounds__(WG_THREADS, 1) wgrad_kernel(const __grid_constant__ WgParams p) {
  griddep_launch();
  using L = WgL<BN, MT, TAPS, KB>;
  extern __shared__ uint8_t dsm_raw[];
  // offset (not integer-cast) the shared array so the compiler keeps the shared state space
  uint8_t* smem = dsm_raw + ((1024u - (smem_u32(dsm_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full_bar[8], empty_bar[8], ld_bar[8], accf_bar, acce_bar;
  __shared__ uint32_t tmem_sh;
  const int cin_pad = p.MG * MT * 128, npad = p.NT * BN;
  const WgCarve cv = wg_carve<BN, MT, TAPS, KB>(p.RA, cin_pad, npad, p.stages, p.dy_pro == BNFF_PRO_BN_DX);
  const int ST = p.stages;
  float* ptab = reinterpret_cast<float*>(smem + cv.ptab);
  float* qtab = reinterpret_cast<float*>(smem + cv.qtab);
  int* rowx = reinterpret_cast<int*>(smem + cv.rowx);
  int* rowg = reinterpret_cast<int*>(smem + cv.rowg);
  float* bred = reinterpret_cast<float*>(smem + cv.bred);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nun = (p.units - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  const bool xb = p.dy_pro == BNFF_PRO_BN_DX;

  if (tid == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full_bar[s], LT);
      mbar_init(&empty_bar[s], 1);
      mbar_init(&ld_bar[s], 1);
    }
    mbar_init(&accf_bar, 1);
    mbar_init(&acce_bar, 128);
    fence_mbar_init();
    tma_prefetch_desc(&p.tma_x);
    tma_prefetch_desc(&p.tma_dy);
    if (xb) tma_prefetch_desc(&p.tma_dyx);
  }
  if (warp == NLW) tmem_alloc<L::TCOLS>(&tmem_sh);
  // stage buffers start zeroed: rows past what the TMA writes (the K tail of B, the A
  // rows beyond the window) must be finite zeros for the full-K MMAs
  for (int i = tid; i < ST * cv.stage_bytes / 16; i += WG_THREADS)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  // row geometry tables (identical for every k-block)
  if (TAPS == 9) {
    for (int r = tid; r < p.Rld; r += WG_THREADS) {
      const int i = r / p.WPI, rem = r - i * p.WPI;
      const int ry = rem / p.wp, rx = rem - ry * p.wp;
      rowx[r] = (i << 20) | (ry << 10) | rx;
    }
    const int opi = p.tmode == 2 ? p.hp * p.wp : KB;
    for (int m = tid; m < KB; m += WG_THREADS) {
      const int i = m / opi, rem = m - i * opi;
      const int yo = rem / p.wp, x = rem - yo * p.wp;
      rowg[m] = (i << 20) | (yo << 10) | x;
    }
  }
  fence_proxy_async_smem();  // zeroed stage buffers -> visible to the async proxy (TMA, UMMA)
  __syncthreads();           // ... and the barrier initialisation to every role
  griddep_wait();            // everything below reads data of the preceding launches
  // the producer warp (the last warp) starts streaming at once; the others build the tables
  constexpr int GS_THREADS = WG_THREADS - 32;
  static_assert(WG_PRODUCER * 32 == GS_THREADS, "producer is the last warp");
  if (warp != WG_PRODUCER) {
  for (int c = tid; c < cin_pad; c += GS_THREADS) {  // x prologue: (scale, beta - mean*scale)
    float t0 = 1.f, t1 = 0.f;
    if (c < p.cin && p.x_pro == BNFF_PRO_BN_RELU) {
      t0 = p.x_coef.b[c];
      t1 = p.x_coef.c[c] - p.x_coef.a[c] * t0;
    }
    ptab[c] = t0;
    ptab[cin_pad + c] = t1;
  }
  for (int c = tid; c < npad; c += GS_THREADS) {  // dy prologue (BN_DX)
    float t0 = 1.f, t1 = 0.f, t2 = 0.f;
    if (c < p.cout && xb) {
      const float m = p.dy_coef.a[c], inv = p.dy_coef.b[c], k1 = p.dy_coef.c[c],
                  k2 = p.dy_coef.d[c], g = p.dy_coef.e[c];
      t0 = g;
      t1 = -g * k2 * inv;
      t2 = g * (k2 * inv * m - k1);
    }
    qtab[c] = t0;
    qtab[npad + c] = t1;
    qtab[2 * npad + c] = t2;
  }
  tc_fence_before();
  asm volatile("bar.sync 6, %0;" ::"n"(GS_THREADS) : "memory");
  tc_fence_after();
  }
  const uint32_t tmem = tmem_sh;
  auto unit_of = [&](int ui, int& mg, int& nt, int& sp) {
    const int u = (int)blockIdx.x + ui * (int)gridDim.x;
    sp = u % p.splits;
    const int r = u / p.splits;
    nt = r % p.NT;
    mg = r / p.NT;
  };
  auto stage_a = [&](int s) { return smem + s * cv.stage_bytes; };
  auto stage_b = [&](int s) { return smem + s * cv.stage_bytes + cv.a_bytes; };
  auto stage_x = [&](int s) { return smem + s * cv.stage_bytes + cv.a_bytes + cv.b_bytes; };
  auto kb_count = [&](int sp) { return min(p.kpt, p.nkb - sp * p.kpt); };
  // k-block origin: first image and the padded-input row the window starts at (3x3)
  auto kb_org = [&](int kb, int& img0, int& y0) {
    if (p.tmode == 1) {
      img0 = kb / p.tpi;
      y0 = (kb - img0 * p.tpi) * p.kt - 1;
    } else {
      img0 = kb * p.kt;
      y0 = -1;
    }
  };

  if (warp < NLW) {
    // =============================== transform warps ===============================
    const int ja = tid & 7, ra0 = tid >> 3;                 // A: chunk column, first row
    const int jb = tid % L::BCH, rb0 = tid / L::BCH;        // B: chunk column, first row
    constexpr int RBS = LT / L::BCH;                        // B row step
    const bool need_a = p.x_pro != BNFF_PRO_NONE;
    const bool need_db = p.wsb != nullptr;
    float bacc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) bacc[i] = 0.f;
    int st = 0;
    uint32_t ph = 0;
    for (int ui = 0; ui < nun; ++ui) {
      int mg, nt, sp;
      unit_of(ui, mg, nt, sp);
      const int cnt = kb_count(sp);
      const int co0 = nt * BN + jb * 8;
      const bool bact = (xb || (need_db && mg == 0)) && co0 < p.cout;
      float q0[8], q1[8], q2[8];
      if (xb && co0 < p.cout) {
        ld8f(qtab + co0, q0);
        ld8f(qtab + npad + co0, q1);
        ld8f(qtab + 2 * npad + co0, q2);
      }
      for (int k = 0; k < cnt; ++k) {
        const int kb = sp * p.kpt + k;
        int img0 = 0, y0 = 0;
        if (TAPS == 9) kb_org(kb, img0, y0);
        mbar_wait(&ld_bar[st], ph);
        bool wrote = false;
        if (need_a) {
          uint8_t* A = stage_a(st);
#pragma unroll
          for (int a = 0; a < L::AAT; ++a) {
            const int c0 = mg * MT * 128 + a * 64 + ja * 8;
            if (c0 >= p.cin) continue;
            float t0[8], t1[8];
            ld8f(ptab + c0, t0);
            ld8f(ptab + cin_pad + c0, t1);
#pragma unroll 4
            for (int u = 0; u < L::UAR; ++u) {
              const int r = ra0 + 32 * u;
              if (r >= p.Rld) break;
              if (TAPS == 9) {  // halo / border positions stay zero
                const int wr = rowx[r];
                const int y = y0 + ((wr >> 10) & 1023), rx = wr & 1023;
                if ((unsigned)y >= (unsigned)p.h || rx < 1 || rx > p.w || img0 + (wr >> 20) >= p.n) continue;
              }
              const uint32_t off = a * p.RA * 128 + r * 128 + ((ja ^ (r & 7)) << 4);
              float f[8];
              unpack8(*reinterpret_cast<const uint4*>(A + off), f);
              if (p.x_pro == BNFF_PRO_BN_RELU) {
#pragma unroll
                for (int i = 0; i < 8; ++i) f[i] = fmaf(f[i], t0[i], t1[i]);
              }
              *reinterpret_cast<uint4*>(A + off) = pack8(f, true);
            }
          }
          wrote = true;
        }
        if (bact) {
          uint8_t* B = stage_b(st);
          const uint8_t* X = stage_x(st);
#pragma unroll
          for (int u = 0; u < L::UB; ++u) {
            const int r = rb0 + RBS * u;
            if (r >= p.Kr) break;
            bool ok;
            if (TAPS == 9) {
              const int wr = rowg[r];
              const int i = wr >> 20, yo = (wr >> 10) & 1023, x = wr & 1023;
              const int y = y0 + 1 + yo;
              ok = x < p.w && y < p.h && (p.tmode == 2 ? img0 + i < p.n : yo < p.kt);
            } else {
              ok = kb * KB + r < p.P;
            }
            if (!ok) continue;
            const int b = jb / L::BCPR, jj = jb % L::BCPR;
            uint32_t off = b * KB * L::BRB + r * L::BRB;
            if constexpr (L::BRB == 128) off += (jj ^ (r & 7)) << 4;
            else off += (jj ^ ((r >> 1) & 3)) << 4;
            float f[8];
            unpack8(*reinterpret_cast<const uint4*>(B + off), f);
            if (xb) {
              float xf[8];
              unpack8(*reinterpret_cast<const uint4*>(X + off), xf);
#pragma unroll
              for (int i = 0; i < 8; ++i) f[i] = fmaf(f[i], q0[i], fmaf(xf[i], q1[i], q2[i]));
              const uint4 o = pack8(f, false);
              *reinterpret_cast<uint4*>(B + off) = o;
              unpack8(o, f);  // dbias sums the operand the MMA sees
            }
            if (need_db && mg == 0) {
#pragma unroll
              for (int i = 0; i < 8; ++i) bacc[i] += f[i];
            }
          }
          wrote = wrote || xb;
        }
        if (wrote) fence_proxy_async_smem();
        mbar_arrive(&full_bar[st]);
        if (++st == ST) { st = 0; ph ^= 1u; }
      }
      if (need_db && mg == 0) {  // fixed-order combine of the unit's dbias partials
#pragma unroll
        for (int i = 0; i < 8; ++i) { bred[i * LT + tid] = bacc[i]; bacc[i] = 0.f; }
        named_bar_sync(1, LT);
        if (tid < L::BCH * 8) {
          const int jc = tid >> 3, i = tid & 7;
          const int co = nt * BN + jc * 8 + i;
          float sacc = 0.f;
          for (int t = jc; t < LT; t += L::BCH) sacc += bred[i * LT + t];
          if (co < p.cout) p.wsb[(long long)sp * p.cout + co] = sacc;
        }
        named_bar_sync(1, LT);
      }
    }
  } else if (warp == WG_PRODUCER) {
    // =============================== TMA producer ===============================
    {  // converged warp; one elected lane issues the copies
      const uint32_t a_bytes = (uint32_t)p.Rld * 128u * L::AAT;
      const uint32_t b_bytes = (uint32_t)p.Kr * L::BRB * L::NBA;
      const uint32_t tx = a_bytes + b_bytes * (xb ? 2u : 1u);
      int st = 0, round = 0;
      for (int ui = 0; ui < nun; ++ui) {
        int mg, nt, sp;
        unit_of(ui, mg, nt, sp);
        const int cnt = kb_count(sp);
        for (int k = 0; k < cnt; ++k) {
          const int kb = sp * p.kpt + k;
          if (round > 0) mbar_wait(&empty_bar[st], (round - 1) & 1);
          if (elect_one()) {
            mbar_arrive_expect_tx(&ld_bar[st], tx);
            const uint32_t A = smem_u32(stage_a(st)), B = smem_u32(stage_b(st)), X = smem_u32(stage_x(st));
            if (TAPS == 9) {
              int img0, y0;
              kb_org(kb, img0, y0);
              const int oy = y0 + 1;
#pragma unroll
              for (int a = 0; a < L::AAT; ++a)
                tma_load_4d(A + a * p.RA * 128, &p.tma_x, mg * MT * 128 + a * 64, -1, y0, img0, &ld_bar[st]);
#pragma unroll
              for (int b = 0; b < L::NBA; ++b) {
                const int c = nt * BN + b * (L::BRB / 2);
                tma_load_4d(B + b * KB * L::BRB, &p.tma_dy, c, 0, p.tmode == 2 ? 0 : oy, img0, &ld_bar[st]);
                if (xb) tma_load_4d(X + b * KB * L::BRB, &p.tma_dyx, c, 0, p.tmode == 2 ? 0 : oy, img0, &ld_bar[st]);
              }
            } else {
#pragma unroll
              for (int a = 0; a < L::AAT; ++a)
                tma_load_2d(A + a * p.RA * 128, &p.tma_x, mg * MT * 128 + a * 64, kb * KB, &ld_bar[st]);
#pragma unroll
              for (int b = 0; b < L::NBA; ++b) {
                const int c = nt * BN + b * (L::BRB / 2);
                tma_load_2d(B + b * KB * L::BRB, &p.tma_dy, c, kb * KB, &ld_bar[st]);
                if (xb) tma_load_2d(X + b * KB * L::BRB, &p.tma_dyx, c, kb * KB, &ld_bar[st]);
              }
            }
          }
          __syncwarp();
          if (++st == ST) { st = 0; ++round; }
        }
      }
    }
    __syncwarp();
  } else if (warp == NLW) {
    // =============================== MMA issuer ===============================
    {  // converged warp, one elected lane issues (see umma_f16_elect)
      constexpr uint32_t idesc = make_idesc(128, BN, kFmtBF16, 1, 1);
      const int ksteps = (p.Kr + 15) / 16;
      int st = 0;
      uint32_t ph = 0;
      for (int ui = 0; ui < nun; ++ui) {
        int mg, nt, sp;
        unit_of(ui, mg, nt, sp);
        const int cnt = kb_count(sp);
        if (ui >= 1) mbar_wait(&acce_bar, (ui - 1) & 1);
        tc_fence_after();
        for (int k = 0; k < cnt; ++k) {
          mbar_wait(&full_bar[st], ph);
          tc_fence_after();
          const uint32_t abase = smem_u32(stage_a(st)), bbase = smem_u32(stage_b(st));
          const uint64_t a0 = make_sdesc(abase, p.RA * 128, 1024, kLayoutSW128);
          const uint64_t b0 = make_sdesc(bbase, KB * L::BRB, 8 * L::BRB, L::BLAY);
#pragma unroll 1
          for (int u = 0; u < TAPS; ++u) {
            const uint32_t shift = TAPS == 9 ? (uint32_t)((u / 3) * p.wp + (u % 3)) : 0u;
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
              const uint64_t am = a0 + ((2u * mt * p.RA * 128u + shift * 128u) >> 4);
#pragma unroll 1
              for (int kk = 0; kk < ksteps; ++kk) {
                umma_f16_elect(tmem + (u * MT + mt) * BN, am + kk * 128, b0 + ((kk * 16 * L::BRB) >> 4), idesc,
                         (k > 0 || kk > 0) ? 1u : 0u);
              }
            }
          }
          umma_commit_elect(&empty_bar[st]);
          if (++st == ST) { st = 0; ph ^= 1u; }
        }
        umma_commit_elect(&accf_bar);
      }
    }
    __syncwarp();
  } else {
    // =============================== epilogue ===============================
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    for (int ui = 0; ui < nun; ++ui) {
      int mg, nt, sp;
      unit_of(ui, mg, nt, sp);
      mbar_wait(&accf_bar, ui & 1);
      tc_fence_after();
#pragma unroll 1
      for (int u = 0; u < TAPS; ++u) {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const int ci = (mg * MT + mt) * 128 + row;
          float* dst = p.ws + (((long long)sp * TAPS + u) * p.cin + ci) * p.cout + nt * BN;
#pragma unroll 1
          for (int c16 = 0; c16 < BN; c16 += 16) {
            float v[16];
            tmem_ld16(tmem + (u * MT + mt) * BN + c16 + ((uint32_t)(quad * 32) << 16), v);
            tmem_ld_wait();
            if (ci < p.cin && nt * BN + c16 < p.cout) {
#pragma unroll
              for (int q = 0; q < 16; q += 4)
                *reinterpret_cast<float4*>(dst + c16 + q) = make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&acce_bar);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == NLW) tmem_dealloc<L::TCOLS>(tmem);
}

// dW[co][ci][tap] = sum_s ws[s][tap*cin + ci][co]: block = 32 float4 columns x 8 split
// groups; each (group, column) sums its splits in order, then the 8 groups combine in
// order (deterministic).  dbias rides in block 0.
__global__ void __launch_bounds__(256) wg_reduce_kernel(const float* __restrict__ ws, int splits, int taps,
                                                        int cin, int cout, int cin_real,
                                                        float* __restrict__ dw,
                                                        const float* __restrict__ wsb,
                                                        float* __restrict__ dbias) {
  griddep_launch();
  griddep_wait();
  __shared__ float4 sh[8][32];
  const int M = taps * cin;
  const int n4 = cout >> 2;
  const int total = M * n4;
  const long long sstride = (long long)M * cout;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  if (dbias != nullptr && blockIdx.x == 0) {
    for (int c = threadIdx.x; c < cout; c += blockDim.x) {
      float a = 0.f;
      for (int s = 0; s < splits; ++s) a += wsb[(long long)s * cout + c];
      dbias[c] = a;
    }
  }
  for (int base = blockIdx.x * 32; base < total; base += gridDim.x * 32) {
    const int i = base + tx;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i < total) {
      const int m = i / n4, c4 = (i - m * n4) * 4;
      const float* src = ws + (long long)m * cout + c4;
      int s = ty;
      for (; s + 8 < splits; s += 16) {
        const float4 v = *reinterpret_cast<const float4*>(src + s * sstride);
        const float4 w = *reinterpret_cast<const float4*>(src + (s + 8) * sstride);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        acc.x += w.x; acc.y += w.y; acc.z += w.z; acc.w += w.w;
      }
      for (; s < splits; s += 8) {
        const float4 v = *reinterpret_cast<const float4*>(src + s * sstride);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
    }
    sh[ty][tx] = acc;
    __syncthreads();
    if (ty == 0 && i < total) {
      float4 t = sh[0][tx];
      for (int k = 1; k < 8; ++k) {
        const float4 v = sh[k][tx];
        t.x += v.x; t.y += v.y; t.z += v.z; t.w += v.w;
      }
      const int m = i / n4, c4 = (i - m * n4) * 4;
      const int tap = m / cin, ci = m - tap * cin;
      if (ci < cin_real) {
        const float a[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) dw[((long long)(c4 + q) * cin_real + ci) * taps + tap] = a[q];
      }
    }
    __syncthreads();
  }
}

template <int BN, int MT, int TAPS, int KB>
static int launch_wg(WgParams p, cudaStream_t st) {
  auto kern = wgrad_kernel<BN, MT, TAPS, KB>;
  const int cin_pad = p.MG * MT * 128, npad = p.NT * BN;
  const bool xop = p.dy_pro == BNFF_PRO_BN_DX;
  int stages = 8;
  WgCarve c{};
  for (; stages >= 2; --stages) {
    c = wg_carve<BN, MT, TAPS, KB>(p.RA, cin_pad, npad, stages, xop);
    if (c.total <= SMEM_BUDGET) break;
  }
  if (stages < 2) return kWindowNoFit;
  p.stages = stages;
  static int attr = 0;
  if (c.total > attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, c.total);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(wgrad window)");
    attr = c.total;
  }
  const int grid = p.units < num_sms_wc() ? p.units : num_sms_wc();
  launch(kern, dim3(grid), dim3(WG_THREADS), c.total, st, p);
  return check_launch("wgrad window");
}

// ---------------------------------------------------------------------------
// weight packing: fp32 (co, ci, kh, kw) -> pre-swizzled bf16 blocks [slab][tap][npad][RB]
// ---------------------------------------------------------------------------
__global__ void pack_window_kernel(const float* __restrict__ w, int co_n, int ci_n, int kh, int kw,
                                   int dgrad, int CI, int N, int npad, int RB, int nslab,
                                   __nv_bfloat16* __restrict__ out) {
  griddep_launch();
  griddep_wait();
  const int taps = kh * kw;
  const int slabw = RB / 2;
  const long long total = (long long)nslab * taps * npad * slabw;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(i % slabw);
    long long t = i / slabw;
    const int n = (int)(t % npad);
    t /= npad;
    const int u = (int)(t % taps);
    const int s = (int)(t / taps);
    const int ch = s * slabw + k;  // reduction channel
    float v = 0.f;
    if (n < N && ch < CI) {
      int ky = u / kw, kx = u % kw;
      int co, ci;
      if (dgrad) { ky = kh - 1 - ky; kx = kw - 1 - kx; co = ch; ci = n; }
      else { co = n; ci = ch; }
      v = w[(((long long)co * ci_n + ci) * kh + ky) * kw + kx];
    }
    const int kb = k * 2;
    int chunk = kb >> 4;
    chunk ^= RB == 128 ? (n & 7) : ((n >> 1) & 3);
    const long long byte = (((long long)s * taps + u) * npad + n) * RB + chunk * 16 + (kb & 15);
    out[byte / 2] = __float2bfloat16_rn(v);
  }
}

// fp32 (3xTF32) pack: [slab][tap][plane][npad][RB] with plane 0 = TF32(w) (round to nearest),
// plane 1 = TF32(w - hi); slabs of RB/4 channels, same 16-byte chunk swizzle
__device__ __forceinline__ void pack_f32_elem(const float* __restrict__ w, int co_n, int ci_n, int kh, int kw,
                                              int dgrad, int CI, int N, int npad, int RB, long long i,
                                              float* __restrict__ out) {
  const int taps = kh * kw;
  const int slabw = RB / 4;
  const int k = (int)(i % slabw);
  long long t = i / slabw;
  const int n = (int)(t % npad);
  t /= npad;
  const int u = (int)(t % taps);
  const int s = (int)(t / taps);
  const int ch = s * slabw + k;
  float v = 0.f;
  if (n < N && ch < CI) {
    int ky = u / kw, kx = u % kw;
    int co, ci;
    if (dgrad) { ky = kh - 1 - ky; kx = kw - 1 - kx; co = ch; ci = n; }
    else { co = n; ci = ch; }
    v = w[(((long long)co * ci_n + ci) * kh + ky) * kw + kx];
  }
  const float hi = tf32_rn(v), lo = tf32_rn(v - hi);
  const int kb = k * 4;
  int chunk = kb >> 4;
  chunk ^= RB == 128 ? (n & 7) : ((n >> 1) & 3);
  const long long row = ((long long)s * taps + u) * 2;  // plane 0 row block; plane 1 = +1
  const long long b0 = (row * npad + n) * RB + chunk * 16 + (kb & 15);
  const long long b1 = ((row + 1) * npad + n) * RB + chunk * 16 + (kb & 15);
  out[b0 / 4] = hi;
  out[b1 / 4] = lo;
}
__global__ void pack_window_f32_kernel(const float* __restrict__ w, int co_n, int ci_n, int kh, int kw, int dgrad,
                                       int CI, int N, int npad, int RB, int nslab, float* __restrict__ out) {
  griddep_launch();
  griddep_wait();
  const long long total = (long long)nslab * kh * kw * npad * (RB / 4);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x)
    pack_f32_elem(w, co_n, ci_n, kh, kw, dgrad, CI, N, npad, RB, i, out);
}
__global__ void pack_window_multi_f32_kernel(const bnff_pack_job* __restrict__ jobs) {
  griddep_launch();
  griddep_wait();
  const bnff_pack_job jb = jobs[blockIdx.y];
  const int d = blockIdx.z;
  void* out = d ? jb.wdgrad : jb.wfwd;
  if (!out) return;
  const int CI = d ? jb.c_out : jb.c_in, N = d ? jb.c_in : jb.c_out;
  const Geo gg = geo(CI, N, jb.kh, jb.kw, d, 4);
  const long long total = (long long)gg.nslab * jb.kh * jb.kw * gg.npad * (gg.RB / 4);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x)
    pack_f32_elem(jb.w, jb.c_out, jb.c_in, jb.kh, jb.kw, d, CI, N, gg.npad, gg.RB, i, (float*)out);
}

// one launch re-packing many convs (after each optimizer step): grid (x, job, fwd|dgrad)
__global__ void pack_window_multi_kernel(const bnff_pack_job* __restrict__ jobs) {
  griddep_launch();
  griddep_wait();
  const bnff_pack_job jb = jobs[blockIdx.y];
  const int d = blockIdx.z;
  void* out = d ? jb.wdgrad : jb.wfwd;
  if (!out) return;
  const int CI = d ? jb.c_out : jb.c_in, N = d ? jb.c_in : jb.c_out;
  const int taps = jb.kh * jb.kw;
  const Geo gg = geo(CI, N, jb.kh, jb.kw, d);  // the layout the conv kernels read
  const int RB = gg.RB, npad = gg.npad;
  const int slabw = RB / 2;
  const int nslab = (CI + slabw - 1) / slabw;
  // one thread per 16-byte chunk (8 consecutive reduction channels of one row n):
  // 32-bit index math, one vector store
  const int cpr = slabw / 8;
  const int total = nslab * taps * npad * cpr;
  __nv_bfloat16* o = (__nv_bfloat16*)out;
  const int tapsz = jb.kh * jb.kw;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int kc = i % cpr;
    int t = i / cpr;
    const int n = t % npad;
    t /= npad;
    const int u = t % taps;
    const int sl = t / taps;
    int ky = u / jb.kw, kx = u % jb.kw;
    if (d) { ky = jb.kh - 1 - ky; kx = jb.kw - 1 - kx; }
    const int tap = ky * jb.kw + kx;
    __align__(16) __nv_bfloat16 v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int ch = sl * slabw + kc * 8 + e;
      float f = 0.f;
      if (n < N && ch < CI) {
        const int co = d ? ch : n, ci = d ? n : ch;
        f = jb.w[(co * jb.c_in + ci) * tapsz + tap];
      }
      v[e] = __float2bfloat16_rn(f);
    }
    int chunk = kc;  // (k*2) >> 4 for the first k of the chunk
    chunk ^= RB == 128 ? (n & 7) : ((n >> 1) & 3);
    const long long byte = (((long long)sl * taps + u) * npad + n) * RB + chunk * 16;
    *reinterpret_cast<uint4*>(o + byte / 2) = *reinterpret_cast<const uint4*>(v);
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
int num_sms_wc() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
  }
  return n;
}

template <int BN, int RB, int TAPS, int MODE, bool SW = false, int ES = 2>
static int launch_t(WcParams p, cudaStream_t st) {
  auto kern = wconv_kernel<BN, RB, TAPS, MODE, SW, ES>;
  int stages = 8;
  Carve c{};
  const bool xop = MODE == M_DGRAD && p.pro == BNFF_PRO_BN_DX;
  bool gb = fold_tma<BN, RB, TAPS, MODE, SW, ES>(p);
  for (; stages >= 2; --stages) {
    c = carve<BN, RB, TAPS, MODE, SW, ES>(p.R, p.nslab, p.npad, stages, xop, gb, wtables<MODE>(p));
    if (c.total <= SMEM_BUDGET) break;
  }
  if (stages < 2) return kWindowNoFit;  // caller falls back to the generic kernel
  p.stages = stages;
  static int attr = 0;
  if (c.total > attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, c.total);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(wconv)");
    attr = c.total;
  }
  // a CTA's N tile must not change between its tiles (column sums stay in registers):
  // the grid is a multiple of the N-tile count
  int grid = p.tiles < num_sms_wc() ? p.tiles : num_sms_wc();
  if (grid > p.ntiles) grid -= grid % p.ntiles;
  launch(kern, dim3(grid), dim3(WC_THREADS), c.total, st, p);
  return check_launch("wconv");
}

inline bool wres1_enabled() {  // BNFF_WRES1=0: stream 1x1 fprop weights per stage (A/B timing)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BNFF_WRES1");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v != 0;
}
// fp32 (3xTF32) instantiations: 1x1 with 128-byte slabs, N tiles 32..128 (dgrad <= 64);
// 3x3 with 64-byte slabs and streamed weights, N tiles 32 / 64
template <int MODE, int TAPS>
static int dispatch_f32(const WcParams& p, int BN, int RB, cudaStream_t st, int sw = 1) {
  if (TAPS == 9) {
    if constexpr (MODE == M_DGRAD)
      if (!sw && BN == 32) return launch_t<32, 64, TAPS, MODE, false, 4>(p, st);  // resident weights
    if (BN == 32) return launch_t<32, 64, TAPS, MODE, true, 4>(p, st);
    return launch_t<64, 64, TAPS, MODE, true, 4>(p, st);
  }
  if (RB == 64) {
    if constexpr (MODE == M_DGRAD)
      if (BN == 64) return launch_t<64, 64, TAPS, MODE, false, 4>(p, st);
    return launch_t<32, 64, TAPS, MODE, false, 4>(p, st);
  }
  switch (BN) {
    case 32: return launch_t<32, 128, TAPS, MODE, false, 4>(p, st);
    case 64: return launch_t<64, 128, TAPS, MODE, false, 4>(p, st);
    default:
      if constexpr (MODE == M_FPROP) return launch_t<128, 128, TAPS, MODE, false, 4>(p, st);
      else return kWindowNoFit;
  }
}
template <int MODE, int TAPS>
static int dispatch(const WcParams& p, int BN, int RB, cudaStream_t st, int sw = 0) {
  if (TAPS == 9 && sw) return launch_t<64, 64, TAPS, MODE, true>(p, st);
  // 1x1 fprop with <= 64 KB of weights per N tile: weights resident, the freed half of every
  // stage goes to a deeper window ring (more bytes in flight per SM)
  if (TAPS == 1 && MODE == M_FPROP && RB == 128 && BN <= 128 && p.nslab * BN * RB <= 64 * 1024 &&
      wres1_enabled()) {
    if (BN == 128) return launch_t<128, 128, 1, MODE, true>(p, st);
    if (BN == 64) return launch_t<64, 128, 1, MODE, true>(p, st);
  }
  if (RB == 64) {
    switch (BN) {
      case 32: return launch_t<32, 64, TAPS, MODE>(p, st);
      case 64: return launch_t<64, 64, TAPS, MODE>(p, st);
      case 128: return launch_t<128, 64, TAPS, MODE>(p, st);
      default: return launch_t<256, 64, TAPS, MODE>(p, st);
    }
  }
  switch (BN) {
    case 32: return launch_t<32, 128, TAPS, MODE>(p, st);
    case 64: return launch_t<64, 128, TAPS, MODE>(p, st);
    case 128: return launch_t<128, 128, TAPS, MODE>(p, st);
    default: return launch_t<256, 128, TAPS, MODE>(p, st);
  }
}

}  // namespace wc
}  // namespace bnff

using namespace bnff;

namespace bnff {
namespace wc {
template <int MODE, int TAPS>
static bool fits2_f32(int BN, int RB, int R, int nslab, int npad, bool xop, int tf = 3, int sw = 1) {
  Carve c{};
  if (TAPS == 9 && !sw && BN == 32 && MODE == M_DGRAD) c = carve<32, 64, TAPS, MODE, false, 4>(R, nslab, npad, 2, xop, false, tf);
  else if (TAPS == 9) c = BN == 32 ? carve<32, 64, TAPS, MODE, true, 4>(R, nslab, npad, 2, xop, false, tf)
                              : carve<64, 64, TAPS, MODE, true, 4>(R, nslab, npad, 2, xop, false, tf);
  else if (RB == 64 && MODE == M_DGRAD && BN == 64) c = carve<64, 64, TAPS, MODE, false, 4>(R, nslab, npad, 2, xop, true, tf);
  else if (RB == 64) c = carve<32, 64, TAPS, MODE, false, 4>(R, nslab, npad, 2, xop, false, tf);
  else if (BN == 32) c = carve<32, 128, TAPS, MODE, false, 4>(R, nslab, npad, 2, xop, false, tf);
  else if (BN == 64) c = carve<64, 128, TAPS, MODE, false, 4>(R, nslab, npad, 2, xop, false, tf);
  else if (MODE == M_FPROP) c = carve<128, 128, TAPS, MODE, false, 4>(R, nslab, npad, 2, xop, false, tf);
  else return false;
  return c.total <= SMEM_BUDGET;
}
template <int MODE, int TAPS>
static bool fits2(int BN, int RB, int R, int nslab, int npad, bool xop, int sw = 0, int tf = 3) {
  Carve c{};
#define BNFF_FIT(bn, rb) c = carve<bn, rb, TAPS, MODE>(R, nslab, npad, 2, xop, false, tf)
  if (TAPS == 9 && sw) {
    c = carve<64, 64, TAPS, MODE, true>(R, nslab, npad, 2, xop, false, tf);
    return c.total <= SMEM_BUDGET;
  }
  if (RB == 64) {
    if (BN == 32) BNFF_FIT(32, 64); else if (BN == 64) BNFF_FIT(64, 64);
    else if (BN == 128) BNFF_FIT(128, 64); else BNFF_FIT(256, 64);
  } else {
    if (BN == 32) BNFF_FIT(32, 128); else if (BN == 64) BNFF_FIT(64, 128);
    else if (BN == 128) BNFF_FIT(128, 128); else BNFF_FIT(256, 128);
  }
#undef BNFF_FIT
  return c.total <= SMEM_BUDGET;
}
}  // namespace wc
}  // namespace bnff

// eligibility of the window kernels for a conv (bf16, stride 1, 1x1/p0 or 3x3/p1), for all
// three passes: the shared-memory plan must fit with >= 2 stages in the worst case
extern "C" int bnff_window_ok_ex(int32_t dtype, int32_t c_in, int32_t c_out, int32_t kh, int32_t kw,
                                 int32_t stride, int32_t pad, int32_t h, int32_t w, int32_t tables) {
  if ((dtype != BNFF_BF16 && dtype != BNFF_F32) || stride != 1) return 0;
  const int es = dtype == BNFF_F32 ? 4 : 2;
  if (!((kh == 1 && kw == 1 && pad == 0) || (kh == 3 && kw == 3 && pad == 1))) return 0;
  if (c_in % 16 || c_out % 16) return 0;
  if (kh == 3) {
    const int wp = w + 2;
    if (128 + 2 * wp + 2 > wc::RMAX) return 0;
  }
  (void)h;
  const int R = 128 + (kh == 3 ? 2 * (w + 2) + 2 : 0);
  for (int d = 0; d < 2; ++d) {
    const int CI = d ? c_out : c_in, N = d ? c_in : c_out;
    const int tf = d ? ((tables & BNFF_WT_DGRAD_PRO) ? 1 : 0) | ((tables & BNFF_WT_DGRAD_NRC) ? 2 : 0)
                     : ((tables & BNFF_WT_FPROP_PRO) ? 1 : 0);
    const wc::Geo g = wc::geo(CI, N, kh, kw, d, es);
    if (es == 4) {
      const bool ok4 = kh == 3 ? (d ? wc::fits2_f32<wc::M_DGRAD, 9>(g.BN, g.RB, R, g.nslab, g.npad, true, tf, g.sw)
                                    : wc::fits2_f32<wc::M_FPROP, 9>(g.BN, g.RB, R, g.nslab, g.npad, false, tf))
                               : (d ? wc::fits2_f32<wc::M_DGRAD, 1>(g.BN, g.RB, R, g.nslab, g.npad, true, tf)
                                    : wc::fits2_f32<wc::M_FPROP, 1>(g.BN, g.RB, R, g.nslab, g.npad, false, tf));
      if (!ok4) return 0;
      continue;
    }
    const bool ok = kh == 3 ? (d ? wc::fits2<wc::M_DGRAD, 9>(g.BN, g.RB, R, g.nslab, g.npad, true, g.sw, tf)
                                 : wc::fits2<wc::M_FPROP, 9>(g.BN, g.RB, R, g.nslab, g.npad, false, g.sw, tf))
                            : (d ? wc::fits2<wc::M_DGRAD, 1>(g.BN, g.RB, R, g.nslab, g.npad, true, 0, tf)
                                 : wc::fits2<wc::M_FPROP, 1>(g.BN, g.RB, R, g.nslab, g.npad, false, 0, tf));
    if (!ok) return 0;
  }
  return 1;
}

extern "C" int bnff_window_ok(int32_t dtype, int32_t c_in, int32_t c_out, int32_t kh, int32_t kw,
                              int32_t stride, int32_t pad, int32_t h, int32_t w) {
  return bnff_window_ok_ex(dtype, c_in, c_out, kh, kw, stride, pad, h, w,
                           BNFF_WT_FPROP_PRO | BNFF_WT_DGRAD_PRO | BNFF_WT_DGRAD_NRC);
}

extern "C" int64_t bnff_window_pack_size(int32_t dtype, int32_t c_out, int32_t c_in, int32_t kh,
                                         int32_t kw, int32_t dgrad) {
  if (dtype != BNFF_BF16 && dtype != BNFF_F32) return 0;
  const int es = dtype == BNFF_F32 ? 4 : 2;
  const int CI = dgrad ? c_out : c_in, N = dgrad ? c_in : c_out;
  const wc::Geo g = wc::geo(CI, N, kh, kw, dgrad, es);
  // elements: [slab][tap][plane][npad][RB bytes]; fp32 has hi and lo planes
  return (int64_t)g.nslab * g.taps * g.npad * (g.RB / es) * (es == 4 ? 2 : 1);
}

extern "C" int bnff_pack_window(int32_t dtype, const float* w, int32_t c_out, int32_t c_in, int32_t kh,
                                int32_t kw, void* fwd, void* dgr, void* stream) {
  if (dtype == BNFF_F32) {
    for (int d = 0; d < 2; ++d) {
      void* out = d ? dgr : fwd;
      if (!out) continue;
      const int CI = d ? c_out : c_in, N = d ? c_in : c_out;
      const wc::Geo g = wc::geo(CI, N, kh, kw, d, 4);
      const long long total = (long long)g.nslab * g.taps * g.npad * (g.RB / 4);
      int blocks = (int)((total + 255) / 256);
      if (blocks > 148 * 8) blocks = 148 * 8;
      launch(wc::pack_window_f32_kernel, dim3(blocks), dim3(256), 0, (cudaStream_t)stream, w, c_out, c_in, kh,
             kw, d, CI, N, g.npad, g.RB, g.nslab, (float*)out);
      int rc = check_launch("pack_window f32");
      if (rc) return rc;
    }
    return BNFF_OK;
  }
  if (dtype != BNFF_BF16) return set_error(BNFF_ERR_UNSUPPORTED, "pack_window: bf16 / f32");
  for (int d = 0; d < 2; ++d) {
    void* out = d ? dgr : fwd;
    if (!out) continue;
    const int CI = d ? c_out : c_in, N = d ? c_in : c_out;
    const wc::Geo g = wc::geo(CI, N, kh, kw, d);
    const long long total = (long long)g.nslab * g.taps * g.npad * (g.RB / 2);
    int blocks = (int)((total + 255) / 256);
    if (blocks > 148 * 8) blocks = 148 * 8;
    launch(wc::pack_window_kernel, dim3(blocks), dim3(256), 0, (cudaStream_t)stream, 
        w, c_out, c_in, kh, kw, d, CI, N, g.npad, g.RB, g.nslab, (__nv_bfloat16*)out);
    int rc = check_launch("pack_window");
    if (rc) return rc;
  }
  return BNFF_OK;
}

static unsigned long long* g_wc_trace = nullptr;
extern "C" int bnff_debug_trace(void* buf) {
  g_wc_trace = (unsigned long long*)buf;
  return BNFF_OK;
}

// internal entry used by bnff_conv_fprop / bnff_conv_dgrad when bnff_window_ok()
extern "C" int bnff_window_conv(int32_t dtype, int32_t mode, int32_t kh, int32_t pad, bnff_view in, bnff_view in_x,
                                int32_t pro, bnff_coef pcoef, bnff_view out, const void* wwin,
                                const float* bias, int32_t epi, bnff_view ex, bnff_coef ecoef,
                                double* stat_part, void* stream) {
  wc::WcParams p{};
  p.n = (int)in.n; p.h = (int)in.h; p.w = (int)in.w;
  p.pad = pad;
  p.hp = p.h + 2 * pad; p.wp = p.w + 2 * pad;
  const long long Q = (long long)p.n * p.hp * p.wp;
  if (Q >= (1ll << 31)) return set_error(BNFF_ERR_UNSUPPORTED, "wconv: grid too large");
  p.Q = (int)Q;
  p.P = (int)(in.n * in.h * in.w);
  p.fd_hpwp = make_fastdiv(p.hp * p.wp);
  p.fd_wp = make_fastdiv(p.wp);
  p.ci = (int)in.c;
  p.N = (int)out.c;
  const int es = dtype == BNFF_F32 ? 4 : 2;
  wc::Geo g = wc::geo(p.ci, p.N, kh, kh, mode, es);
  if (es == 4 && mode == 1 && epi >= BNFF_DG_NRC_ACC && g.BN < 64)  // fp32 fold: TMA G tile (32 columns)
    return set_error(BNFF_ERR_UNSUPPORTED, "wconv: the fp32 block-gradient fold needs >= 33 channels");
  p.nslab = g.nslab;
  p.npad = g.npad;
  p.ntiles = g.ntiles;
  const int slabw = g.RB / es;
  uint32_t box[4];
  int rank;
  if (kh == 3) {
    const int hpwp = p.hp * p.wp;
    if (hpwp <= 128) {  // whole images per tile
      p.tmode = 2;
      p.kt = 128 / hpwp;
      p.BR = p.hp;
      p.BI = p.kt;
      p.WPI = hpwp;
      p.mtiles = (p.n + p.kt - 1) / p.kt;
    } else {            // kt output rows of one image per tile
      p.tmode = 1;
      p.kt = 128 / p.wp;
      if (p.kt > p.h) p.kt = p.h;
      p.BR = p.kt + 2;
      p.BI = 1;
      p.WPI = p.BR * p.wp;
      p.tpi = (p.h + p.kt - 1) / p.kt;
      p.mtiles = p.n * p.tpi;
    }
    p.Rld = p.BR * p.BI * p.wp;
    const int rmma = 128 + 2 * p.wp + 2;  // rows the (discarded) last MMA rows may touch
    p.R = wc::align_up(p.Rld > rmma ? p.Rld : rmma, 8);
    if (p.R > wc::RMAX) return wc::kWindowNoFit;
    rank = 4;
    box[0] = slabw; box[1] = p.wp; box[2] = p.BR; box[3] = p.BI;
  } else {
    p.tmode = 0;
    p.Rld = 128;
    p.R = 128;
    p.mtiles = (p.P + 127) / 128;
    rank = 2;
    box[0] = slabw; box[1] = 128;
    // small-M 1x1 fprop (DenseNet's 14^2 / 7^2 blocks: 98 / 25 pixel tiles at b64): halve the
    // N tile while the launch has fewer tiles than BNFF_SMALLM (default 0 = off) so more SMs
    // share it (each N tile re-reads the A tile, from L2).  N stays a multiple of the tile,
    // so npad -- the packed weight layout -- does not change
    if (mode == 0) {
      const int tgt = wc::smallm_tiles();
      while (tgt > 0 && g.BN > 32 && p.N % g.BN == 0 && p.mtiles * g.ntiles < tgt) {
        g.BN /= 2;
        g.ntiles *= 2;
      }
      p.ntiles = g.ntiles;
    }
  }
  p.tiles = p.mtiles * p.ntiles;
  // TMA epilogue for 128-byte staged chunks (bf16: 64 columns, BN >= 128; fp32: 32 columns,
  // BN >= 64): the output (and dgrad x mask) descriptors are required; if they cannot be
  // encoded the window kernel declines (generic implicit GEMM)
  p.tstore = 0;
  const int cw128 = 128 / es;  // columns of a 128-byte staged row
  if (es == 4 ? g.BN >= 64 : g.BN >= 128) {
    uint32_t ob[4];
    if (kh == 3) {
      ob[0] = cw128; ob[1] = p.wp; ob[2] = p.tmode == 2 ? p.hp : p.kt; ob[3] = p.tmode == 2 ? p.kt : 1;
    } else {
      ob[0] = cw128; ob[1] = 128;
    }
    p.tstore = encode_nhwc(&p.tma_out, es, out.ptr, out.n, out.h, out.w, out.c, out.row_stride, rank, ob) ? 1 : 0;
    if (p.tstore && mode == 1 && epi != BNFF_DG_PLAIN &&
        !encode_nhwc(&p.tma_ex, es, ex.ptr, ex.n, ex.h, ex.w, ex.c, ex.row_stride, rank, ob))
      p.tstore = 0;
    if (!p.tstore) return wc::kWindowNoFit;
  }
  if (!encode_nhwc(&p.tma_a, es, in.ptr, in.n, in.h, in.w, in.c, in.row_stride, rank, box))
    return set_error(BNFF_ERR_CUDA, "wconv: cuTensorMapEncodeTiled failed (window operand)");
  if (mode == 1 && pro == BNFF_PRO_BN_DX &&
      !encode_nhwc(&p.tma_x, es, in_x.ptr, in_x.n, in_x.h, in_x.w, in_x.c, in_x.row_stride, rank, box))
    return set_error(BNFF_ERR_CUDA, "wconv: cuTensorMapEncodeTiled failed (x operand)");
  p.pro = pro;
  p.pcoef = pcoef;
  p.wpk = (const uint8_t*)wwin;
  p.out = out.ptr; p.out_rs = out.row_stride;
  p.bias = bias;
  p.epi = epi;
  p.ex = ex.ptr; p.ex_rs = ex.row_stride;
  p.ecoef = ecoef;
  p.stat_part = stat_part;
  p.trace = g_wc_trace;
  if (kh == 3 && !g.sw && g.ntiles != 1 && es == 2) return set_error(BNFF_ERR_UNSUPPORTED, "wconv: 3x3 needs one N tile");
  if (kh == 3 && mode == 1 && epi >= BNFF_DG_NRC_ACC)
    return set_error(BNFF_ERR_UNSUPPORTED, "wconv: the block-gradient fold is a 1x1 dgrad epilogue");
  cudaStream_t st = (cudaStream_t)stream;
  if (es == 4) {
    if (mode == 0)
      return kh == 3 ? wc::dispatch_f32<wc::M_FPROP, 9>(p, g.BN, g.RB, st) : wc::dispatch_f32<wc::M_FPROP, 1>(p, g.BN, g.RB, st);
    return kh == 3 ? wc::dispatch_f32<wc::M_DGRAD, 9>(p, g.BN, g.RB, st, g.sw)
                   : wc::dispatch_f32<wc::M_DGRAD, 1>(p, g.BN, g.RB, st);
  }
  if (mode == 0) {
    return kh == 3 ? wc::dispatch<wc::M_FPROP, 9>(p, g.BN, g.RB, st, g.sw)
                   : wc::dispatch<wc::M_FPROP, 1>(p, g.BN, g.RB, st);
  }
  return kh == 3 ? wc::dispatch<wc::M_DGRAD, 9>(p, g.BN, g.RB, st, g.sw)
                 : wc::dispatch<wc::M_DGRAD, 1>(p, g.BN, g.RB, st);
}

// ---------------------------------------------------------------------------
// window wgrad host side
// ---------------------------------------------------------------------------
namespace bnff {
namespace wc {
// minimum k-blocks per wgrad split (BNFF_WG_MINKPT overrides, A/B).  Default 1: longer splits
// write fewer partial bytes but lengthen the 14^2/7^2 weight gradients, and the step measured
// slower at 4 (+0.5% fp32, +2.3% bf16) and 8 (+2%, +10%)
inline int wg_min_kpt() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BNFF_WG_MINKPT");
    v = e ? atoi(e) : 1;
    if (v < 1) v = 1;
  }
  return v;
}
struct WgPlan {
  int ok, taps, BN, MT, KB, NT, MG, RA, nkb, kpt, splits, hp, wp, Q;
  int tmode, kt, BR, BI, WPI, tpi, Rld, Kr, P;
};
// k-blocks are the forward kernel's tiles (3x3: kt padded output rows of one image, or
// kt whole images; 1x1: KB pixels); splits spread them over the SMs
static WgPlan wg_plan(int n, int h, int w, int cin, int cout, int kh, int pad) {
  WgPlan q{};
  q.taps = kh * kh;
  q.hp = h + 2 * pad;
  q.wp = w + 2 * pad;
  const long long Q = (long long)n * q.hp * q.wp;
  if (Q >= (1ll << 30)) return q;
  q.Q = (int)Q;
  q.P = n * h * w;
  if (q.taps == 9) {
    q.BN = 32; q.MT = 1; q.KB = 128;
    const int hpwp = q.hp * q.wp;
    if (hpwp <= 128) {
      q.tmode = 2;
      q.kt = 128 / hpwp;
      q.BR = q.hp; q.BI = q.kt; q.WPI = hpwp;
      q.nkb = (n + q.kt - 1) / q.kt;
      q.Kr = q.kt * hpwp;
    } else {
      q.tmode = 1;
      q.kt = 128 / q.wp;
      if (q.kt > h) q.kt = h;
      if (q.kt < 1) return q;
      q.BR = q.kt + 2; q.BI = 1; q.WPI = q.BR * q.wp;
      q.tpi = (h + q.kt - 1) / q.kt;
      q.nkb = n * q.tpi;
      q.Kr = q.kt * q.wp;
    }
    q.Rld = q.BR * q.BI * q.wp;
    const int rmma = 128 + 2 * q.wp + 2;
    q.RA = align_up(q.Rld > rmma ? q.Rld : rmma, 8);
    if (q.RA > RMAX) return q;  // window taller than the allocation: generic kernel
  } else {
    q.BN = pick_bn(cout);
    q.MT = ((q.BN == 64 || q.BN == 128) && cin > 128) ? 2 : 1;  // the instantiated MT=2 variants
    q.KB = 64;
    q.RA = q.Rld = q.Kr = q.KB;
    q.nkb = (q.P + q.KB - 1) / q.KB;
  }
  q.NT = (cout + q.BN - 1) / q.BN;
  q.MG = (cin + q.MT * 128 - 1) / (q.MT * 128);
  const int target = num_sms_wc();
  int splits = (target + q.MG * q.NT - 1) / (q.MG * q.NT);
  // every split writes a TAPS x 128 x BN fp32 partial tile: keep >= min_kpt k-blocks per split so
  // the partials stay below the operand bytes they summarise (small maps: fewer, longer splits)
  const int maxs = q.nkb / wg_min_kpt() > 0 ? q.nkb / wg_min_kpt() : 1;
  if (splits > maxs) splits = maxs;
  if (splits < 1) splits = 1;
  q.kpt = (q.nkb + splits - 1) / splits;
  q.splits = (q.nkb + q.kpt - 1) / q.kpt;
  q.ok = 1;
  return q;
}
}  // namespace wc
}  // namespace bnff

extern "C" int64_t bnff_window_wgrad_ws(int32_t n, int32_t h, int32_t w, int32_t kh, int32_t c_in,
                                        int32_t c_out) {
  const int pad = kh / 2;
  const wc::WgPlan q = wc::wg_plan(n, h, w, c_in, c_out, kh, pad);
  if (!q.ok) return 0;
  return (int64_t)q.splits * q.taps * c_in * c_out + (int64_t)q.splits * c_out;
}

// dW (and partials) of a window-eligible conv; dbias is left to the caller
extern "C" int bnff_window_wgrad(bnff_view x, int32_t x_pro, bnff_coef x_coef, bnff_view dy, bnff_view dy_x,
                                 int32_t dy_pro, bnff_coef dy_coef, int32_t kh, float* ws, float* dw,
                                 int32_t dw_cin, float* dbias, void* stream) {
  const int pad = kh / 2;
  const wc::WgPlan q = wc::wg_plan((int)x.n, (int)x.h, (int)x.w, (int)x.c, (int)dy.c, kh, pad);
  if (!q.ok) return wc::kWindowNoFit;  // caller uses the generic kernel
  wc::WgParams p{};
  p.n = (int)x.n; p.h = (int)x.h; p.w = (int)x.w; p.hp = q.hp; p.wp = q.wp; p.pad = pad; p.Q = q.Q;
  p.tmode = q.tmode; p.kt = q.kt; p.BR = q.BR; p.BI = q.BI; p.WPI = q.WPI; p.tpi = q.tpi;
  p.Rld = q.Rld; p.Kr = q.Kr; p.P = q.P;
  p.fd_hpwp = make_fastdiv(q.hp * q.wp);
  p.fd_wp = make_fastdiv(q.wp);
  p.cin = (int)x.c; p.cout = (int)dy.c;
  p.KB = q.KB; p.RA = q.RA; p.nkb = q.nkb; p.kpt = q.kpt; p.splits = q.splits;
  p.MG = q.MG; p.NT = q.NT; p.units = q.MG * q.NT * q.splits;
  p.x_pro = x_pro; p.x_coef = x_coef;
  p.dy_pro = dy_pro; p.dy_coef = dy_coef;
  p.ws = ws;
  p.wsb = dbias ? ws + (long long)q.splits * q.taps * p.cin * p.cout : nullptr;
  // TMA boxes: x window {64, wp, BR, BI} / {64, KB}; dy (and dy_x) {brb/2, wp, rows, imgs} / {brb/2, KB}
  const uint32_t bch = (q.BN * 2 >= 128 ? 128 : q.BN * 2) / 2;
  uint32_t bx[4], bd[4];
  int rank;
  if (q.taps == 9) {
    rank = 4;
    bx[0] = 64; bx[1] = q.wp; bx[2] = q.BR; bx[3] = q.BI;
    bd[0] = bch; bd[1] = q.wp; bd[2] = q.tmode == 2 ? q.hp : q.kt; bd[3] = q.tmode == 2 ? q.kt : 1;
  } else {
    rank = 2;
    bx[0] = 64; bx[1] = q.KB;
    bd[0] = bch; bd[1] = q.KB;
  }
  if (!encode_nhwc_bf16(&p.tma_x, x.ptr, x.n, x.h, x.w, x.c, x.row_stride, rank, bx) ||
      !encode_nhwc_bf16(&p.tma_dy, dy.ptr, dy.n, dy.h, dy.w, dy.c, dy.row_stride, rank, bd) ||
      (dy_pro == BNFF_PRO_BN_DX &&
       !encode_nhwc_bf16(&p.tma_dyx, dy_x.ptr, dy_x.n, dy_x.h, dy_x.w, dy_x.c, dy_x.row_stride, rank, bd)))
    return set_error(BNFF_ERR_CUDA, "wgrad window: cuTensorMapEncodeTiled failed");
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  if (q.taps == 9) rc = wc::launch_wg<32, 1, 9, 128>(p, st);
  else if (q.BN == 32) rc = wc::launch_wg<32, 1, 1, 64>(p, st);
  else if (q.BN == 64) rc = q.MT == 2 ? wc::launch_wg<64, 2, 1, 64>(p, st) : wc::launch_wg<64, 1, 1, 64>(p, st);
  else if (q.BN == 128) rc = q.MT == 2 ? wc::launch_wg<128, 2, 1, 64>(p, st) : wc::launch_wg<128, 1, 1, 64>(p, st);
  else rc = wc::launch_wg<256, 1, 1, 64>(p, st);
  if (rc) return rc;
  const int M4 = q.taps * p.cin * (p.cout / 4);
  int blocks = (M4 + 31) / 32;
  if (blocks > 148 * 8) blocks = 148 * 8;
  launch(wc::wg_reduce_kernel, dim3(blocks), dim3(256), 0, st, ws, q.splits, q.taps, p.cin, p.cout,
                                               dw_cin > 0 ? dw_cin : p.cin, dw, p.wsb, dbias);
  return check_launch("wgrad window reduce");
}

// fixed-order split reduction of [splits][taps][cin][cout] partials into dW (co, ci, kh, kw) and
// of [splits][cout] into dbias (shared by the bf16 window wgrad and wgrad32.cu)
extern "C" int bnff_wgrad_reduce(const float* ws, int32_t splits, int32_t taps, int32_t cin, int32_t cout,
                                 int32_t cin_real, float* dw, const float* wsb, float* dbias, void* stream) {
  const int M4 = taps * cin * (cout / 4);
  int blocks = (M4 + 31) / 32;
  if (blocks > 148 * 8) blocks = 148 * 8;
  launch(wc::wg_reduce_kernel, dim3(blocks), dim3(256), 0, (cudaStream_t)stream, ws, splits, taps, cin, cout,
         cin_real > 0 ? cin_real : cin, dw, wsb, dbias);
  return check_launch("wgrad reduce");
}

extern "C" int bnff_pack_window_multi(int32_t dtype, int32_t njobs, const bnff_pack_job* jobs_dev,
                                      int64_t max_elems, void* stream) {
  if (dtype != BNFF_BF16 && dtype != BNFF_F32) return set_error(BNFF_ERR_UNSUPPORTED, "pack_window_multi: dtype");
  if (njobs <= 0) return BNFF_OK;
  if (dtype == BNFF_F32) {
    long long bx = (max_elems / 2 + 255) / 256;  // one thread per (hi, lo) element pair
    if (bx > 64) bx = 64;
    if (bx < 1) bx = 1;
    launch(wc::pack_window_multi_f32_kernel, dim3((unsigned)bx, (unsigned)njobs, 2), dim3(256), 0,
           (cudaStream_t)stream, jobs_dev);
    return check_launch("pack_window_multi f32");
  }
  long long bx = (max_elems / 8 + 255) / 256;  // one thread per 16-byte chunk
  if (bx > 32) bx = 32;
  if (bx < 1) bx = 1;
  dim3 grid((unsigned)bx, (unsigned)njobs, 2);
  launch(wc::pack_window_multi_kernel, dim3(grid), dim3(256), 0, (cudaStream_t)stream, jobs_dev);
  return check_launch("pack_window_multi");
}
