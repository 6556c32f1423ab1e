// wgrad32.cu -- fp32 (3xTF32) weight gradients on tcgen05 / TMEM with TMA tap boxes (sm_100a).
//
// dW[tap][ci][co] = sum_m  pro(x)[m + s_tap, ci] * pro(dy)[m, co]      (conv2d_bwd dw, ops.py:178-204)
//
// The bf16 window wgrad (wconv.cu) loads one zero-haloed window per k-block and reads all 9
// taps through row-shifted descriptors; in fp32 every operand element takes 8 bytes of shared
// memory (TF32 hi + lo planes), and a 128-channel window of ~240 rows would not fit.  Here a
// stage is one (k-block, tap) pair instead: the producer warp loads the tap's SHIFTED input box
// straight from the NHWC tensor ({32 channels, bw, kt, 1} per 32-channel atom, the map borders
// zero-filled by the TMA engine) and the dy box of the k-block; the transform warps apply the
// operand prologues (x: ReLU / BN+ReLU -- padding positions forced back to zero, padding applies
// after normalize; dy: the deferred BN dx), split both operands into TF32 hi/lo planes, and the
// MMA warp issues hi*hi + hi*lo + lo*hi (MN-major A and B) into the tap's TMEM accumulator.
// A k-block is kt whole output rows of bw pixels (bw*kt = 56 for the 7..56 maps; 112-wide maps
// take half rows), the same for 1x1 (one tap, shift 0) and 3x3.  Work units are (128 input
// channels, N tile, K split) spread over the SMs; the fp32 partials [split][tap][ci][co] are
// reduced in fixed split order by wconv.cu's wg_reduce_kernel (deterministic).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "sm100.cuh"
#include "common.cuh"

namespace bnff {
namespace wg32 {

constexpr int NTW = 8;                       // transform warps
constexpr int LT = NTW * 32;
constexpr int THREADS = (NTW + 1 + 4 + 1) * 32;  // + MMA warp, 4 epilogue warps, TMA producer
constexpr int PRODUCER = NTW + 1 + 4;
constexpr int SMEM_BUDGET = 225 * 1024;
constexpr int MAXST = 6;

struct P {
  CUtensorMap tma_x, tma_dy, tma_dyx;
  int n, h, w, cin, cout, kh, pad;
  int bw, kt, xb, tpi, KBr, nkb, kpt, splits, MG, NT, units, stages;
  int RS, rows;  // box row stride (3x3: bw + 2, the two trailing columns are junk) and box rows
  int x_pro;
  bnff_coef x_coef;
  int dy_pro;
  bnff_coef dy_coef;
  float* ws;   // [splits][taps][cin][cout]
  float* wsb;  // nullable: dbias partials [splits][cout]
};

__host__ __device__ inline int a_bytes(int KBr) { return 4 * KBr * 128; }            // 128 channels
template <int BN> __host__ __device__ inline int b_bytes(int KBr) { return (BN / 32) * KBr * 128; }
template <int BN>
__host__ __device__ inline int stage_bytes(int KBr, bool xop) {
  // A hi | A lo | B hi | B lo | x (BN_DX).  Landing x in the B lo plane (read before it is
  // rewritten) gives three 64 KB stages instead of two 80 KB ones, but measured 5% slower in
  // the step (the weight gradients share HBM with the dgrad chain), so x keeps its own plane
  const int s = 2 * a_bytes(KBr) + 2 * b_bytes<BN>(KBr) + (xop ? b_bytes<BN>(KBr) : 0);
  return (s + 1023) / 1024 * 1024;
}
template <int BN>
__host__ __device__ inline int smem_total(int KBr, bool xop, int stages, int cin_pad, int npad) {
  return stages * stage_bytes<BN>(KBr, xop) + 2 * cin_pad * 4 + 3 * npad * 4 + 4 * LT * 4 + 1024;
}

__device__ __forceinline__ void split4(const float* f, float4& hi, float4& lo) {
  hi.x = tf32_rn(f[0]); hi.y = tf32_rn(f[1]); hi.z = tf32_rn(f[2]); hi.w = tf32_rn(f[3]);
  lo.x = f[0] - hi.x; lo.y = f[1] - hi.y; lo.z = f[2] - hi.z; lo.w = f[3] - hi.w;
}

template <int BN, int TAPS>
__global__ void __launch_bounds__(THREADS, 1) wgrad_f32_kernel(const __grid_constant__ P p) {
  griddep_launch();
  constexpr int NBA = BN / 32;  // B (dy) atoms of 32 fp32 channels
  constexpr int SPK = TAPS == 9 ? 3 : 1;  // stages per k-block (vertical taps)
  constexpr int TPS = TAPS == 9 ? 3 : 1;  // taps per stage (horizontal taps)
  extern __shared__ uint8_t dsm_raw[];
  uint8_t* smem = dsm_raw + ((1024u - (smem_u32(dsm_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full_bar[MAXST], empty_bar[MAXST], ld_bar[MAXST], accf_bar, acce_bar;
  __shared__ uint32_t tmem_sh;
  const bool xb = p.dy_pro == BNFF_PRO_BN_DX;
  const int ST = p.stages;
  const int SB = stage_bytes<BN>(p.KBr, xb);
  const int AB = a_bytes(p.KBr), BB = b_bytes<BN>(p.KBr);
  const int cin_pad = p.MG * 128, npad = p.NT * BN;
  float* ptab = reinterpret_cast<float*>(smem + ST * SB);
  float* qtab = ptab + 2 * cin_pad;
  float* bred = qtab + 3 * npad;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nun = (p.units - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  // 1x1: stacked B (A_hi x [B_hi | B_lo] in one N = 2*BN MMA, A_lo x B_hi into the cross-term
  // half, summed by the epilogue); 3x3 keeps three MMAs (9 taps x 64 columns would not fit TMEM)
  constexpr bool STK = BNFF_TF32_STACK && TAPS == 1;
  constexpr int AC = STK ? 2 * BN : BN;  // TMEM columns per tap accumulator
  constexpr int TCOLS = TAPS * AC <= 32 ? 32 : (TAPS * AC <= 64 ? 64 : (TAPS * AC <= 128 ? 128 : (TAPS * AC <= 256 ? 256 : 512)));

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
  if (warp == NTW) tmem_alloc<TCOLS>(&tmem_sh);
  // rows past a box (KBr > bw*kt) must be finite zeros for the full-K MMAs
  for (int i = tid; i < ST * SB / 16; i += THREADS) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  __syncthreads();
  griddep_wait();
  constexpr int GS = THREADS - 32;
  if (warp != PRODUCER) {
    for (int c = tid; c < cin_pad; c += GS) {  // x prologue: (scale, beta - mean*scale)
      float t0 = 1.f, t1 = 0.f;
      if (c < p.cin && p.x_pro == BNFF_PRO_BN_RELU) {
        t0 = p.x_coef.b[c];
        t1 = p.x_coef.c[c] - p.x_coef.a[c] * t0;
      }
      ptab[c] = t0;
      ptab[cin_pad + c] = t1;
    }
    for (int c = tid; c < npad; c += GS) {  // dy prologue (BN_DX): g, -g*k2*inv, g*(k2*inv*mean - k1)
      float t0 = 1.f, t1 = 0.f, t2 = 0.f;
      if (c < p.cout && xb) {
        const float m = p.dy_coef.a[c], inv = p.dy_coef.b[c], k1 = p.dy_coef.c[c], k2 = p.dy_coef.d[c],
                    g = p.dy_coef.e[c];
        t0 = g;
        t1 = -g * k2 * inv;
        t2 = g * (k2 * inv * m - k1);
      }
      qtab[c] = t0;
      qtab[npad + c] = t1;
      qtab[2 * npad + c] = t2;
    }
    tc_fence_before();
    asm volatile("bar.sync 6, %0;" ::"n"(GS) : "memory");
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
  auto kb_count = [&](int sp) { return min(p.kpt, p.nkb - sp * p.kpt); };
  // k-block -> (image, first output row, first output column)
  auto kb_org = [&](int kb, int& img, int& y0, int& x0) {
    const int xbk = kb % p.xb;
    const int t = kb / p.xb;
    img = t / p.tpi;
    y0 = (t - img * p.tpi) * p.kt;
    x0 = xbk * p.bw;
  };
  // the k-blocks of a split are consecutive: step (image, row block, column block) without
  // the two integer divisions per k-block
  auto kb_next = [&](int& img, int& y0, int& x0) {
    x0 += p.bw;
    if (x0 >= p.xb * p.bw) {
      x0 = 0;
      y0 += p.kt;
      if (y0 >= p.tpi * p.kt) {
        y0 = 0;
        ++img;
      }
    }
  };
  auto stage = [&](int s) { return smem + s * SB; };

  if (warp < NTW) {
    // =============================== transform warps ===============================
    const bool need_db = p.wsb != nullptr;
    float bacc[NBA][4];
#pragma unroll
    for (int b = 0; b < NBA; ++b)
#pragma unroll
      for (int i = 0; i < 4; ++i) bacc[b][i] = 0.f;
    const int j = tid & 7;          // 16-byte chunk of a 128-byte row
    const int r0 = tid >> 3;        // rows r0, r0 + 32 (KBr <= 64)
    // (box row, box column) of this thread's rows; rows past the box stay zero
    int gly[2], glx[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int r = r0 + 32 * q;
      gly[q] = r < p.rows ? r / p.RS : 1 << 20;
      glx[q] = r < p.rows ? r - gly[q] * p.RS : 0;
    }
    int st = 0;
    uint32_t ph = 0;
    for (int ui = 0; ui < nun; ++ui) {
      int mg, nt, sp;
      unit_of(ui, mg, nt, sp);
      const int cnt = kb_count(sp);
      int img, y0, x0;
      kb_org(sp * p.kpt, img, y0, x0);
      for (int k = 0; k < cnt; ++k, kb_next(img, y0, x0)) {
        for (int u = 0; u < SPK; ++u) {  // one stage per vertical tap (3x3) -- the 3 horizontal
          const int ty = TAPS == 9 ? u - 1 : 0;  // taps read it through K-row-shifted descriptors
          mbar_wait(&ld_bar[st], ph);
          uint8_t* A = stage(st);
          uint8_t* AL = A + AB;
          uint8_t* B = A + 2 * AB;
          uint8_t* BL = B + BB;
          const uint8_t* X = B + 2 * BB;
          // A: x at the tap-shifted positions, 4 atoms of 32 channels
#pragma unroll 1
          for (int a = 0; a < 4; ++a) {
            const int c0 = mg * 128 + a * 32 + j * 4;
            float t0[4], t1[4];
            const bool live = c0 < p.cin;
            if (live) {
#pragma unroll
              for (int i = 0; i < 4; ++i) { t0[i] = ptab[c0 + i]; t1[i] = ptab[cin_pad + c0 + i]; }
            }
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int r = r0 + 32 * q;
              if (r >= p.KBr) break;
              const int ly = gly[q], lx = glx[q];
              // input position of box row r: row y0+ly+ty, column x0+lx (1x1) / x0-1+lx (3x3)
              const int y = y0 + ly + ty, xx = x0 + lx - (TAPS == 9 ? 1 : 0);
              const bool in = live && ly < p.kt && (unsigned)y < (unsigned)p.h && (unsigned)xx < (unsigned)p.w &&
                              (TAPS == 9 || x0 + lx < p.w);
              // the TMA writes 128B-swizzled rows (16-byte chunk j at j ^ (r & 7)); the MN-major
              // TF32 operand layout (128B_BASE32B) wants 32-byte chunks at (j/2) ^ (r & 3): every
              // row is permuted in place by its 8 threads (all read, then all write)
              const uint32_t rowb = a * p.KBr * 128 + r * 128;
              const uint32_t off = rowb + ((j ^ (r & 7)) << 4);
              const uint32_t dst = rowb + ((((j >> 1) ^ (r & 3)) << 5) | ((j & 1) << 4));
              float4 hi = make_float4(0.f, 0.f, 0.f, 0.f), lo = hi;
              if (in) {
                const float4 v = *reinterpret_cast<const float4*>(A + off);
                float f[4] = {v.x, v.y, v.z, v.w};
                if (p.x_pro == BNFF_PRO_BN_RELU) {
#pragma unroll
                  for (int i = 0; i < 4; ++i) f[i] = fmaxf(fmaf(f[i], t0[i], t1[i]), 0.f);
                } else if (p.x_pro == BNFF_PRO_RELU) {
#pragma unroll
                  for (int i = 0; i < 4; ++i) f[i] = fmaxf(f[i], 0.f);
                }
                split4(f, hi, lo);
              }
              __syncwarp();
              *reinterpret_cast<float4*>(A + dst) = hi;
              *reinterpret_cast<float4*>(AL + dst) = lo;
            }
          }
          // B: dy (BN_DX-transformed when deferred) at the k-block's output positions
          const bool dbias_here = need_db && mg == 0 && u == 0;  // dy is the same in every stage
#pragma unroll
          for (int b = 0; b < NBA; ++b) {
            const int co = nt * BN + b * 32 + j * 4;
            const bool live = co < p.cout;
            float q0[4] = {1.f, 1.f, 1.f, 1.f}, q1[4] = {0.f, 0.f, 0.f, 0.f}, q2[4] = {0.f, 0.f, 0.f, 0.f};
            if (live && xb) {
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                q0[i] = qtab[co + i]; q1[i] = qtab[npad + co + i]; q2[i] = qtab[2 * npad + co + i];
              }
            }
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int r = r0 + 32 * q;
              if (r >= p.KBr) break;
              const int ly = gly[q], lx = glx[q];
              // output position of K row r: (y0+ly, x0+lx); 3x3 rows carry 2 junk columns
              const bool in = live && ly < p.kt && y0 + ly < p.h && x0 + lx < p.w && lx < p.bw;
              const uint32_t rowb = b * p.KBr * 128 + r * 128;
              const uint32_t off = rowb + ((j ^ (r & 7)) << 4);
              const uint32_t dst = rowb + ((((j >> 1) ^ (r & 3)) << 5) | ((j & 1) << 4));
              float4 hi = make_float4(0.f, 0.f, 0.f, 0.f), lo = hi;
              if (in) {
                const float4 v = *reinterpret_cast<const float4*>(B + off);
                float f[4] = {v.x, v.y, v.z, v.w};
                if (xb) {
                  const float4 xv = *reinterpret_cast<const float4*>(X + off);
                  const float xf[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
                  for (int i = 0; i < 4; ++i) f[i] = fmaf(f[i], q0[i], fmaf(xf[i], q1[i], q2[i]));
                }
                if (dbias_here) {
#pragma unroll
                  for (int i = 0; i < 4; ++i) bacc[b][i] += f[i];
                }
                split4(f, hi, lo);
              }
              __syncwarp();
              *reinterpret_cast<float4*>(B + dst) = hi;
              *reinterpret_cast<float4*>(BL + dst) = lo;
            }
          }
          fence_proxy_async_smem();
          mbar_arrive(&full_bar[st]);
          if (++st == ST) { st = 0; ph ^= 1u; }
        }
      }
      if (need_db && mg == 0) {  // this unit's dbias partials, combined in fixed thread order
#pragma unroll
        for (int b = 0; b < NBA; ++b) {
#pragma unroll
          for (int i = 0; i < 4; ++i) { bred[i * LT + tid] = bacc[b][i]; bacc[b][i] = 0.f; }
          named_bar_sync(1, LT);
          if (tid < 32) {
            const int jc = tid >> 2, i = tid & 3;
            const int c = nt * BN + b * 32 + jc * 4 + i;
            float s = 0.f;
            for (int t = jc; t < LT; t += 8) s += bred[i * LT + t];
            if (c < p.cout) p.wsb[(long long)sp * p.cout + c] = s;
          }
          named_bar_sync(1, LT);
        }
      }
    }
  } else if (warp == PRODUCER) {
    // =============================== TMA producer ===============================
    const uint32_t tx_bytes = (uint32_t)p.rows * 128u * (4u + NBA * (xb ? 2u : 1u));
    int st = 0, round = 0;
    for (int ui = 0; ui < nun; ++ui) {
      int mg, nt, sp;
      unit_of(ui, mg, nt, sp);
      const int cnt = kb_count(sp);
      int img, y0, x0;
      kb_org(sp * p.kpt, img, y0, x0);
      for (int k = 0; k < cnt; ++k, kb_next(img, y0, x0)) {
        for (int u = 0; u < SPK; ++u) {
          const int ty = TAPS == 9 ? u - 1 : 0, xa = TAPS == 9 ? x0 - 1 : x0;
          if (round > 0) mbar_wait(&empty_bar[st], (round - 1) & 1);
          if (elect_one()) {
            mbar_arrive_expect_tx(&ld_bar[st], tx_bytes);
            const uint32_t A = smem_u32(stage(st));
            const uint32_t B = A + 2 * AB, X = B + 2 * BB;
#pragma unroll
            for (int a = 0; a < 4; ++a)
              tma_load_4d(A + a * p.KBr * 128, &p.tma_x, mg * 128 + a * 32, xa, y0 + ty, img, &ld_bar[st]);
#pragma unroll
            for (int b = 0; b < NBA; ++b) {
              tma_load_4d(B + b * p.KBr * 128, &p.tma_dy, nt * BN + b * 32, x0, y0, img, &ld_bar[st]);
              if (xb) tma_load_4d(X + b * p.KBr * 128, &p.tma_dyx, nt * BN + b * 32, x0, y0, img, &ld_bar[st]);
            }
          }
          __syncwarp();
          if (++st == ST) { st = 0; ++round; }
        }
      }
    }
    __syncwarp();
  } else if (warp == NTW) {
    // =============================== MMA issuer ===============================
    constexpr uint32_t idesc = make_idesc(128, BN, kFmtTF32, 1, 1);
    const int ksteps = (p.rows + 7) / 8;
    int st = 0;
    uint32_t ph = 0;
    for (int ui = 0; ui < nun; ++ui) {
      int mg, nt, sp;
      unit_of(ui, mg, nt, sp);
      const int cnt = kb_count(sp);
      if (ui >= 1) mbar_wait(&acce_bar, (ui - 1) & 1);
      tc_fence_after();
      for (int k = 0; k < cnt; ++k) {
        for (int u = 0; u < SPK; ++u) {
          mbar_wait(&full_bar[st], ph);
          tc_fence_after();
          const uint32_t A = smem_u32(stage(st));
          const uint32_t AL = A + AB, B = A + 2 * AB, BL = B + BB;
#pragma unroll 1
          for (int tx = 0; tx < TPS; ++tx) {  // horizontal taps: A shifted by tx rows (128 B)
            const uint32_t d = tmem + (u * TPS + tx) * AC;
#pragma unroll 1
            for (int kk = 0; kk < ksteps; ++kk) {
              // MN-major TF32 operands: 128-byte rows of 32 channels per K index, atoms KBr rows apart
              const uint64_t ah = make_sdesc(A + tx * 128 + kk * 1024, p.KBr * 128, 512, kLayoutSW128Base32);
              const uint64_t al = make_sdesc(AL + tx * 128 + kk * 1024, p.KBr * 128, 512, kLayoutSW128Base32);
              const uint64_t bh = make_sdesc(B + kk * 1024, p.KBr * 128, 512, kLayoutSW128Base32);
              const uint64_t bl = make_sdesc(BL + kk * 1024, p.KBr * 128, 512, kLayoutSW128Base32);
              const uint32_t acc = (k > 0 || kk > 0) ? 1u : 0u;
              if constexpr (STK) {  // B_lo's atoms follow B_hi's at the same atom stride
                constexpr uint32_t idesc2 = make_idesc(128, 2 * BN, kFmtTF32, 1, 1);
                umma_tf32_elect(d, ah, bh, idesc2, acc);
                umma_tf32_elect(d + BN, al, bh, idesc, 1u);
                (void)bl;
              } else {
                umma_tf32_elect(d, ah, bh, idesc, acc);
                umma_tf32_elect(d, ah, bl, idesc, 1u);
                umma_tf32_elect(d, al, bh, idesc, 1u);
              }
            }
          }
          umma_commit_elect(&empty_bar[st]);
          if (++st == ST) { st = 0; ph ^= 1u; }
        }
      }
      umma_commit_elect(&accf_bar);
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
      const int ci = mg * 128 + row;
#pragma unroll 1
      for (int u = 0; u < TAPS; ++u) {
        float* dst = p.ws + (((long long)sp * TAPS + u) * p.cin + ci) * p.cout + nt * BN;
#pragma unroll 1
        for (int c16 = 0; c16 < BN; c16 += 16) {
          float v[16];
          tmem_ld16(tmem + u * AC + c16 + ((uint32_t)(quad * 32) << 16), v);
          if constexpr (STK) {
            float v2[16];
            tmem_ld16(tmem + u * AC + BN + c16 + ((uint32_t)(quad * 32) << 16), v2);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] += v2[i];
          } else {
            tmem_ld_wait();
          }
          if (ci < p.cin && nt * BN + c16 < p.cout) {
#pragma unroll
            for (int q = 0; q < 16; q += 4)
              *reinterpret_cast<float4*>(dst + c16 + q) = make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&acce_bar);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == NTW) tmem_dealloc<TCOLS>(tmem);
}

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
struct Plan {
  int ok, BN, bw, kt, xb, tpi, KBr, nkb, kpt, splits, MG, NT, stages, RS, rows;
};

inline int num_sms32() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
  }
  return n;
}

template <int BN>
inline int pick_stages(int KBr, bool xop, int cin_pad, int npad) {
  for (int s = MAXST; s >= 2; --s)
    if (smem_total<BN>(KBr, xop, s, cin_pad, npad) <= SMEM_BUDGET) return s;
  return 0;
}

inline Plan plan(int n, int h, int w, int cin, int cout, int kh, bool xop) {
  Plan q{};
  if (cin % 32 || cout % 32) return q;
  // N tile: 3x3 -> 32 (9 taps x 32 TMEM columns); 1x1 -> up to 128 (one x transform serves all
  // output channels; BNFF_WG32_BN caps it for A/B)
  static int bn_cap = -1;
  if (bn_cap < 0) {
    const char* e = getenv("BNFF_WG32_BN");
    bn_cap = e ? atoi(e) : 128;
  }
  q.BN = (kh == 3 || cout <= 32) ? 32 : (cout >= 128 && bn_cap >= 128 ? 128 : 64);
  // k-blocks of ~32 pixels (whole rows of small maps, row pieces of wide ones): short stages
  // keep 3-4 of them in flight at 8 bytes per operand element.  3x3: box rows of bw + 2
  // (the input row with its halo; for the output side the 2 trailing columns are junk, zeroed)
  // so the horizontal taps are K-row shifts of one box; A needs 2 rows past the last K row
  if (kh == 3) {
    q.bw = w < 30 ? w : 30;
    q.kt = w < 30 ? 32 / (w + 2) : 1;
    if (q.kt < 1) q.kt = 1;
    q.RS = q.bw + 2;
  } else {
    // 32-row k-blocks (BNFF_WG32_KB overrides them for the 128-wide tiles, A/B only: 16-row
    // blocks with four stages in flight measured 14% slower than two 32-row stages)
    static int kb_env = -1;
    if (kb_env < 0) {
      const char* e = getenv("BNFF_WG32_KB");
      kb_env = e ? atoi(e) : 32;
    }
    const int tgt = q.BN == 128 ? kb_env : 32;
    q.bw = w < tgt ? w : tgt;
    for (int d = tgt; w > tgt && d > tgt / 2; --d)  // row pieces that tile the row exactly
      if (w % d == 0) { q.bw = d; break; }
    q.kt = w < tgt ? tgt / w : 1;
    if (q.kt < 1) q.kt = 1;
    q.RS = q.bw;
  }
  if (q.kt > h) q.kt = h;
  q.xb = (w + q.bw - 1) / q.bw;
  q.tpi = (h + q.kt - 1) / q.kt;
  q.rows = q.kt * q.RS;
  q.KBr = ((q.rows + 7) / 8 * 8 + (kh == 3 ? 2 : 0) + 7) / 8 * 8;
  if (q.KBr > 64) return q;
  q.nkb = n * q.tpi * q.xb;
  q.MG = (cin + 127) / 128;
  q.NT = (cout + q.BN - 1) / q.BN;
  q.stages = q.BN == 32 ? pick_stages<32>(q.KBr, xop, q.MG * 128, q.NT * q.BN)
           : q.BN == 64 ? pick_stages<64>(q.KBr, xop, q.MG * 128, q.NT * q.BN)
                        : pick_stages<128>(q.KBr, xop, q.MG * 128, q.NT * q.BN);
  if (q.stages < 2) return q;
  // CTA targets of the split planning (BNFF_WG32_T3 / BNFF_WG32_T1, A/B; default one per SM):
  // every split writes a taps x 128 x BN fp32 partial tile, and the weight gradients run beside
  // the dgrad chain on the side stream
  static int t3 = -1, t1 = -1;
  if (t3 < 0) {
    const char* e = getenv("BNFF_WG32_T3");
    t3 = e ? atoi(e) : 0;
    e = getenv("BNFF_WG32_T1");
    t1 = e ? atoi(e) : 0;
  }
  const int tk = kh == 3 ? t3 : t1;
  const int target = tk > 0 ? tk : num_sms32();
  int splits = (target + q.MG * q.NT - 1) / (q.MG * q.NT);
  // >= min_kpt k-blocks per split (the partial tile a split writes is TAPS x 128 x BN floats)
  const int maxs = q.nkb / wg_min_kpt() > 0 ? q.nkb / wg_min_kpt() : 1;
  if (splits > maxs) splits = maxs;
  if (splits < 1) splits = 1;
  q.kpt = (q.nkb + splits - 1) / splits;
  q.splits = (q.nkb + q.kpt - 1) / q.kpt;
  q.ok = 1;
  return q;
}

template <int BN, int TAPS>
int launch(P p, cudaStream_t st) {
  auto kern = wgrad_f32_kernel<BN, TAPS>;
  const bool xop = p.dy_pro == BNFF_PRO_BN_DX;
  const int smem = smem_total<BN>(p.KBr, xop, p.stages, p.MG * 128, p.NT * BN);
  static int attr = 0;
  if (smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(wgrad f32)");
    attr = smem;
  }
  const int grid = p.units < num_sms32() ? p.units : num_sms32();
  bnff::launch(kern, dim3(grid), dim3(THREADS), smem, st, p);
  return check_launch("wgrad f32");
}

}  // namespace wg32
}  // namespace bnff

using namespace bnff;

// workspace floats of bnff_window_wgrad_f32: [splits][taps][cin][cout] + [splits][cout]
extern "C" int64_t bnff_wgrad_f32_ws(int32_t n, int32_t h, int32_t w, int32_t kh, int32_t c_in, int32_t c_out) {
  const wg32::Plan q = wg32::plan(n, h, w, c_in, c_out, kh, true);
  if (!q.ok) return 0;
  return (int64_t)q.splits * kh * kh * c_in * c_out + (int64_t)q.splits * c_out;
}

// fp32 weight gradient of a stride-1 1x1 / 3x3 (pad 1) conv; wg_reduce_kernel sums the splits.
// Returns -100 when the shape has no plan (the caller uses the generic implicit GEMM).
extern "C" int bnff_wgrad_f32_partials(bnff_view x, int32_t x_pro, bnff_coef x_coef, bnff_view dy, bnff_view dy_x,
                                       int32_t dy_pro, bnff_coef dy_coef, int32_t kh, float* ws, int32_t want_db,
                                       int32_t* splits_out, void* stream) {
  const bool xop = dy_pro == BNFF_PRO_BN_DX;
  const wg32::Plan q = wg32::plan((int)x.n, (int)x.h, (int)x.w, (int)x.c, (int)dy.c, kh, xop);
  if (!q.ok) return -100;
  wg32::P p{};
  p.n = (int)x.n; p.h = (int)x.h; p.w = (int)x.w; p.cin = (int)x.c; p.cout = (int)dy.c;
  p.kh = kh; p.pad = kh / 2;
  p.bw = q.bw; p.kt = q.kt; p.xb = q.xb; p.tpi = q.tpi; p.KBr = q.KBr; p.nkb = q.nkb; p.kpt = q.kpt;
  p.RS = q.RS; p.rows = q.rows;
  p.splits = q.splits; p.MG = q.MG; p.NT = q.NT; p.units = q.MG * q.NT * q.splits; p.stages = q.stages;
  p.x_pro = x_pro; p.x_coef = x_coef; p.dy_pro = dy_pro; p.dy_coef = dy_coef;
  p.ws = ws;
  p.wsb = want_db ? ws + (long long)q.splits * kh * kh * p.cin * p.cout : nullptr;
  const uint32_t box[4] = {32u, (uint32_t)q.RS, (uint32_t)q.kt, 1u};
  if (!encode_nhwc(&p.tma_x, 4, x.ptr, x.n, x.h, x.w, x.c, x.row_stride, 4, box) ||
      !encode_nhwc(&p.tma_dy, 4, dy.ptr, dy.n, dy.h, dy.w, dy.c, dy.row_stride, 4, box) ||
      (xop && !encode_nhwc(&p.tma_dyx, 4, dy_x.ptr, dy_x.n, dy_x.h, dy_x.w, dy_x.c, dy_x.row_stride, 4, box)))
    return set_error(BNFF_ERR_CUDA, "wgrad f32: cuTensorMapEncodeTiled failed");
  *splits_out = q.splits;
  cudaStream_t st = (cudaStream_t)stream;
  if (kh == 3) return wg32::launch<32, 9>(p, st);  // 9 taps x 32 TMEM columns
  if (q.BN == 128) return wg32::launch<128, 1>(p, st);
  return q.BN == 32 ? wg32::launch<32, 1>(p, st) : wg32::launch<64, 1>(p, st);
}
