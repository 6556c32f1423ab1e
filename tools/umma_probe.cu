// umma_probe.cu -- B200 validation of the UMMA operand layouts / descriptors used
// by libbnff.  Runs small single-CTA GEMMs C[128,N] = A[128,K] * B[N,K]^T with
// operands written to shared memory by ordinary st.shared in a given canonical
// layout, and compares against a host reference.  Prints one PASS/FAIL line per
// configuration.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I..
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>
#include "../paper_1807_01702_b200/csrc/sm100.cuh"

using namespace bnff;

struct ProbeCfg {
  int esize;        // 2 = bf16 (kind::f16), 4 = tf32
  int a_mn, b_mn;   // operand majorness (0 = K-major, 1 = MN-major)
  int N;            // 64 or 128
  int K;            // total K
  int layout_mn;    // layout type for MN-major operands
  int mn_kgroup;    // rows per K group for MN-major (8 for SW128, 4 for base32)
  int swap_lbo_sbo; // MN-major: swap the meaning of LBO/SBO
  int row_shift;    // K-major A: start descriptor at this row of a 136-row tile
  int base_off_mode;// 0: base_offset = 0, 1: base_offset = row_shift & 7
  int k_sw64;       // K-major operands use 64B rows (SW64) instead of 128B (SW128)
  int mn_kshift;    // MN-major A: start the K rows at this offset of a (K+16)-row tile
};

// byte offset of (mn, k) for an operand with `rows` MN entries and `K` k entries
__device__ uint32_t op_off(const ProbeCfg& c, int mn_major, int mn, int k, int rows, int krows) {
  const int kb_elems = 128 / c.esize;  // elements of K per 128B row (K-major)
  if (!mn_major) {
    if (c.k_sw64) {                    // 64B rows: chunk ^= (row>>1)&3 (absolute-address swizzle)
      int kb = k / (64 / c.esize);
      int kbyte = (k % (64 / c.esize)) * c.esize;
      uint32_t off = kb * rows * 64 + mn * 64 + kbyte;
      return off ^ (((off >> 7) & 3u) << 4);
    }
    int kb = k / kb_elems;             // K block -> separate region
    int kbyte = (k % kb_elems) * c.esize;
    return kb * rows * 128 + kmajor_sw128_off(mn, kbyte);
  }
  // MN-major: region per 128B MN atom; inside it K rows of 128 B.
  uint32_t mnbyte = mn * c.esize;
  uint32_t atom = mnbyte >> 7;
  uint32_t inb = mnbyte & 127;
  uint32_t atom_bytes = krows * 128;
  if (c.layout_mn == kLayoutSW64 || c.layout_mn == kLayoutSW32) {
    uint32_t rowb = c.layout_mn == kLayoutSW64 ? 64 : 32;
    uint32_t atomb = rowb * krows;  // one atom holds all K rows
    uint32_t a2 = mnbyte / rowb, in2 = mnbyte % rowb;
    uint32_t off = a2 * atomb + k * rowb + in2;
    uint32_t mask = c.layout_mn == kLayoutSW64 ? 3 : 1;
    return off ^ (((off >> 7) & mask) << 4);
  }
  if (c.layout_mn == kLayoutSW128Base32) {
    // Swizzle<2,5,2>: 32B chunk index ^= (row & 3)
    uint32_t chunk = ((inb >> 5) ^ (k & 3)) & 3;
    return atom * atom_bytes + k * 128 + (chunk << 5) + (inb & 31);
  }
  return atom * atom_bytes + k * 128 + ((((inb >> 4) ^ (k & 7)) & 7) << 4) + (inb & 15);
}

__global__ void probe_kernel(ProbeCfg c, const float* A, const float* B, float* C) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int M = 128;
  const int arows = (c.row_shift >= 0 && !c.a_mn) ? 136 : 128;
  const int akrows = c.K + ((c.mn_kshift > 0 && c.a_mn) ? 16 : 0);
  uint8_t* sa = smem;
  uint8_t* sb = smem + 64 * 1024;
  int tid = threadIdx.x;
  // zero fill
  for (int i = tid; i < 64 * 1024 / 4; i += blockDim.x) {
    reinterpret_cast<uint32_t*>(sa)[i] = 0;
    reinterpret_cast<uint32_t*>(sb)[i] = 0;
  }
  __syncthreads();
  for (int i = tid; i < arows * akrows; i += blockDim.x) {
    int m = i / akrows, k = i % akrows;
    float v = A[m * akrows + k];
    uint32_t off = op_off(c, c.a_mn, m, k, arows, akrows);
    if (c.esize == 2) *reinterpret_cast<__nv_bfloat16*>(sa + off) = __float2bfloat16(v);
    else *reinterpret_cast<float*>(sa + off) = v;
  }
  for (int i = tid; i < c.N * c.K; i += blockDim.x) {
    int n = i / c.K, k = i % c.K;
    float v = B[n * c.K + k];
    uint32_t off = op_off(c, c.b_mn, n, k, c.N, c.K);
    if (c.esize == 2) *reinterpret_cast<__nv_bfloat16*>(sb + off) = __float2bfloat16(v);
    else *reinterpret_cast<float*>(sb + off) = v;
  }
  fence_proxy_async_smem();
  if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (tid < 32) tmem_alloc<256>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem = tmem_base;

  if (tid == 0) {
    const int ustep = 32 / c.esize;  // K per UMMA
    const uint32_t fmt = c.esize == 2 ? kFmtBF16 : kFmtTF32;
    const uint32_t idesc = make_idesc(M, c.N, fmt, c.a_mn, c.b_mn);
    const int kb_elems = 128 / c.esize;
    for (int k0 = 0; k0 < c.K; k0 += ustep) {
      uint64_t ad, bd;
      if (!c.a_mn && c.k_sw64) {
        int kbe = 64 / c.esize;
        int kb = k0 / kbe;
        uint32_t addr = smem_u32(sa) + kb * arows * 64 + (k0 % kbe) * c.esize;
        int rs = c.row_shift > 0 ? c.row_shift : 0;
        addr += rs * 64;
        ad = make_sdesc(addr, 16, 512, kLayoutSW64);
      } else if (!c.a_mn) {
        int kb = k0 / kb_elems;
        uint32_t addr = smem_u32(sa) + kb * arows * 128 + (k0 % kb_elems) * c.esize;
        int rs = c.row_shift > 0 ? c.row_shift : 0;
        addr += rs * 128;
        ad = make_sdesc(addr, 16, 1024, kLayoutSW128, c.base_off_mode ? (rs & 7) : 0);
      } else {
        uint32_t addr = smem_u32(sa) + (k0 + (c.mn_kshift > 0 ? c.mn_kshift : 0)) * 128;
        uint32_t lbo = akrows * 128, sbo = c.mn_kgroup * 128;
        if (c.swap_lbo_sbo) { uint32_t t = lbo; lbo = sbo; sbo = t; }
        ad = make_sdesc(addr, lbo, sbo, c.layout_mn);
      }
      if (!c.b_mn && c.k_sw64) {
        int kbe = 64 / c.esize;
        int kb = k0 / kbe;
        uint32_t addr = smem_u32(sb) + kb * c.N * 64 + (k0 % kbe) * c.esize;
        bd = make_sdesc(addr, 16, 512, kLayoutSW64);
      } else if (!c.b_mn) {
        int kb = k0 / kb_elems;
        uint32_t addr = smem_u32(sb) + kb * c.N * 128 + (k0 % kb_elems) * c.esize;
        bd = make_sdesc(addr, 16, 1024, kLayoutSW128);
      } else {
        uint32_t rowb = c.layout_mn == kLayoutSW64 ? 64 : (c.layout_mn == kLayoutSW32 ? 32 : 128);
        uint32_t addr = smem_u32(sb) + k0 * rowb;
        uint32_t lbo = c.K * rowb, sbo = c.mn_kgroup * rowb;
        if (c.swap_lbo_sbo) { uint32_t t = lbo; lbo = sbo; sbo = t; }
        bd = make_sdesc(addr, lbo, sbo, c.layout_mn);
      }
      if (c.esize == 2) umma_f16(tmem, ad, bd, idesc, k0 > 0);
      else umma_tf32(tmem, ad, bd, idesc, k0 > 0);
    }
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  int warp = tid / 32, lane = tid % 32;
  int row = warp * 32 + lane;
  for (int n0 = 0; n0 < c.N; n0 += 8) {
    float v[8];
    tmem_ld8(tmem + ((warp * 32) << 16) + n0, v);
    tmem_ld_wait();
    for (int j = 0; j < 8; ++j) C[row * c.N + n0 + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_dealloc<256>(tmem);
}

static float round_op(float x, int esize) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if (esize == 2) {  // bf16 RNE
    uint32_t r = ((u >> 16) & 1) + 0x7FFF;
    u = (u + r) & 0xFFFF0000u;
  } else {
    u &= 0xFFFFE000u;  // tf32 truncation (what the MMA reads)
  }
  float y;
  memcpy(&y, &u, 4);
  return y;
}

static int run(const char* name, ProbeCfg c) {
  const int M = 128;
  int arows = (c.row_shift >= 0 && !c.a_mn) ? 136 : 128;
  int akrows = c.K + ((c.mn_kshift > 0 && c.a_mn) ? 16 : 0);
  std::vector<float> A(arows * akrows), B(c.N * c.K), C(M * c.N), R(M * c.N);
  srand(1234);
  for (auto& v : A) v = round_op((rand() % 2001 - 1000) / 500.0f, c.esize);
  for (auto& v : B) v = round_op((rand() % 2001 - 1000) / 500.0f, c.esize);
  int rs = c.row_shift > 0 ? c.row_shift : 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < c.N; ++n) {
      double s = 0;
      int ks = (c.mn_kshift > 0 && c.a_mn) ? c.mn_kshift : 0;
      for (int k = 0; k < c.K; ++k) s += (double)A[(m + rs) * akrows + k + ks] * B[n * c.K + k];
      R[m * c.N + n] = (float)s;
    }
  float *dA, *dB, *dC;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dC, C.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dC, 0, C.size() * 4);
  int smem = 129 * 1024 + 1024;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_kernel<<<1, 128, smem>>>(c, dA, dB, dC);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%-48s CUDA ERROR %s\n", name, cudaGetErrorString(e));
    exit(1);
  }
  cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0, maxref = 0;
  for (int i = 0; i < M * c.N; ++i) {
    maxerr = fmax(maxerr, fabs(C[i] - R[i]));
    maxref = fmax(maxref, fabs(R[i]));
  }
  bool ok = maxerr <= 1e-3 * maxref;
  printf("%-48s %s maxerr=%.3e maxref=%.3e C[0]=%g R[0]=%g\n", name, ok ? "PASS" : "FAIL", maxerr,
         maxref, C[0], R[0]);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dC);
  return ok;
}

int main() {
  //                      es amn bmn  N    K  lay_mn kg swap shift bo
  run("bf16 K/K N64 K128", {2, 0, 0, 64, 128, 2, 8, 0, -1, 0});
  run("bf16 K/K N128 K128", {2, 0, 0, 128, 128, 2, 8, 0, -1, 0});
  run("bf16 MN/MN N64 K64", {2, 1, 1, 64, 64, 2, 8, 0, -1, 0});
  run("bf16 MN/MN N128 K64", {2, 1, 1, 128, 64, 2, 8, 0, -1, 0});
  run("bf16 MN/MN N128 K64 swapped", {2, 1, 1, 128, 64, 2, 8, 1, -1, 0});
  run("bf16 MN/K N128 K64", {2, 1, 0, 128, 64, 2, 8, 0, -1, 0});
  run("bf16 K/MN N64 K64", {2, 0, 1, 64, 64, 2, 8, 0, -1, 0});
  run("tf32 K/K N64 K64", {4, 0, 0, 64, 64, 2, 8, 0, -1, 0});
  run("tf32 K/K N128 K64", {4, 0, 0, 128, 64, 2, 8, 0, -1, 0});
  run("tf32 MN/MN N64 K32 sw128", {4, 1, 1, 64, 32, 2, 8, 0, -1, 0});
  run("tf32 MN/MN N64 K32 base32", {4, 1, 1, 64, 32, 1, 4, 0, -1, 0});
  run("tf32 MN/MN N64 K32 base32 kg8", {4, 1, 1, 64, 32, 1, 8, 0, -1, 0});
  for (int s = 1; s < 8; s += 3) {
    char nm[64];
    snprintf(nm, 64, "bf16 K/K rowshift %d bo=0", s);
    run(nm, {2, 0, 0, 64, 64, 2, 8, 0, s, 0});
    snprintf(nm, 64, "bf16 K/K rowshift %d bo=s", s);
    run(nm, {2, 0, 0, 64, 64, 2, 8, 0, s, 1});
  }
  run("bf16 K/K rowshift 8 bo=0", {2, 0, 0, 64, 64, 2, 8, 0, 8, 0});
  run("bf16 K/MN N32 sw64 (B)", {2, 0, 1, 32, 64, 4, 8, 0, -1, 0});
  run("bf16 K/MN N32 sw32 (B)", {2, 0, 1, 32, 64, 6, 8, 0, -1, 0});
  run("bf16 K/MN N16 sw32 (B)", {2, 0, 1, 16, 64, 6, 8, 0, -1, 0});
  run("tf32 K/MN N32 base32 (B)", {4, 0, 1, 32, 32, 1, 4, 0, -1, 0});
  run("tf32 MN/MN N128 K64 base32", {4, 1, 1, 128, 64, 1, 4, 0, -1, 0});
  run("bf16 MN/MN N256 K64", {2, 1, 1, 256, 64, 2, 8, 0, -1, 0});
  run("bf16 K/K N256 K64", {2, 0, 0, 256, 64, 2, 8, 0, -1, 0});
  // round 1b: layouts for the window-shift conv kernels
  for (int s = 0; s < 8; s += 3) {
    char nm[64];
    ProbeCfg c{2, 0, 0, 32, 64, 2, 8, 0, s, 0, 1, 0};
    snprintf(nm, 64, "bf16 K/K sw64 N32 K64 rowshift %d", s);
    run(nm, c);
    c.N = 128;
    snprintf(nm, 64, "bf16 K/K sw64 N128 K32 rowshift %d", s);
    c.K = 32;
    run(nm, c);
  }
  for (int s = 1; s < 16; s += 4) {
    char nm[64];
    ProbeCfg c{2, 1, 1, 32, 64, 2, 8, 0, -1, 0, 0, s};
    snprintf(nm, 64, "bf16 MN/MN N32(sw128 B) kshift %d", s);
    c.layout_mn = kLayoutSW128;
    run(nm, c);
  }
  {
    ProbeCfg c{2, 1, 1, 128, 64, 2, 8, 0, -1, 0, 0, 5};
    run("bf16 MN/MN N128 kshift 5", c);
  }
  return 0;
}
