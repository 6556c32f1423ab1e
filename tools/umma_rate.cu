// umma_rate.cu -- issue-rate microbenchmark of tcgen05.mma kind::f16 (M=128, K=16 per
// instruction) on one CTA per SM: cycles per UMMA for N = 32..256, 128B vs 64B K-major
// swizzle, and A descriptors started at a row offset that is not a multiple of the
// swizzle atom (the 3x3 window taps).  Operand contents are irrelevant (zeros).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_rate tools/umma_rate.cu
#include <cstdio>
#include <cstdint>
#include "../paper_1807_01702_b200/csrc/sm100.cuh"

using namespace bnff;

struct Cfg {
  int N, sw64, row_shift, reps, kpm;  // kpm: UMMAs per commit
  int warp_issue;                     // 1: the whole warp runs the loop, elect.sync issues
};

__global__ void __launch_bounds__(128, 1) rate_kernel(Cfg c, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x;
  for (int i = tid; i < 160 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (tid < 32) tmem_alloc<512>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  if (c.warp_issue && tid < 32) {
    const uint32_t idesc = make_idesc(128, c.N, kFmtBF16, 0, 0);
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 96 * 1024);
    const uint32_t rowb = c.sw64 ? 64 : 128;
    const uint32_t lay = c.sw64 ? kLayoutSW64 : kLayoutSW128;
    const uint64_t a0 = make_sdesc(sa + c.row_shift * rowb, 16, 8 * rowb, lay);
    const uint64_t b0 = make_sdesc(sb, 16, 8 * rowb, lay);
    const int kk = (int)rowb / 32;
    uint32_t ph = 0;
    const unsigned long long t0 = clock64();
    for (int r = 0; r < c.reps; ++r) {
      for (int i = 0; i < c.kpm; ++i) {
        const int k = i % kk;
        umma_f16_elect(tmem + (r & 1) * 256, a0 + k * 2, b0 + k * 2, idesc, i > 0 ? 1u : 0u);
      }
      umma_commit_elect(&bar);
      mbar_wait(&bar, ph);
      ph ^= 1u;
    }
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0 && tid == 0) out[0] = t1 - t0;
  } else if (!c.warp_issue && tid == 0) {
    const uint32_t idesc = make_idesc(128, c.N, kFmtBF16, 0, 0);
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 96 * 1024);
    const uint32_t rowb = c.sw64 ? 64 : 128;
    const uint32_t lay = c.sw64 ? kLayoutSW64 : kLayoutSW128;
    const uint64_t a0 = make_sdesc(sa + c.row_shift * rowb, 16, 8 * rowb, lay);
    const uint64_t b0 = make_sdesc(sb, 16, 8 * rowb, lay);
    const int kk = (int)rowb / 32;  // K=16 steps per row
    uint32_t ph = 0;
    const unsigned long long t0 = clock64();
    for (int r = 0; r < c.reps; ++r) {
      for (int i = 0; i < c.kpm; ++i) {
        const int k = i % kk;
        umma_f16(tmem + (r & 1) * 256, a0 + k * 2, b0 + k * 2, idesc, i > 0 ? 1u : 0u);
      }
      umma_commit(&bar);
      mbar_wait(&bar, ph);
      ph ^= 1u;
    }
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_dealloc<512>(tmem);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int Ns[] = {32, 64, 128, 256};
  printf("%-5s %-6s %-5s %-9s %-5s %10s %12s %10s\n", "warp", "N", "sw", "rowshift", "kpm", "cyc/umma", "MAC/clk/SM", "pct_peak");
  for (int wi = 0; wi < 2; ++wi)
  for (int sw64 = 0; sw64 < 2; ++sw64)
    for (int rs : {0, 3})
      for (int N : Ns)
        for (int kpm : {8, 64}) {
          Cfg c{N, sw64, rs, 50, kpm, wi};
          rate_kernel<<<148, 128, 200 * 1024>>>(c, d);
          rate_kernel<<<148, 128, 200 * 1024>>>(c, d);
          unsigned long long cyc = 0;
          cudaError_t e = cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
          if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
          const double per = (double)cyc / (c.reps * kpm);
          const double mac = 128.0 * N * 16 / per;
          printf("%-5d %-6d %-5s %-9d %-5d %10.1f %12.0f %9.1f%%\n", wi, N, sw64 ? "64B" : "128B", rs, kpm, per, mac,
                 100.0 * mac / 8192.0);
        }
  return 0;
}
