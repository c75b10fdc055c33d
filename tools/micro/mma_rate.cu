// Microbenchmark: cycles per tcgen05.mma (kind::f16, cta_group::1, M=128, K=16)
// for N in {64, 128, 256}, SS (A and B from shared memory) and TS (A from
// TMEM).  One CTA per SM, one issuing warp; operands are zero tiles.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 mma_rate.cu -o mma_rate
#include <cstdio>
#include "../../paper_2509_21841_b200/csrc/zp_ptx.cuh"
using namespace zp;

template <int N, bool TS, int AMN = 0, int BMN = 0>
__global__ void __launch_bounds__(128, 1) mma_rate(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(smem_u32(&slot), 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0) {
    const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
    // K-major: LBO unused (16), SBO 1 KB between 8-row groups; MN-major: LBO =
    // 16 KB between 64-element swizzle atoms along M/N, SBO 1 KB between 8-row
    // groups along K (the backward's K^T / dS^T / dO operands)
    const uint64_t a = umma_desc_sw128(base, AMN ? 16384 : 16, 1024);
    const uint64_t b = umma_desc_sw128(base + 32768, BMN ? 16384 : 16, 1024);
    constexpr uint32_t idesc = idesc_bf16_f32(128, N, AMN, BMN);
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      // walk along K: 32 B inside the atom (K-major) or 2 KB = 16 rows (MN-major)
      const uint64_t offa = AMN ? uint64_t((i & 3) * 128) : uint64_t((i & 3) * 2);
      const uint64_t offb = BMN ? uint64_t((i & 3) * 128) : uint64_t((i & 3) * 2);
      if constexpr (TS) mma_ts_w(tmem + 256, tmem, b + offb, idesc, 1u);
      else mma_ss_w(tmem, a + offa, b + offb, idesc, 1u);
    }
    tc_commit_w(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int N, bool TS, int AMN = 0, int BMN = 0>
void run(int sms, unsigned long long* d, int iters) {
  auto k = mma_rate<N, TS, AMN, BMN>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<<<sms, 128, 100 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[1024];
  cudaMemcpy(h, d, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += double(h[i]);
  avg /= sms;
  printf("%s N=%3d A %s B %s: %.1f cycles/MMA (nominal %d) %s\n", TS ? "TS" : "SS", N, AMN ? "MN" : "K ",
         BMN ? "MN" : "K ", avg / iters, 128 * N / 256,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, sizeof(unsigned long long) * 1024);
  const int iters = 4096;
  run<64, false>(sms, d, iters);
  run<128, false>(sms, d, iters);
  run<256, false>(sms, d, iters);
  run<64, true>(sms, d, iters);
  run<128, true>(sms, d, iters);
  run<256, true>(sms, d, iters);
  run<64, false, 1, 1>(sms, d, iters);   // dQ^T = K^T dS^T in the backward
  run<64, false, 0, 1>(sms, d, iters);
  run<64, false, 1, 0>(sms, d, iters);
  run<128, false, 1, 1>(sms, d, iters);
  run<128, true, 0, 1>(sms, d, iters);   // dV += P^T dO (A in TMEM, B MN-major)
  return 0;
}
