// Microbenchmark: tcgen05.ld (32x32b.x32, 4 KB per warp-load) throughput per SM
// with W loading warps (warp w reads its lane quarter w%4), one CTA per SM.
// Each warp issues DEPTH loads before one wait::ld (DEPTH x 32 registers in
// flight), ITERS times.  Prints bytes per SM clock.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tmem_rate.cu -o tmem_rate
#include <cstdio>
#include "../../paper_2509_21841_b200/csrc/zp_ptx.cuh"
using namespace zp;

template <int DEPTH>
__global__ void __launch_bounds__(512, 1) tmem_rate(int iters, int loaders, unsigned long long* out,
                                                    unsigned* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(smem_u32(&slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  unsigned acc = 0;
  unsigned long long t0 = 0, t1 = 0;
  if (warp < loaders) {
    const uint32_t base = tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t((warp >> 2) * 32 * DEPTH % 512);
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      uint32_t r[DEPTH][32];
#pragma unroll
      for (int d = 0; d < DEPTH; ++d) tmem_ld32(base + ((32 * d) & 511), r[d]);
      tmem_wait_ld();
#pragma unroll
      for (int d = 0; d < DEPTH; ++d) acc += r[d][0] ^ r[d][31];
    }
    t1 = clock64();
  }
  __syncthreads();
  if (warp < loaders && (threadIdx.x & 31) == 0) {
    atomicMax(&out[blockIdx.x], t1 - t0);
    sink[blockIdx.x * 16 + warp] = acc;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int DEPTH>
void run(int sms, unsigned long long* d, unsigned* sink, int loaders, int iters) {
  cudaMemset(d, 0, sizeof(unsigned long long) * 1024);
  tmem_rate<DEPTH><<<sms, 512>>>(iters, loaders, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[1024];
  cudaMemcpy(h, d, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += double(h[i]);
  avg /= sms;
  const double bytes = double(loaders) * iters * DEPTH * 4096.0;
  printf("loaders=%2d depth=%d: %.1f B/clk per SM (%.0f cycles per 4 KB warp-load per warp) %s\n", loaders, DEPTH,
         bytes / avg, avg / (iters * DEPTH), e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  unsigned* sink;
  cudaMalloc(&d, sizeof(unsigned long long) * 1024);
  cudaMalloc(&sink, sizeof(unsigned) * 16 * 1024);
  const int iters = 2048;
  for (int w : {1, 4, 8, 12, 16}) {
    run<1>(sms, d, sink, w, iters);
    run<2>(sms, d, sink, w, iters);
  }
  return 0;
}
