// Probe: can one kernel mix tcgen05.mma.cta_group::2 (issued by the leader for
// the CTA pair) with tcgen05.mma.cta_group::1 (issued by each CTA on its own)?
#include <cstdio>
#include <vector>
#include "/root/repo/paper_2509_21841_b200/csrc/zp_ptx.cuh"
using namespace zp;

__device__ uint32_t sw_off(int r, int k) {  // bf16 element (r, k), K-major SW128, 64-wide rows
  const int byte = k * 2;
  return uint32_t((r >> 3) * 1024 + (r & 7) * 128 + ((((byte >> 4) ^ (r & 7)) & 7) << 4) + (byte & 15));
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) probe(float* out_pair, float* out_own) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* g = smem_raw + (base - raw);
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bars[2];
  const uint32_t cta = cluster_ctarank();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // A: 128 rows x 64 (16 KB) at +0; B half: 32 rows x 64 at +16384 (pair operand);
  // B own: 64 rows x 64 at +20480
  __nv_bfloat16* A = reinterpret_cast<__nv_bfloat16*>(g);
  for (int i = tid; i < 128 * 64; i += 128) {
    const int r = i / 64, k = i % 64;
    const float a = float(((r + 128 * int(cta)) * 3 + k * 5) % 7 - 3);
    *reinterpret_cast<__nv_bfloat16*>(g + sw_off(r, k)) = __float2bfloat16(a);
  }
  for (int i = tid; i < 32 * 64; i += 128) {
    const int r = i / 64, k = i % 64;  // global B row n = 32*cta + r
    const float b = float(((32 * int(cta) + r) * 2 + k * 3) % 5 - 2);
    *reinterpret_cast<__nv_bfloat16*>(g + 16384 + sw_off(r, k)) = __float2bfloat16(b);
  }
  for (int i = tid; i < 64 * 64; i += 128) {
    const int r = i / 64, k = i % 64;
    const float b = float((r * 7 + k * (1 + int(cta))) % 9 - 4);
    *reinterpret_cast<__nv_bfloat16*>(g + 20480 + sw_off(r, k)) = __float2bfloat16(b);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    mbar_init(smem_u32(&bars[0]), 1);
    mbar_init(smem_u32(&bars[1]), 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc_pair(smem_u32(&slot), 512);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0) {
    const uint64_t a_desc = umma_desc_sw128(base, 16, 1024);
    const uint64_t bp_desc = umma_desc_sw128(base + 16384, 16, 1024);
    const uint64_t bo_desc = umma_desc_sw128(base + 20480, 16, 1024);
    if (cta == 0) {
      // pair: D[256 x 64] at column 0 of both CTAs
      for (int kk = 0; kk < 4; ++kk)
        mma_ss_pair_w(tmem, a_desc + 2 * kk, bp_desc + 2 * kk, idesc_bf16_f32(256, 64, 0, 0), kk > 0 ? 1u : 0u);
      tc_commit_pair_w(smem_u32(&bars[0]), 0x3);
    }
    // own: D[128 x 64] at column 128 of this CTA
    for (int kk = 0; kk < 4; ++kk)
      mma_ss_w(tmem + 128, a_desc + 2 * kk, bo_desc + 2 * kk, idesc_bf16_f32(128, 64, 0, 0), kk > 0 ? 1u : 0u);
    tc_commit_w(smem_u32(&bars[1]));
  }
  mbar_wait(smem_u32(&bars[0]), 0);
  mbar_wait(smem_u32(&bars[1]), 0);
  tc_fence_after();
  uint32_t r0[32], r1[32], s0[32], s1[32];
  const uint32_t lb = uint32_t(warp * 32) << 16;
  tmem_ld32(tmem + lb, r0);
  tmem_ld32(tmem + lb + 32, r1);
  tmem_ld32(tmem + lb + 128, s0);
  tmem_ld32(tmem + lb + 160, s1);
  tmem_wait_ld();
  const int row = warp * 32 + lane + 128 * int(cta);
  for (int c = 0; c < 32; ++c) {
    out_pair[row * 64 + c] = __uint_as_float(r0[c]);
    out_pair[row * 64 + 32 + c] = __uint_as_float(r1[c]);
    out_own[row * 64 + c] = __uint_as_float(s0[c]);
    out_own[row * 64 + 32 + c] = __uint_as_float(s1[c]);
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) tmem_dealloc_pair(tmem, 512);
}

int main() {
  float *dp, *dn;
  cudaMalloc(&dp, 256 * 64 * 4);
  cudaMalloc(&dn, 256 * 64 * 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 1024 + 1024);
  probe<<<2, 128, 32 * 1024 + 1024>>>(dp, dn);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<float> hp(256 * 64), hn(256 * 64);
  cudaMemcpy(hp.data(), dp, hp.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hn.data(), dn, hn.size() * 4, cudaMemcpyDeviceToHost);
  int bad_p = 0, bad_n = 0;
  for (int R = 0; R < 256; ++R)
    for (int n = 0; n < 64; ++n) {
      double ep = 0, en = 0;
      const int cta = R / 128, r = R % 128;
      for (int k = 0; k < 64; ++k) {
        const double a = ((R * 3 + k * 5) % 7) - 3;
        const double b = ((n * 2 + k * 3) % 5) - 2;
        const double bo = ((n * 7 + k * (1 + cta)) % 9) - 4;
        ep += a * b;
        en += a * bo;
      }
      (void)r;
      if (hp[R * 64 + n] != float(ep)) { if (bad_p < 6) printf("pair R %d n %d got %f exp %f\n", R, n, hp[R*64+n], ep); ++bad_p; }
      if (hn[R * 64 + n] != float(en)) { if (bad_n < 6) printf("own R %d n %d got %f exp %f\n", R, n, hn[R*64+n], en); ++bad_n; }
    }
  printf("pair mismatches %d / %d, own mismatches %d / %d\n", bad_p, 256 * 64, bad_n, 256 * 64);
  printf("sample pair %f vs own %f\n", hp[5 * 64 + 7], hn[130 * 64 + 3]);
  return 0;
}
