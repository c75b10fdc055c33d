// Byte-movement kernels of the hot path (HBM / NVLink bound, no tensor cores):
//   * copy_rows   - 16-byte vectorised row-range gather/scatter; packs the KV
//                   set a ring position sends onward (attention_engine.py:
//                   247-251) and moves kept / tail rows of the remap
//                   (remapping.py:187-245, permutation rule in DESIGN.md).
//   * remap push  - the remap's all-to-allv fused into one kernel: rows of
//                   M[me][d] are stored straight into rank d's landing buffer
//                   through CUDA-IPC peer pointers (NVLink), then per-pair
//                   release/acquire flags replace the collective's handshake.
#include "zp_host.h"
#include "../../include/zeppelin_b200.h"

namespace zp {

constexpr int kMoveThreads = 256;
constexpr int kUnroll = 4;

struct Range3 {
  int32_t dst_row0, src_row0, n_rows;
};

// grid.y = range, grid.x strides over the range's 16-byte vectors.
__global__ void __launch_bounds__(kMoveThreads)
    copy_rows_kernel(uint8_t* __restrict__ dst, int64_t dst_stride, const uint8_t* __restrict__ src,
                     int64_t src_stride, int64_t row_vecs, const Range3* __restrict__ ranges) {
  const Range3 r = ranges[blockIdx.y];
  const int64_t total = int64_t(r.n_rows) * row_vecs;
  const int64_t step = int64_t(gridDim.x) * kMoveThreads;
  int64_t i = int64_t(blockIdx.x) * kMoveThreads + threadIdx.x;
  for (; i + (kUnroll - 1) * step < total; i += kUnroll * step) {
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t e = i + u * step;
      const int64_t row = e / row_vecs, col = e - row * row_vecs;
      v[u] = __ldg(reinterpret_cast<const uint4*>(src + (r.src_row0 + row) * src_stride) + col);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t e = i + u * step;
      const int64_t row = e / row_vecs, col = e - row * row_vecs;
      reinterpret_cast<uint4*>(dst + (r.dst_row0 + row) * dst_stride)[col] = v[u];
    }
  }
  for (; i < total; i += step) {
    const int64_t row = i / row_vecs, col = i - row * row_vecs;
    reinterpret_cast<uint4*>(dst + (r.dst_row0 + row) * dst_stride)[col] =
        __ldg(reinterpret_cast<const uint4*>(src + (r.src_row0 + row) * src_stride) + col);
  }
}

// grid.y = destination rank; peer stores (st.global on IPC-mapped pointers).
__global__ void __launch_bounds__(kMoveThreads)
    remap_push_kernel(const uint8_t* __restrict__ src, int64_t row_bytes,
                      const int64_t* __restrict__ dst_ptrs, const int32_t* __restrict__ src_row0,
                      const int32_t* __restrict__ dst_row0, const int32_t* __restrict__ count) {
  const int d = blockIdx.y;
  const int n = count[d];
  if (n <= 0) return;
  const int64_t row_vecs = row_bytes / 16;
  const uint4* s = reinterpret_cast<const uint4*>(src + int64_t(src_row0[d]) * row_bytes);
  uint4* t = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(dst_ptrs[d]) +
                                      int64_t(dst_row0[d]) * row_bytes);
  const int64_t total = int64_t(n) * row_vecs;
  const int64_t step = int64_t(gridDim.x) * kMoveThreads;
  int64_t i = int64_t(blockIdx.x) * kMoveThreads + threadIdx.x;
  for (; i + (kUnroll - 1) * step < total; i += kUnroll * step) {
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) v[u] = __ldg(s + i + u * step);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) t[i + u * step] = v[u];
  }
  for (; i < total; i += step) t[i] = __ldg(s + i);
  __threadfence_system();
}

// Flag layout per rank (int32[2*world], IPC-shared): [0, world) "done" —
// sender s finished storing epoch e into my buffer; [world, 2*world) "ready" —
// rank s reached epoch e, so every earlier read of its buffers is complete.
__device__ __forceinline__ void st_release_sys(int32_t* p, int32_t v) {
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int32_t ld_acquire_sys(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Entry handshake: tell every peer we reached `epoch`, then wait until every
// rank we are about to store into has reached it too.
__global__ void remap_ready_kernel(const int64_t* __restrict__ flags_ptrs,
                                   const int32_t* __restrict__ count, int world, int me,
                                   int32_t epoch) {
  __threadfence_system();
  for (int d = threadIdx.x; d < world; d += blockDim.x)
    if (d != me) st_release_sys(reinterpret_cast<int32_t*>(flags_ptrs[d]) + world + me, epoch);
  for (int d = threadIdx.x; d < world; d += blockDim.x) {
    if (d == me || count[d] <= 0) continue;
    const int32_t* f = reinterpret_cast<const int32_t*>(flags_ptrs[me]) + world + d;
    while (ld_acquire_sys(f) < epoch) {
    }
  }
}

// Exit handshake: publish "done" to every rank we stored into, then wait for
// "done" from every rank that stores into us.
__global__ void remap_done_kernel(const int64_t* __restrict__ flags_ptrs,
                                  const int32_t* __restrict__ count,
                                  const int32_t* __restrict__ expect, int world, int me,
                                  int32_t epoch) {
  __threadfence_system();
  for (int d = threadIdx.x; d < world; d += blockDim.x)
    if (d != me && count[d] > 0) st_release_sys(reinterpret_cast<int32_t*>(flags_ptrs[d]) + me, epoch);
  for (int s = threadIdx.x; s < world; s += blockDim.x) {
    if (s == me || expect[s] == 0) continue;
    const int32_t* f = reinterpret_cast<const int32_t*>(flags_ptrs[me]) + s;
    while (ld_acquire_sys(f) < epoch) {
    }
  }
}

}  // namespace zp

static int grid_for(int64_t vecs, int per_y) {
  int64_t blocks = (vecs + zp::kMoveThreads * zp::kUnroll - 1) / (zp::kMoveThreads * zp::kUnroll);
  if (blocks < 1) blocks = 1;
  const int64_t cap = 148 * 8 / (per_y > 0 ? per_y : 1) + 1;
  return int(blocks < cap ? blocks : cap);
}

extern "C" int zp_copy_rows(void* dst, int64_t dst_stride_bytes, const void* src,
                            int64_t src_stride_bytes, int64_t row_bytes, const int32_t* ranges,
                            int n_ranges, int max_rows_per_range, void* stream) {
  if (n_ranges == 0 || max_rows_per_range == 0 || row_bytes == 0) return ZP_OK;
  if (n_ranges < 0 || n_ranges > 65535 || max_rows_per_range < 0 || row_bytes < 0)
    return zp_fail(ZP_EINVAL, "zp_copy_rows: bad range count");
  if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15u) ||
      ((dst_stride_bytes | src_stride_bytes | row_bytes) & 15))
    return zp_fail(ZP_EINVAL, "zp_copy_rows: pointers, strides and row bytes must be 16-byte aligned");
  if (!dst || !src || !ranges) return zp_fail(ZP_EINVAL, "zp_copy_rows: null pointer");
  if (zp_check_device() != ZP_OK) return ZP_ENODEV;
  const int64_t row_vecs = row_bytes / 16;
  dim3 grid(grid_for(int64_t(max_rows_per_range) * row_vecs, n_ranges), n_ranges);
  zp::copy_rows_kernel<<<grid, zp::kMoveThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<uint8_t*>(dst), dst_stride_bytes, reinterpret_cast<const uint8_t*>(src),
      src_stride_bytes, row_vecs, reinterpret_cast<const zp::Range3*>(ranges));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return zp_fail_cuda(e, "zp_copy_rows: launch");
  return ZP_OK;
}

extern "C" int zp_remap_push(const void* src, int64_t row_bytes, const int64_t* dst_ptrs,
                             const int32_t* src_row0, const int32_t* dst_row0, const int32_t* count,
                             const int64_t* flags_ptrs, const int32_t* expect, int world,
                             int my_rank, int32_t epoch, int max_count, void* stream) {
  if (world < 1 || world > 64 || my_rank < 0 || my_rank >= world || max_count < 0)
    return zp_fail(ZP_EINVAL, "zp_remap_push: bad world/rank");
  if ((reinterpret_cast<uintptr_t>(src) & 15u) || (row_bytes & 15) || row_bytes <= 0)
    return zp_fail(ZP_EINVAL, "zp_remap_push: src and row bytes must be 16-byte aligned");
  if (!dst_ptrs || !src_row0 || !dst_row0 || !count || !flags_ptrs || !expect)
    return zp_fail(ZP_EINVAL, "zp_remap_push: null table");
  if (zp_check_device() != ZP_OK) return ZP_ENODEV;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  zp::remap_ready_kernel<<<1, 64, 0, st>>>(flags_ptrs, count, world, my_rank, epoch);
  cudaError_t e0 = cudaGetLastError();
  if (e0 != cudaSuccess) return zp_fail_cuda(e0, "zp_remap_push: ready launch");
  if (max_count > 0) {
    dim3 grid(grid_for(int64_t(max_count) * (row_bytes / 16), world), world);
    zp::remap_push_kernel<<<grid, zp::kMoveThreads, 0, st>>>(
        reinterpret_cast<const uint8_t*>(src), row_bytes, dst_ptrs, src_row0, dst_row0, count);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return zp_fail_cuda(e, "zp_remap_push: launch");
  }
  zp::remap_done_kernel<<<1, 64, 0, st>>>(flags_ptrs, count, expect, world, my_rank, epoch);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return zp_fail_cuda(e, "zp_remap_push: signal launch");
  return ZP_OK;
}
