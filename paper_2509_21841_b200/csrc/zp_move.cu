// Byte-movement kernels of the hot path (HBM / NVLink bound, no tensor cores):
//   * copy_rows   - 16-byte vectorised row-range gather/scatter; packs the KV
//                   set a ring position sends onward (attention_engine.py:
//                   247-251) and moves kept / tail rows of the remap
//                   (remapping.py:187-245, permutation rule in DESIGN.md).
//   * remap push  - the remap's all-to-allv fused into one kernel: rows of
//                   M[me][d] are stored straight into rank d's landing buffer
//                   through CUDA-IPC peer pointers (NVLink), then per-pair
//                   release/acquire flags replace the collective's handshake.
#include <cstdio>

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

// dst[i] += src[i] (fp32, 16-byte vectors): the ring backward's running dK/dV
// partial sum of a travelling KV set (received total + this position's share).
__global__ void __launch_bounds__(kMoveThreads)
    add_f32_kernel(float4* __restrict__ dst, const float4* __restrict__ src, int64_t n_vec) {
  const int64_t step = int64_t(gridDim.x) * kMoveThreads;
  for (int64_t i = int64_t(blockIdx.x) * kMoveThreads + threadIdx.x; i < n_vec; i += step) {
    float4 a = dst[i];
    const float4 b = __ldg(src + i);
    a.x += b.x;
    a.y += b.y;
    a.z += b.z;
    a.w += b.w;
    dst[i] = a;
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

// Pull variant: the receiver reads its incoming rows straight out of the
// senders' buffers over NVLink (peer LDG.128, L1 no-allocate) and writes them
// locally.  grid.y = source rank.
__device__ __forceinline__ uint4 ld_peer(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

#ifndef ZP_PULL_UNROLL
#define ZP_PULL_UNROLL 8
#endif
// Each CTA copies one contiguous span of the source's rows: a warp's U loads
// cover U*512 consecutive bytes, keeping the remote DRAM access sequential.
__global__ void __launch_bounds__(kMoveThreads)
    remap_pull_kernel(uint8_t* __restrict__ dst, int64_t row_bytes, const int64_t* __restrict__ src_ptrs,
                      const int32_t* __restrict__ src_row0, const int32_t* __restrict__ dst_row0,
                      const int32_t* __restrict__ count) {
  constexpr int U = ZP_PULL_UNROLL;
  constexpr int64_t kSpan = int64_t(kMoveThreads) * U;  // vectors per CTA iteration
  const int sr = blockIdx.y;
  const int n = count[sr];
  if (n <= 0) return;
  const int64_t row_vecs = row_bytes / 16;
  const uint4* s = reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(src_ptrs[sr]) +
                                                  int64_t(src_row0[sr]) * row_bytes);
  uint4* t = reinterpret_cast<uint4*>(dst + int64_t(dst_row0[sr]) * row_bytes);
  const int64_t total = int64_t(n) * row_vecs;
  for (int64_t base = int64_t(blockIdx.x) * kSpan; base < total; base += int64_t(gridDim.x) * kSpan) {
    if (base + kSpan <= total) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ld_peer(s + base + u * kMoveThreads + threadIdx.x);
#pragma unroll
      for (int u = 0; u < U; ++u) t[base + u * kMoveThreads + threadIdx.x] = v[u];
    } else {
      for (int64_t i = base + threadIdx.x; i < total; i += kMoveThreads) t[i] = ld_peer(s + i);
    }
  }
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

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Bounded acquire-spin: a peer that never arrives (crashed rank, mismatched
// epochs) ends in a trap with a message instead of a hung GPU.
__device__ __forceinline__ void spin_until(const int32_t* f, int32_t epoch, uint64_t timeout_ns,
                                           const char* what, int me, int peer) {
  const uint64_t t0 = globaltimer_ns();
  while (int32_t(uint32_t(ld_acquire_sys(f)) - uint32_t(epoch)) < 0) {
    if (globaltimer_ns() - t0 > timeout_ns) {
      printf("zeppelin-b200: %s handshake timed out (rank %d waiting for rank %d, epoch %d, flag %d)\n", what, me,
             peer, epoch, ld_acquire_sys(f));
      __trap();
    }
  }
}

// Entry handshake: tell every peer we reached `epoch`, then wait until every
// rank we are about to store into has reached it too.
__global__ void remap_ready_kernel(const int64_t* __restrict__ flags_ptrs,
                                   const int32_t* __restrict__ count, int world, int me,
                                   int32_t epoch, uint64_t timeout_ns) {
  __threadfence_system();
  for (int d = threadIdx.x; d < world; d += blockDim.x)
    if (d != me) st_release_sys(reinterpret_cast<int32_t*>(flags_ptrs[d]) + world + me, epoch);
  for (int d = threadIdx.x; d < world; d += blockDim.x) {
    if (d == me || count[d] <= 0) continue;
    spin_until(reinterpret_cast<const int32_t*>(flags_ptrs[me]) + world + d, epoch, timeout_ns, "remap ready", me, d);
  }
}

// Exit handshake: publish "done" to every rank we stored into, then wait for
// "done" from every rank that stores into us.
__global__ void remap_done_kernel(const int64_t* __restrict__ flags_ptrs,
                                  const int32_t* __restrict__ count,
                                  const int32_t* __restrict__ expect, int world, int me,
                                  int32_t epoch, uint64_t timeout_ns) {
  __threadfence_system();
  for (int d = threadIdx.x; d < world; d += blockDim.x)
    if (d != me && count[d] > 0) st_release_sys(reinterpret_cast<int32_t*>(flags_ptrs[d]) + me, epoch);
  for (int s = threadIdx.x; s < world; s += blockDim.x) {
    if (s == me || expect[s] == 0) continue;
    spin_until(reinterpret_cast<const int32_t*>(flags_ptrs[me]) + s, epoch, timeout_ns, "remap done", me, s);
  }
}

}  // namespace zp

static int grid_for(int64_t vecs, int per_y) {
  int64_t blocks = (vecs + zp::kMoveThreads * zp::kUnroll - 1) / (zp::kMoveThreads * zp::kUnroll);
  if (blocks < 1) blocks = 1;
  const int64_t cap = 148 * 8 / (per_y > 0 ? per_y : 1) + 1;
  return int(blocks < cap ? blocks : cap);
}

extern "C" int zp_add_f32(float* dst, const float* src, int64_t n, void* stream) {
  if (n == 0) return ZP_OK;
  if (n < 0 || (n & 3) || !dst || !src || ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15u))
    return zp_fail(ZP_EINVAL, "zp_add_f32: need 16-byte aligned pointers and n % 4 == 0");
  if (zp_check_device() != ZP_OK) return ZP_ENODEV;
  const int64_t n_vec = n / 4;
  int64_t blocks = (n_vec + zp::kMoveThreads - 1) / zp::kMoveThreads;
  if (blocks > 148 * 8) blocks = 148 * 8;
  zp::add_f32_kernel<<<int(blocks), zp::kMoveThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<float4*>(dst), reinterpret_cast<const float4*>(src), n_vec);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return zp_fail_cuda(e, "zp_add_f32: launch");
  return ZP_OK;
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

namespace {
uint64_t g_spin_timeout_ns = 30ull * 1000000000ull;  // zp_set_spin_timeout_ms

enum : int { kPhaseReady = 1, kPhaseMove = 2, kPhaseDone = 4 };

int launch_ready(const int64_t* flags_ptrs, const int32_t* count, int world, int me, int32_t epoch,
                 cudaStream_t st, const char* what) {
  zp::remap_ready_kernel<<<1, 64, 0, st>>>(flags_ptrs, count, world, me, epoch, g_spin_timeout_ns);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ZP_OK : zp_fail_cuda(e, what);
}
int launch_done(const int64_t* flags_ptrs, const int32_t* count, const int32_t* expect, int world, int me,
                int32_t epoch, cudaStream_t st, const char* what) {
  zp::remap_done_kernel<<<1, 64, 0, st>>>(flags_ptrs, count, expect, world, me, epoch, g_spin_timeout_ns);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ZP_OK : zp_fail_cuda(e, what);
}
}  // namespace

extern "C" int zp_set_spin_timeout_ms(int64_t ms) {
  const uint64_t prev = g_spin_timeout_ns / 1000000ull;
  g_spin_timeout_ns = ms > 0 ? uint64_t(ms) * 1000000ull : 30ull * 1000000000ull;
  return int(prev);
}

extern "C" int zp_remap_push_phased(const void* src, int64_t row_bytes, const int64_t* dst_ptrs,
                                    const int32_t* src_row0, const int32_t* dst_row0, const int32_t* count,
                                    const int64_t* flags_ptrs, const int32_t* expect, int world, int my_rank,
                                    int32_t epoch, int max_count, int phases, void* stream) {
  if (world < 1 || world > 64 || my_rank < 0 || my_rank >= world || max_count < 0 || phases < 0 || phases > 7)
    return zp_fail(ZP_EINVAL, "zp_remap_push: bad world/rank/phases");
  if ((reinterpret_cast<uintptr_t>(src) & 15u) || (row_bytes & 15) || row_bytes <= 0)
    return zp_fail(ZP_EINVAL, "zp_remap_push: src and row bytes must be 16-byte aligned");
  if (!dst_ptrs || !src_row0 || !dst_row0 || !count || !flags_ptrs || !expect)
    return zp_fail(ZP_EINVAL, "zp_remap_push: null table");
  if (zp_check_device() != ZP_OK) return ZP_ENODEV;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int rc;
  if ((phases & kPhaseReady) &&
      (rc = launch_ready(flags_ptrs, count, world, my_rank, epoch, st, "zp_remap_push: ready launch")) != ZP_OK)
    return rc;
  if ((phases & kPhaseMove) && max_count > 0) {
    dim3 grid(grid_for(int64_t(max_count) * (row_bytes / 16), world), world);
    zp::remap_push_kernel<<<grid, zp::kMoveThreads, 0, st>>>(
        reinterpret_cast<const uint8_t*>(src), row_bytes, dst_ptrs, src_row0, dst_row0, count);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return zp_fail_cuda(e, "zp_remap_push: launch");
  }
  if (phases & kPhaseDone)
    return launch_done(flags_ptrs, count, expect, world, my_rank, epoch, st, "zp_remap_push: signal launch");
  return ZP_OK;
}

extern "C" int zp_remap_push(const void* src, int64_t row_bytes, const int64_t* dst_ptrs,
                             const int32_t* src_row0, const int32_t* dst_row0, const int32_t* count,
                             const int64_t* flags_ptrs, const int32_t* expect, int world,
                             int my_rank, int32_t epoch, int max_count, void* stream) {
  return zp_remap_push_phased(src, row_bytes, dst_ptrs, src_row0, dst_row0, count, flags_ptrs, expect, world,
                              my_rank, epoch, max_count, 7, stream);
}

extern "C" int zp_remap_pull_phased(void* dst, int64_t row_bytes, const int64_t* src_ptrs,
                                    const int32_t* src_row0, const int32_t* dst_row0, const int32_t* count,
                                    const int64_t* flags_ptrs, const int32_t* readers, int world, int my_rank,
                                    int32_t epoch, int max_count, int phases, void* stream) {
  if (world < 1 || world > 64 || my_rank < 0 || my_rank >= world || max_count < 0 || phases < 0 || phases > 7)
    return zp_fail(ZP_EINVAL, "zp_remap_pull: bad world/rank/phases");
  if ((reinterpret_cast<uintptr_t>(dst) & 15u) || (row_bytes & 15) || row_bytes <= 0)
    return zp_fail(ZP_EINVAL, "zp_remap_pull: dst and row bytes must be 16-byte aligned");
  if (!src_ptrs || !src_row0 || !dst_row0 || !count || !flags_ptrs || !readers)
    return zp_fail(ZP_EINVAL, "zp_remap_pull: null table");
  if (zp_check_device() != ZP_OK) return ZP_ENODEV;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int rc;
  // ready: my source rows are final for this epoch; wait for my sources (count > 0)
  if ((phases & kPhaseReady) &&
      (rc = launch_ready(flags_ptrs, count, world, my_rank, epoch, st, "zp_remap_pull: ready launch")) != ZP_OK)
    return rc;
  if ((phases & kPhaseMove) && max_count > 0) {
    dim3 grid(grid_for(int64_t(max_count) * (row_bytes / 16), world), world);
    zp::remap_pull_kernel<<<grid, zp::kMoveThreads, 0, st>>>(reinterpret_cast<uint8_t*>(dst), row_bytes,
                                                             src_ptrs, src_row0, dst_row0, count);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return zp_fail_cuda(e, "zp_remap_pull: launch");
  }
  // done: tell each source I finished reading it; wait until every reader of my
  // rows finished, so the caller may overwrite them
  if (phases & kPhaseDone)
    return launch_done(flags_ptrs, count, readers, world, my_rank, epoch, st, "zp_remap_pull: done launch");
  return ZP_OK;
}

extern "C" int zp_remap_pull(void* dst, int64_t row_bytes, const int64_t* src_ptrs,
                             const int32_t* src_row0, const int32_t* dst_row0, const int32_t* count,
                             const int64_t* flags_ptrs, const int32_t* readers, int world,
                             int my_rank, int32_t epoch, int max_count, void* stream) {
  return zp_remap_pull_phased(dst, row_bytes, src_ptrs, src_row0, dst_row0, count, flags_ptrs, readers, world,
                              my_rank, epoch, max_count, 7, stream);
}

extern "C" int zp_remap_pull_ce(void* dst, int64_t row_bytes, const int64_t* src_ptrs_host,
                                const int32_t* src_row0_host, const int32_t* dst_row0_host,
                                const int32_t* count_host, const int64_t* flags_ptrs,
                                const int32_t* count_dev, const int32_t* readers_dev, int world,
                                int my_rank, int32_t epoch, void* stream) {
  if (world < 1 || world > 64 || my_rank < 0 || my_rank >= world)
    return zp_fail(ZP_EINVAL, "zp_remap_pull_ce: bad world/rank");
  if (!src_ptrs_host || !src_row0_host || !dst_row0_host || !count_host || !flags_ptrs ||
      !count_dev || !readers_dev)
    return zp_fail(ZP_EINVAL, "zp_remap_pull_ce: null table");
  if (zp_check_device() != ZP_OK) return ZP_ENODEV;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int rc = launch_ready(flags_ptrs, count_dev, world, my_rank, epoch, st, "zp_remap_pull_ce: ready launch");
  if (rc != ZP_OK) return rc;
  cudaError_t e;
  for (int s = 0; s < world; ++s) {
    if (count_host[s] <= 0) continue;
    e = cudaMemcpyAsync(reinterpret_cast<uint8_t*>(dst) + int64_t(dst_row0_host[s]) * row_bytes,
                        reinterpret_cast<const uint8_t*>(src_ptrs_host[s]) + int64_t(src_row0_host[s]) * row_bytes,
                        size_t(count_host[s]) * size_t(row_bytes), cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return zp_fail_cuda(e, "zp_remap_pull_ce: copy");
  }
  return launch_done(flags_ptrs, count_dev, readers_dev, world, my_rank, epoch, st, "zp_remap_pull_ce: done launch");
}

extern "C" int zp_remap_push_ce(const void* src, int64_t row_bytes, const int64_t* dst_ptrs_host,
                                const int32_t* src_row0_host, const int32_t* dst_row0_host,
                                const int32_t* count_host, const int64_t* flags_ptrs,
                                const int32_t* count_dev, const int32_t* expect_dev, int world,
                                int my_rank, int32_t epoch, void* stream) {
  if (world < 1 || world > 64 || my_rank < 0 || my_rank >= world)
    return zp_fail(ZP_EINVAL, "zp_remap_push_ce: bad world/rank");
  if (!dst_ptrs_host || !src_row0_host || !dst_row0_host || !count_host || !flags_ptrs ||
      !count_dev || !expect_dev)
    return zp_fail(ZP_EINVAL, "zp_remap_push_ce: null table");
  if (zp_check_device() != ZP_OK) return ZP_ENODEV;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int rc = launch_ready(flags_ptrs, count_dev, world, my_rank, epoch, st, "zp_remap_push_ce: ready launch");
  if (rc != ZP_OK) return rc;
  cudaError_t e;
  for (int d = 0; d < world; ++d) {
    if (count_host[d] <= 0) continue;
    e = cudaMemcpyAsync(reinterpret_cast<uint8_t*>(dst_ptrs_host[d]) + int64_t(dst_row0_host[d]) * row_bytes,
                        reinterpret_cast<const uint8_t*>(src) + int64_t(src_row0_host[d]) * row_bytes,
                        size_t(count_host[d]) * size_t(row_bytes), cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return zp_fail_cuda(e, "zp_remap_push_ce: copy");
  }
  return launch_done(flags_ptrs, count_dev, expect_dev, world, my_rank, epoch, st, "zp_remap_push_ce: done launch");
}
