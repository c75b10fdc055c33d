// Backward, query-stationary dQ pass for sm_100a.
//
// The fused backward (zp_attn_bwd.cu) is key-tile stationary: every (key
// tile, query block) step reduces a dQ tile into global memory through a
// shared-memory staging tile and TMA reduce-adds, and those bytes compete
// with the tensor-core operands for shared-memory bandwidth.  This pass
// computes dQ the other way round, like the forward: one CTA per (128-row
// query tile, query head) walks the KV tiles the tile can see (the same
// causal walk as the forward, attention_engine.py:113-136), recomputes
//
//   S  = Q K^T                  (SS, M=128 queries, N=128 keys)  -> TMEM
//   dP = dO V^T                 (SS)                             -> TMEM
//   dS = exp2(S*c - LSE2) * (dP - Delta)   (softmax warps, thread == query row)
//   dQ += dS K                  (TS: dS bf16 from TMEM, K MN-major) -> TMEM
//
// and writes dQ once per tile (read-modify-write of the fp32 accumulator, so
// ring rounds add up; no atomics: one CTA owns a (tile, head) per launch).
// The key-stationary kernel then runs without its dQ path (kDQ = false).
//
// TMEM (512 columns): S double-buffered [0,128) / [128,256) — dS (bf16x2)
// overwrites the first 64 columns of its S buffer once they are read — dP
// [256,384), dQ [384,512).  Shared memory: Q, dO (32 KB each), K ring (3 x 32
// KB: K is read by S(j) and, one tile later, by dQ(j)), V ring (2 x 32 KB).
//
// Roles (256 threads): warp 0 TMA producer, warp 1 TMEM allocator + MMA
// issuer, warps 4-7 dS (thread == query row) and the dQ epilogue.
#include "zp_tiles.cuh"

namespace zp {
namespace bwdq {

constexpr int kD = 128;
constexpr int kBM = 128;
constexpr int kThreads = 256;
constexpr uint32_t kTile = kBM * kD * 2;     // 32 KB
constexpr uint32_t kBox = 128 * 64 * 2;      // 16 KB (64 columns x 128 rows)
constexpr int kKStages = 3;
constexpr int kVStages = 2;
constexpr uint32_t kSmemQ = 0;
constexpr uint32_t kSmemDO = kTile;
constexpr uint32_t kSmemK = 2 * kTile;
constexpr uint32_t kSmemV = kSmemK + kKStages * kTile;
constexpr uint32_t kSmemBar = kSmemV + kVStages * kTile;
constexpr uint32_t kSmemBytes = kSmemBar + 256 + 1024;
static_assert(kSmemBytes <= 232448, "smem budget");

enum : int {
  B_QFULL = 0,
  B_KFULL = 1,    // +stage (3)
  B_KEMPTY = 4,   // +stage (3)
  B_VFULL = 7,    // +stage (2)
  B_VEMPTY = 9,   // +stage (2)
  B_SDP = 11,     // +buf (2): S(j), dP(j) in TMEM
  B_DPREAD = 13,  // dP(j) read by the dS warps
  B_DS = 14,      // +buf (2): dS(j) written
  B_DQ = 16,      // every dQ MMA done
  B_COUNT = 17
};

struct DqArgs {
  const zp_attn_item* items;  // head_pair field = the query head of the item
  const zp_kv_seg* segs;
  const float* lse;
  const float* delta;
  int lse_stride;
  float* dq;
  int hq;
  int group;
  float scale;
  float scale_log2;
};

__global__ void __launch_bounds__(kThreads, 1)
    attn_bwd_dq_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                       const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                       const DqArgs args) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t sbase = (raw + 1023u) & ~1023u;
  uint8_t* sgen = smem_raw + (sbase - raw);
  const uint32_t bar0 = sbase + kSmemBar;
  auto bar = [&](int i) -> uint32_t { return bar0 + 8u * uint32_t(i); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sgen + kSmemBar + 8 * B_COUNT);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const zp_attn_item it = args.items[blockIdx.x];
  const int h = it.head_pair;
  const int kvh = h / args.group;
  const int max_qpos = it.q_pos0 + it.q_len - 1;

  if (threadIdx.x == 0) {
    mbar_init(bar(B_QFULL), 1);
    for (int s = 0; s < kKStages; ++s) {
      mbar_init(bar(B_KFULL + s), 1);
      mbar_init(bar(B_KEMPTY + s), 1);
    }
    for (int s = 0; s < kVStages; ++s) {
      mbar_init(bar(B_VFULL + s), 1);
      mbar_init(bar(B_VEMPTY + s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar(B_SDP + b), 1);
      mbar_init(bar(B_DS + b), 4);
    }
    mbar_init(bar(B_DPREAD), 4);
    mbar_init(bar(B_DQ), 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(smem_u32(tmem_slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS[2] = {tmem, tmem + 128};
  const uint32_t tDP = tmem + 256, tDQ = tmem + 384;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- producer: Q, dO once; then K / V rings
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_do);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_last();
      mbar_expect_tx(bar(B_QFULL), 2 * kTile);
      for (int b = 0; b < 2; ++b) {
        tma_load_2d(sbase + kSmemQ + b * kBox, &tm_q, bar(B_QFULL), h * kD + b * 64, it.q_row0, pol_q);
        tma_load_2d(sbase + kSmemDO + b * kBox, &tm_do, bar(B_QFULL), h * kD + b * 64, it.q_row0, pol_q);
      }
      TileCursor cur(args.segs, it.seg_begin, it.seg_count, max_qpos);
      for (uint32_t j = 0; cur.next(); ++j) {
        const int ks = int(j % kKStages), vs = int(j % kVStages);
        if (j >= uint32_t(kKStages)) mbar_wait(bar(B_KEMPTY + ks), ((j / kKStages) - 1) & 1);
        mbar_expect_tx(bar(B_KFULL + ks), kTile);
        for (int b = 0; b < 2; ++b)
          tma_load_2d(sbase + kSmemK + ks * kTile + b * kBox, &tm_k, bar(B_KFULL + ks), kvh * kD + b * 64,
                      cur.row(), pol_kv);
        if (j >= uint32_t(kVStages)) mbar_wait(bar(B_VEMPTY + vs), ((j / kVStages) - 1) & 1);
        mbar_expect_tx(bar(B_VFULL + vs), kTile);
        for (int b = 0; b < 2; ++b)
          tma_load_2d(sbase + kSmemV + vs * kTile + b * kBox, &tm_v, bar(B_VFULL + vs), kvh * kD + b * 64,
                      cur.row(), pol_kv);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (whole warp, one elected lane per op)
    constexpr uint32_t idesc_ss = idesc_bf16_f32(128, 128, 0, 0);  // S, dP: A, B K-major
    constexpr uint32_t idesc_dq = idesc_bf16_f32(128, 128, 0, 1);  // dQ: A from TMEM, B = K MN-major
    const uint64_t q_desc = umma_desc_sw128(sbase + kSmemQ, 16, 1024);
    const uint64_t do_desc = umma_desc_sw128(sbase + kSmemDO, 16, 1024);
    const uint64_t k_kmaj = umma_desc_sw128(sbase + kSmemK, 16, 1024);
    const uint64_t v_kmaj = umma_desc_sw128(sbase + kSmemV, 16, 1024);
    const uint64_t k_mn = umma_desc_sw128(sbase + kSmemK, kBox, 1024);
    constexpr uint64_t t_step = kTile >> 4;
    int n = 0;
    {
      TileCursor cur(args.segs, it.seg_begin, it.seg_count, max_qpos);
      while (cur.next()) ++n;
    }
    mbar_wait(bar(B_QFULL), 0);
    tc_fence_after();
    for (int j = 0; j <= n; ++j) {
      if (j < n) {
        const int ks = j % kKStages, vs = j % kVStages;
        mbar_wait(bar(B_KFULL + ks), (j / kKStages) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int kk = 0; kk < kD / 16; ++kk) {
          const uint64_t off = ((kk >> 2) * kBox + (kk & 3) * 32) >> 4;
          mma_ss_w(tS[j & 1], q_desc + off, k_kmaj + t_step * ks + off, idesc_ss, kk > 0 ? 1u : 0u);
        }
        mbar_wait(bar(B_VFULL + vs), (j / kVStages) & 1);
        if (j > 0) mbar_wait(bar(B_DPREAD), (j - 1) & 1);  // dP(j-1) read out of TMEM
        tc_fence_after();
#pragma unroll 1
        for (int kk = 0; kk < kD / 16; ++kk) {
          const uint64_t off = ((kk >> 2) * kBox + (kk & 3) * 32) >> 4;
          mma_ss_w(tDP, do_desc + off, v_kmaj + t_step * vs + off, idesc_ss, kk > 0 ? 1u : 0u);
        }
        tc_commit_w(bar(B_SDP + (j & 1)));
        tc_commit_w(bar(B_VEMPTY + vs));
      }
      if (j > 0) {
        // dQ += dS(j-1) K(j-1): A = dS (bf16x2, 8 TMEM columns per 16 keys)
        const int p = j - 1, ks = p % kKStages;
        mbar_wait(bar(B_DS + (p & 1)), (p >> 1) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int kk = 0; kk < kTileKeys / 16; ++kk)
          mma_ts_w(tDQ, tS[p & 1] + kk * 8, k_mn + t_step * ks + uint64_t(kk * (2048 >> 4)), idesc_dq,
                   (p > 0 || kk > 0) ? 1u : 0u);
        tc_commit_w(bar(B_KEMPTY + ks));
      }
    }
    tc_commit_w(bar(B_DQ));
  } else if (warp >= 4) {
    // ---------------- dS = P * (dP - Delta), thread == query row; then dQ out
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    const uint32_t lane_bits = uint32_t(quad * 32) << 16;
    const bool ok = row < it.q_len;
    const int qpos = it.q_pos0 + row;
    const size_t ix = size_t(h) * args.lse_stride + it.q_row0 + row;
    // invalid rows: LSE = +inf makes P (and dS) exactly 0
    const float lse2 = ok ? args.lse[ix] * 1.4426950408889634f : INFINITY;
    const float dlt = ok ? args.delta[ix] : 0.f;
    const float c1 = args.scale_log2;
    TileCursor cur(args.segs, it.seg_begin, it.seg_count, max_qpos);
    int j = 0;
    for (; cur.next(); ++j) {
      const int buf = j & 1;
      mbar_wait(bar(B_SDP + buf), (j >> 1) & 1);
      tc_fence_after();
      const int kpos0 = cur.pos(), kv_valid = cur.valid();
      const bool masked = kv_valid < kTileKeys || kpos0 + kTileKeys - 1 > it.q_pos0;
      const int lim = min(kv_valid - 1, qpos - kpos0);  // last visible key column
      // the whole dP row first: dP(j+1) may then overwrite it while this
      // tile's dS is formed (dP minus Delta kept in registers)
      float dd[128];
      {
        uint32_t d0[32], d1[32], d2[32], d3[32];
        tmem_ld32(tDP + lane_bits + 0, d0);
        tmem_ld32(tDP + lane_bits + 32, d1);
        tmem_ld32(tDP + lane_bits + 64, d2);
        tmem_ld32(tDP + lane_bits + 96, d3);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar(B_DPREAD));
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          dd[u] = __uint_as_float(d0[u]) - dlt;
          dd[32 + u] = __uint_as_float(d1[u]) - dlt;
          dd[64 + u] = __uint_as_float(d2[u]) - dlt;
          dd[96 + u] = __uint_as_float(d3[u]) - dlt;
        }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t sr[32];
        tmem_ld32(tS[buf] + lane_bits + 32 * c, sr);
        tmem_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          float ds[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = 32 * c + 2 * u + e;
            float p = ex2(__uint_as_float(sr[2 * u + e]) * c1 - lse2);
            if (masked && col > lim) p = 0.f;
            ds[e] = p * dd[col];
          }
          pk[u] = pack_bf16(ds[0], ds[1]);
        }
        // dS over the S columns already read (chunk c reads [32c, 32c+32), writes [16c, 16c+16))
        tmem_st16(tS[buf] + lane_bits + 16 * c, pk);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(B_DS + buf));
    }
    // ---------------- dQ of this tile: fp32 read-modify-write (one owner per launch)
    mbar_wait(bar(B_DQ), 0);
    tc_fence_after();
    uint8_t* dst = reinterpret_cast<uint8_t*>(args.dq + (size_t(it.q_row0 + row) * args.hq + h) * kD);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t rr[32];
      tmem_ld32(tDQ + lane_bits + 32 * c, rr);
      tmem_wait_ld();
      if (ok && j > 0) {
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          uint32_t g8[8];
          ldg_v8(dst + c * 128 + w * 32, g8);
#pragma unroll
          for (int e = 0; e < 8; ++e)
            g8[e] = __float_as_uint(__uint_as_float(g8[e]) + __uint_as_float(rr[8 * w + e]) * args.scale);
          stg_v8(dst + c * 128 + w * 32, g8);
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

}  // namespace bwdq
}  // namespace zp

// ------------------------------------------------------------------ host side
#include "zp_host.h"

extern "C" int zp_attn_bwd_dq(const void* q, const void* k, const void* v, const void* dout, int q_rows,
                              int kv_rows, int kv_row_stride, int hq, int hkv, int head_dim, const float* lse,
                              const float* delta, int lse_stride, float* dq, const zp_attn_item* items,
                              int n_items, const zp_kv_seg* segs, float softmax_scale, void* stream) {
  using namespace zp::bwdq;
  if (head_dim != kD) return zp_fail(ZP_EINVAL, "zp_attn_bwd_dq: head_dim must be 128");
  if (hq <= 0 || hkv <= 0 || hq % hkv != 0) return zp_fail(ZP_EINVAL, "zp_attn_bwd_dq: need hq % hkv == 0");
  if (n_items < 0 || q_rows < 0 || kv_rows < 0 || kv_row_stride < hkv * kD)
    return zp_fail(ZP_EINVAL, "zp_attn_bwd_dq: bad sizes");
  if (n_items == 0) return ZP_OK;
  if (q_rows == 0 || kv_rows == 0) return zp_fail(ZP_EINVAL, "zp_attn_bwd_dq: empty q or kv with items");
  if (!q || !k || !v || !dout || !lse || !delta || !dq || !items || !segs)
    return zp_fail(ZP_EINVAL, "zp_attn_bwd_dq: null pointer");
  if (zp_check_device() != ZP_OK) return ZP_ENODEV;
  CUtensorMap tq, tdo, tk, tv;
  int rc;
  if ((rc = zp_make_tmap_2d_bf16(&tq, q, uint64_t(hq) * kD, uint64_t(q_rows), uint64_t(hq) * kD * 2, 64, 128)) !=
      ZP_OK)
    return rc;
  if ((rc = zp_make_tmap_2d_bf16(&tdo, dout, uint64_t(hq) * kD, uint64_t(q_rows), uint64_t(hq) * kD * 2, 64,
                                 128)) != ZP_OK)
    return rc;
  if ((rc = zp_make_tmap_2d_bf16(&tk, k, uint64_t(hkv) * kD, uint64_t(kv_rows), uint64_t(kv_row_stride) * 2, 64,
                                 128)) != ZP_OK)
    return rc;
  if ((rc = zp_make_tmap_2d_bf16(&tv, v, uint64_t(hkv) * kD, uint64_t(kv_rows), uint64_t(kv_row_stride) * 2, 64,
                                 128)) != ZP_OK)
    return rc;
  static bool attr_done[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return zp_fail(ZP_ENODEV, "zp_attn_bwd_dq: device");
  if (!attr_done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(attn_bwd_dq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(kSmemBytes));
    if (e != cudaSuccess) return zp_fail_cuda(e, "zp_attn_bwd_dq: smem attribute");
    attr_done[dev] = true;
  }
  DqArgs a;
  a.items = items;
  a.segs = segs;
  a.lse = lse;
  a.delta = delta;
  a.lse_stride = lse_stride;
  a.dq = dq;
  a.hq = hq;
  a.group = hq / hkv;
  a.scale = softmax_scale;
  a.scale_log2 = softmax_scale * 1.4426950408889634f;
  attn_bwd_dq_kernel<<<n_items, kThreads, kSmemBytes, reinterpret_cast<cudaStream_t>(stream)>>>(tq, tdo, tk, tv,
                                                                                                 a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return zp_fail_cuda(e, "zp_attn_bwd_dq: launch");
  return ZP_OK;
}
