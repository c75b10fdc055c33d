// Causal varlen / ring-round flash attention BACKWARD for sm_100a.
//
// The reference charges the backward pass as a multiple of the forward
// (topology.py:37, simulator.py:304) and runs it in reverse queue order
// (SURVEY 8(f) row 2).  This kernel executes it for the same
// work the forward executes: LocalTasks (attention_engine.py:260-265) and ring
// rounds (attention_engine.py:229-244, KV of position (i-r) mod g), with the
// causal rule of visible_pairs (attention_engine.py:113-136) in global
// positions.  Given Q, K, V, dO, the forward LSE and Delta = rowsum(dO * O):
//
//   P  = exp(S*scale - LSE),  S = Q K^T
//   dV += P^T dO
//   dS  = scale * P * (dO V^T - Delta)   (the scale folded into dS once)
//   dK += dS^T Q
//   dQ += dS K
//
// CTA = one work item = 128 keys of one KV head (KV-tile stationary) against
// every query block (64 rows) of every query head of the GQA group that can see
// them.  All products are formed transposed so that M = 128 (keys or dims)
// for every tcgen05.mma:
//   S^T  = K  Q^T    (M=128 keys, N=64 queries, K=128 dims)   -> TMEM
//   dP^T = V  dO^T   (same shape)                              -> TMEM
//   dV  += P^T dO    (M=128 keys, N=128 dims, K=64 queries; A in TMEM) -> TMEM
//   dK  += dS^T Q    (same shape, A in TMEM)                            -> TMEM
//   dQ^T = K^T dS^T  (M=128 dims, N=64 queries, K=128 keys)    -> TMEM, then
//                     fp32 reductions into the dQ accumulator
// TMEM (512 columns): S^T/dQ^T buffers [0,128) (2 x 64), dP^T [128,256)
// (2 x 64), dV [256,384), dK [384,512).  The softmax warps write P^T (bf16x2)
// over the S^T columns they have read and dS^T over the dP^T columns: they are
// the TMEM A operands of dV += P^T dO and dK += dS^T Q (no shared-memory A
// traffic).  dS^T also goes to shared memory (SWIZZLE_128B, K-major rows of
// 64 queries) as the MN-major B operand of dQ^T.
//
// Roles (384 threads): warp 0 TMA producer (K, V once; Q, dO per step,
// double-buffered), warp 1 TMEM allocator + MMA issuer, warps 4-7 P/dS
// (thread == key row) and the dK/dV epilogue, warps 8-11 dQ reduction
// (thread == head dim).
#include "zp_ptx.cuh"
#include "../../include/zeppelin_b200.h"

namespace zp {
namespace bwd {

constexpr int kD = 128;
constexpr int kBK = 128;  // keys per item
constexpr int kBQ = 64;   // query rows per step
constexpr int kThreads = 384;
constexpr uint32_t kKVTile = kBK * kD * 2;   // 32 KB
constexpr uint32_t kKVBox = kBK * 64 * 2;    // 16 KB (64 dims x 128 rows)
constexpr uint32_t kQTile = kBQ * kD * 2;    // 16 KB
constexpr uint32_t kQBox = kBQ * 64 * 2;     // 8 KB (64 dims x 64 rows)
constexpr uint32_t kPTile = kBK * kBQ * 2;   // 16 KB (128 keys x 64 queries)

constexpr uint32_t kSmemK = 0;
constexpr uint32_t kSmemV = kSmemK + kKVTile;
constexpr uint32_t kSmemQ = kSmemV + kKVTile;     // kQStages buffers
constexpr int kQStages = 3;                          // Q / dO ring depth (TMA latency > one step; 2 measured 5% slower)
constexpr uint32_t kSmemDO = kSmemQ + kQStages * kQTile;
constexpr uint32_t kSmemDST = kSmemDO + kQStages * kQTile;
constexpr uint32_t kSmemDQ = kSmemDST + 2 * kPTile;   // dQ staging: 4 boxes [64 queries][32 dims] fp32
constexpr uint32_t kDQBox = kBQ * 32 * 4;             // 8 KB
constexpr uint32_t kSmemBar = kSmemDQ + 4 * kDQBox;
// per softmax warp: LSE2 / Delta of the step's 64 queries (broadcast reads
// replace 128 shuffles per thread per step).  No alignment slack: the dynamic
// shared-memory window starts 1024-aligned (checked in the kernel).
constexpr uint32_t kSmemLD = kSmemBar + 256;
constexpr uint32_t kSmemBytes = kSmemLD + 4 * 512;

enum : int {
  B_KV = 0,
  B_QDO_FULL = 1,   // +stage (3)
  B_QDO_EMPTY = 4,  // +stage (3)
  B_SDP_FULL = 7,   // +buf
  B_PDS_FULL = 9,   // +buf
  B_PDS_EMPTY = 11, // +buf
  B_DQ_FULL = 13,   // +buf
  B_DQ_EMPTY = 15,  // +buf
  B_DKV = 17,
  B_COUNT = 18
};
static_assert(kSmemBytes <= 232448, "smem budget");

struct BwdArgs {
  const zp_bwd_item* items;
  const zp_kv_seg* qsegs;
  const float* lse;
  const float* delta;
  int lse_stride;
  float* dq;
  float* dk;
  float* dv;
  int hq;
  int hkv;
  int group;
  float scale;
  float scale_log2;
  int q_rows;   // bounds of q / dO / dq and k / v / dk / dv (checked in -DZP_CHECKS builds)
  int kv_rows;
};

template <bool B>
struct BoolC {
  static constexpr bool value = B;
};

// Steps of an item: query segments in order, 64-row blocks from the first one
// that can see the item's first key, and the query heads of the GQA group.
struct StepCursor {
  const zp_kv_seg* segs;
  int s, end, kv_pos0, group, b, nb, hh;
  zp_kv_seg g;
  __device__ __forceinline__ StepCursor(const zp_kv_seg* sg, int begin, int count, int kvp, int grp)
      : segs(sg), s(begin - 1), end(begin + count), kv_pos0(kvp), group(grp), b(0), nb(0), hh(grp - 1) {}
  __device__ __forceinline__ bool next() {
    if (++hh < group) return true;
    hh = 0;
    if (++b < nb) return true;
    while (++s < end) {
      g = segs[s];
      if (g.len > 0 && g.pos0 + g.len - 1 >= kv_pos0) {
        const int d = kv_pos0 - g.pos0;
        b = d > 0 ? d / kBQ : 0;
        nb = (g.len + kBQ - 1) / kBQ;
        return true;
      }
    }
    return false;
  }
  __device__ __forceinline__ int row() const { return g.row0 + b * kBQ; }
  __device__ __forceinline__ int pos() const { return g.pos0 + b * kBQ; }
  __device__ __forceinline__ int valid() const { return min(kBQ, g.len - b * kBQ); }
};

#ifdef ZP_TRACE
__device__ unsigned long long g_zp_btrace[4096];
// per item (CTA): globaltimer at entry / K,V landed / exit, and the step count
__device__ unsigned long long g_zp_bitems[16384 * 4];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
  return t;
}
#define ZP_BITEM(e, v)                                                    \
  do {                                                                    \
    if (blockIdx.x < 16384) g_zp_bitems[blockIdx.x * 4 + (e)] = (v);      \
  } while (0)
#define ZP_BSTAMP(slot)                                                  \
  do {                                                                   \
    if (blockIdx.x == 0 && (slot) >= 0 && (slot) < 4096) {               \
      unsigned long long c_;                                             \
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(c_)::"memory");        \
      g_zp_btrace[slot] = c_;                                            \
    }                                                                    \
  } while (0)
#else
#define ZP_BSTAMP(slot) \
  do {                  \
  } while (0)
#endif

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// TMA reduce-add of a shared-memory tile into global fp32 (atomic per element in L2).
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* m, uint32_t src, int x, int y) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(x), "r"(y), "r"(src)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void st_shared_f32(uint32_t addr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void ld_shared_v4f(uint32_t addr, float (&v)[4]) {
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "r"(addr)
               : "memory");
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}

// Byte offset of 16-byte chunk `cc` (0..7) of row `r` in a SWIZZLE_128B tile
// of 128-byte rows (the layout TMA writes and UMMA descriptors read).
__device__ __forceinline__ uint32_t sw128_off(int r, int cc) {
  return uint32_t((r >> 3) * 1024 + (r & 7) * 128 + ((cc ^ (r & 7)) << 4));
}

__global__ void __launch_bounds__(kThreads, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                    const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                    const __grid_constant__ CUtensorMap tm_dq, const BwdArgs args) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t sbase = (raw + 1023u) & ~1023u;
  if (sbase != raw) __trap();  // the layout above has no alignment slack
  uint8_t* sgen = smem_raw + (sbase - raw);
  const uint32_t bar0 = sbase + kSmemBar;
  auto bar = [&](int i) -> uint32_t { return bar0 + 8u * uint32_t(i); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sgen + kSmemBar + 8 * B_COUNT);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const zp_bwd_item it = args.items[blockIdx.x];
  ZP_CHECK(it.kv_len >= 1 && it.kv_len <= kBK && it.kv_row0 >= 0 && it.kv_row0 + it.kv_len <= args.kv_rows,
           "bwd item kv rows", it.kv_row0, it.kv_len);
  ZP_CHECK(it.kv_head >= 0 && it.kv_head < args.hkv, "bwd item kv head", it.kv_head, args.hkv);
#ifdef ZP_TRACE
  if (threadIdx.x == 0) ZP_BITEM(0, gtimer());
#endif
  const int kvh = it.kv_head;

  if (threadIdx.x == 0) {
    mbar_init(bar(B_KV), 1);
    for (int b = 0; b < kQStages; ++b) {
      mbar_init(bar(B_QDO_FULL + b), 1);
      mbar_init(bar(B_QDO_EMPTY + b), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar(B_SDP_FULL + b), 1);
      mbar_init(bar(B_PDS_FULL + b), 4);
      mbar_init(bar(B_PDS_EMPTY + b), 1);
      mbar_init(bar(B_DQ_FULL + b), 1);
      mbar_init(bar(B_DQ_EMPTY + b), 4);
    }
    mbar_init(bar(B_DKV), 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(smem_u32(tmem_slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS0 = tmem, tDP0 = tmem + 128, tDV = tmem + 256, tDK = tmem + 384;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- producer
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_do);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      const uint64_t pol_kv = policy_evict_first();
      const uint64_t pol_q = policy_evict_last();  // Q / dO blocks are re-read by other key tiles
      mbar_expect_tx(bar(B_KV), 2 * kKVTile);
      for (int b = 0; b < 2; ++b) {
        tma_load_2d(sbase + kSmemK + b * kKVBox, &tm_k, bar(B_KV), kvh * kD + b * 64, it.kv_row0, pol_kv);
        tma_load_2d(sbase + kSmemV + b * kKVBox, &tm_v, bar(B_KV), kvh * kD + b * 64, it.kv_row0, pol_kv);
      }
      StepCursor cur(args.qsegs, it.qseg_begin, it.qseg_count, it.kv_pos0, args.group);
      for (uint32_t n = 0; cur.next(); ++n) {
        const int qs = int(n % kQStages);
        if (n >= uint32_t(kQStages)) mbar_wait(bar(B_QDO_EMPTY + qs), ((n / kQStages) - 1) & 1);
        mbar_expect_tx(bar(B_QDO_FULL + qs), 2 * kQTile);
        const int h = kvh * args.group + cur.hh;
        ZP_CHECK(cur.g.row0 >= 0 && cur.g.row0 + cur.g.len <= args.q_rows && cur.g.row0 + cur.g.len <= args.lse_stride,
                 "bwd q segment", cur.g.row0, cur.g.len);
        for (int b = 0; b < 2; ++b) {
          tma_load_2d(sbase + kSmemQ + qs * kQTile + b * kQBox, &tm_q, bar(B_QDO_FULL + qs), h * kD + b * 64,
                      cur.row(), pol_q);
          tma_load_2d(sbase + kSmemDO + qs * kQTile + b * kQBox, &tm_do, bar(B_QDO_FULL + qs),
                      h * kD + b * 64, cur.row(), pol_q);
        }
      }
    }
  } else if (warp == 1) {
    {
      // ---------------- MMA issuer (whole warp, warp-uniform operands; one
      // elected lane issues each tcgen05 op)
      constexpr uint32_t idesc_t = idesc_bf16_f32(128, 64, 0, 0);    // S^T, dP^T
      constexpr uint32_t idesc_kv = idesc_bf16_f32(128, 128, 0, 1);  // dV, dK
      constexpr uint32_t idesc_q = idesc_bf16_f32(128, 64, 1, 1);    // dQ^T
      const uint64_t k_kmaj = umma_desc_sw128(sbase + kSmemK, 16, 1024);
      const uint64_t v_kmaj = umma_desc_sw128(sbase + kSmemV, 16, 1024);
      const uint64_t k_mn = umma_desc_sw128(sbase + kSmemK, kKVBox, 1024);
      const uint64_t q_kmaj = umma_desc_sw128(sbase + kSmemQ, 16, 1024);
      const uint64_t do_kmaj = umma_desc_sw128(sbase + kSmemDO, 16, 1024);
      const uint64_t q_mn = umma_desc_sw128(sbase + kSmemQ, kQBox, 1024);
      const uint64_t do_mn = umma_desc_sw128(sbase + kSmemDO, kQBox, 1024);
      const uint64_t dst_mn = umma_desc_sw128(sbase + kSmemDST, kPTile, 1024);
      constexpr uint64_t q_step = kQTile >> 4, p_step = kPTile >> 4;

      int n_steps = 0;
      {
        StepCursor cur(args.qsegs, it.qseg_begin, it.qseg_count, it.kv_pos0, args.group);
        while (cur.next()) ++n_steps;
      }
      // The step count comes from global loads, so ptxas cannot prove it
      // warp-uniform; REDUX returns it in a uniform register, which makes the
      // step loop uniform and lets every descriptor below live in uniform
      // registers (UIADD3.64 per MMA instead of an R2UR chain: the issue loop
      // was the backward's critical path, ~88 cycles per MMA).
      n_steps = int(__reduce_max_sync(0xffffffffu, unsigned(n_steps)));
      mbar_wait(bar(B_KV), 0);
      tc_fence_after();
#ifdef ZP_TRACE
      if (lane == 0) {
        ZP_BITEM(1, gtimer());
        ZP_BITEM(3, (unsigned long long)n_steps);
      }
#endif
      // dP^T(m): its buffer was released by dK(m-2), which precedes it in issue order
      auto issue_dp = [&](int m) {
        const int buf = m & 1, qs = m % kQStages;
        if (lane == 0 && m < 256) ZP_BSTAMP(3072 + m * 4 + 0);
        mbar_wait(bar(B_QDO_FULL + qs), (m / kQStages) & 1);
        if (lane == 0 && m < 256) ZP_BSTAMP(3072 + m * 4 + 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk) {
          const uint64_t ao = ((kk >> 2) * kKVBox + (kk & 3) * 32) >> 4;
          const uint64_t bo = ((kk >> 2) * kQBox + (kk & 3) * 32) >> 4;
          mma_ss_w(tDP0 + 64 * buf, v_kmaj + ao, do_kmaj + q_step * qs + bo, idesc_t, kk > 0 ? 1u : 0u);
        }
      };
      // S^T(m) once dQ^T(m-2) has drained from its columns, then SDP_FULL(m)
      auto issue_s = [&](int m) {
        const int buf = m & 1, qs = m % kQStages;
        if (m >= 2) mbar_wait(bar(B_DQ_EMPTY + buf), ((m >> 1) - 1) & 1);
        if (lane == 0 && m < 256) ZP_BSTAMP(3072 + m * 4 + 2);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk) {
          const uint64_t ao = ((kk >> 2) * kKVBox + (kk & 3) * 32) >> 4;
          const uint64_t bo = ((kk >> 2) * kQBox + (kk & 3) * 32) >> 4;
          mma_ss_w(tS0 + 64 * buf, k_kmaj + ao, q_kmaj + q_step * qs + bo, idesc_t, kk > 0 ? 1u : 0u);
        }
        tc_commit_w(bar(B_SDP_FULL + buf));
        if (lane == 0 && m < 256) ZP_BSTAMP(3072 + m * 4 + 3);
      };
      if (n_steps > 0) {
        issue_dp(0);
        issue_s(0);
      }
      for (int n = 0; n < n_steps; ++n) {
        if (n + 1 < n_steps) {
          issue_dp(n + 1);
          issue_s(n + 1);
        }
        const int buf = n & 1, qs = n % kQStages;
        mbar_wait(bar(B_PDS_FULL + buf), (n >> 1) & 1);
        tc_fence_after();
        if (lane == 0 && n < 256) ZP_BSTAMP(2048 + n * 4 + 0);
#pragma unroll
        for (int kk = 0; kk < kBQ / 16; ++kk) {
          const uint32_t acc = (n > 0 || kk > 0) ? 1u : 0u;
          // A = P^T / dS^T straight from TMEM (bf16x2, 8 columns per 16 queries)
          mma_ts_w(tDV, tS0 + 64 * buf + kk * 8, do_mn + q_step * qs + ((kk * 2048) >> 4), idesc_kv, acc);
          mma_ts_w(tDK, tDP0 + 64 * buf + kk * 8, q_mn + q_step * qs + ((kk * 2048) >> 4), idesc_kv, acc);
        }
        tc_commit_w(bar(B_QDO_EMPTY + qs));
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk)
          mma_ss_w(tS0 + 64 * buf, k_mn + ((kk * 2048) >> 4), dst_mn + p_step * buf + ((kk * 2048) >> 4), idesc_q,
                 kk > 0 ? 1u : 0u);
        tc_commit_w(bar(B_DQ_FULL + buf));
        tc_commit_w(bar(B_PDS_EMPTY + buf));
        if (lane == 0 && n < 256) ZP_BSTAMP(2048 + n * 4 + 1);
      }
      tc_commit_w(bar(B_DKV));
    }
  } else if (warp >= 4 && warp < 8) {
    // ---------------- P^T / dS^T (thread == key row), then the dK / dV epilogue
    const int quad = warp & 3;
    const int k = quad * 32 + lane;
    const uint32_t lane_bits = uint32_t(quad * 32) << 16;
    const bool kval = k < it.kv_len;
    const int kpos = it.kv_pos0 + k;
    const float c1 = args.scale_log2;
    // dS^T carries the softmax scale (dS' = scale * P * (dP - Delta)), so dK
    // and dQ leave their accumulators unscaled
    const float sc = args.scale;
    const uint32_t ld_base = sbase + kSmemLD + quad * 512;
    int n = 0;
    StepCursor cur(args.qsegs, it.qseg_begin, it.qseg_count, it.kv_pos0, args.group);
    // LSE / Delta of the NEXT step are loaded one step ahead (the global-load
    // latency used to sit on the critical path right after S^T landed)
    StepCursor ahead = cur;
    float nl[2], nd[2];
    auto fetch = [&](const StepCursor& c) {
      const int hh = kvh * args.group + c.hh;
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        const int j = lane + 32 * jj;
        const bool ok = j < c.valid();
        const size_t ix = size_t(hh) * args.lse_stride + c.row() + j;
        // invalid query rows: LSE = +inf makes P exactly 0
        nl[jj] = ok ? args.lse[ix] : INFINITY;  // scaled to log2 when stored: no use here
        nd[jj] = ok ? args.delta[ix] : 0.f;
      }
    };
    if (ahead.next()) fetch(ahead);
    for (; cur.next(); ++n) {
      const int buf = n & 1;
      const int qpos0 = cur.pos(), qv = cur.valid();
      // lane j loaded LSE / Delta of queries j and 32 + j of this step one step
      // ago; publish them to this warp's broadcast slots (its previous step has
      // finished reading them: program order), then start the next step's loads
      __syncwarp();
      st_shared_f32(ld_base + lane * 4, nl[0] * 1.4426950408889634f);
      st_shared_f32(ld_base + (32 + lane) * 4, nl[1] * 1.4426950408889634f);
      st_shared_f32(ld_base + 256 + lane * 4, nd[0] * sc);
      st_shared_f32(ld_base + 256 + (32 + lane) * 4, nd[1] * sc);
      __syncwarp();
      if (ahead.next()) fetch(ahead);
      const int tr = (lane == 0 && quad == 0 && n < 256) ? n * 4 : -1;
      ZP_BSTAMP(tr);
      mbar_wait(bar(B_SDP_FULL + buf), (n >> 1) & 1);
      tc_fence_after();
      ZP_BSTAMP(tr < 0 ? -1 : tr + 1);
      if (n >= 2) mbar_wait(bar(B_PDS_EMPTY + buf), ((n >> 1) - 1) & 1);
      ZP_BSTAMP(tr < 0 ? -1 : tr + 2);
      const bool full = kval && it.kv_len == kBK && qpos0 >= it.kv_pos0 + kBK - 1;
      const uint32_t dst_row = sbase + kSmemDST + buf * kPTile;
      // Full steps (every query of the step sees every key of the item: the
      // common case away from the diagonal) run a mask-free copy of the loop.
      auto p_ds = [&](auto kFull) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t sr[32], dr[32];
          tmem_ld32(tS0 + lane_bits + 64 * buf + 32 * c, sr);
          tmem_ld32(tDP0 + lane_bits + 64 * buf + 32 * c, dr);
          tmem_wait_ld();
          uint32_t pk[16], dk[16];
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            float lv[4], dv[4];
            ld_shared_v4f(ld_base + (32 * c + j) * 4, lv);
            ld_shared_v4f(ld_base + 256 + (32 * c + j) * 4, dv);
            float p[4], ds[4];
            if constexpr (decltype(kFull)::value) {  // every (query, key) visible: no mask
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                p[u] = ex2(__uint_as_float(sr[j + u]) * c1 - lv[u]);
                ds[u] = p[u] * (__uint_as_float(dr[j + u]) * sc - dv[u]);
              }
            } else {
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int q = 32 * c + j + u;
                float e = ex2(__uint_as_float(sr[j + u]) * c1 - lv[u]);
                if (!(kval && qpos0 + q >= kpos)) e = 0.f;
                p[u] = e;
                ds[u] = e * (__uint_as_float(dr[j + u]) * sc - dv[u]);
              }
            }
            pk[j / 2] = pack_bf16(p[0], p[1]);
            pk[j / 2 + 1] = pack_bf16(p[2], p[3]);
            dk[j / 2] = pack_bf16(ds[0], ds[1]);
            dk[j / 2 + 1] = pack_bf16(ds[2], ds[3]);
          }
          // P^T / dS^T (bf16x2) over the S^T / dP^T columns this chunk has already
          // read (chunk c covers columns [32c, 32c+32) and writes [16c, 16c+16));
          // they are the TMEM A operands of dV += P^T dO and dK += dS^T Q.
          tmem_st16(tS0 + lane_bits + 64 * buf + 16 * c, pk);
          tmem_st16(tDP0 + lane_bits + 64 * buf + 16 * c, dk);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            st_shared_v4(dst_row + sw128_off(k, 4 * c + i), dk[4 * i], dk[4 * i + 1], dk[4 * i + 2], dk[4 * i + 3]);
        }
      };
      if (full) p_ds(BoolC<true>{});
      else p_ds(BoolC<false>{});
      fence_proxy_async_smem();  // generic-proxy smem writes -> tcgen05.mma operands
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(B_PDS_FULL + buf));
      ZP_BSTAMP(tr < 0 ? -1 : tr + 3);
    }
    // ---------------- dK / dV of this key tile (fp32, accumulated if asked)
    mbar_wait(bar(B_DKV), 0);
    tc_fence_after();
    {
      const size_t row = (size_t(it.kv_row0) + (kval ? k : 0)) * args.hkv + kvh;
      const bool accum = (it.flags & ZP_BWD_ACCUMULATE) != 0;
#pragma unroll 1
      for (int which = 0; which < 2; ++which) {
        float4* dst = reinterpret_cast<float4*>((which ? args.dk : args.dv) + row * kD);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t rr[32];
          tmem_ld32((which ? tDK : tDV) + lane_bits + 32 * c, rr);  // collective: every lane loads
          tmem_wait_ld();
          if (!kval) continue;
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            float4 x = n > 0 ? make_float4(__uint_as_float(rr[4 * v]), __uint_as_float(rr[4 * v + 1]),
                                           __uint_as_float(rr[4 * v + 2]), __uint_as_float(rr[4 * v + 3]))
                             : make_float4(0.f, 0.f, 0.f, 0.f);
            if (accum) {
              const float4 y = dst[8 * c + v];
              x.x += y.x;
              x.y += y.y;
              x.z += y.z;
              x.w += y.w;
            }
            dst[8 * c + v] = x;
          }
        }
      }
    }
  } else if (warp >= 8) {
    // ---------------- dQ reduction (thread == head dim): the dQ^T tile goes
    // through a shared-memory staging tile ([64 queries][128 dims] as four
    // 32-dim boxes) and leaves with four TMA reduce-adds (atomic in L2).
    // Query rows past the segment end carry exact zeros (P = dS = 0 there).
    const int quad = warp & 3;
    const uint32_t lane_bits = uint32_t(quad * 32) << 16;
    const uint32_t box = sbase + kSmemDQ + quad * kDQBox;
    // Each warp owns one 32-dim box and issues its own reduce: a box waits
    // only for its own previous reduce, with no 128-thread barrier (one issuer
    // for all four boxes measured 6% slower on 64K).
    StepCursor cur(args.qsegs, it.qseg_begin, it.qseg_count, it.kv_pos0, args.group);
    for (int n = 0; cur.next(); ++n) {
      const int buf = n & 1;
      const int h = kvh * args.group + cur.hh;
      mbar_wait(bar(B_DQ_FULL + buf), (n >> 1) & 1);
      tc_fence_after();
      if (lane == 0 && quad == 0 && n < 256) ZP_BSTAMP(1024 + n * 4);
      uint32_t r0[32], r1[32];
      tmem_ld32(tS0 + lane_bits + 64 * buf, r0);
      tmem_ld32(tS0 + lane_bits + 64 * buf + 32, r1);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(B_DQ_EMPTY + buf));
      if (lane == 0) bulk_wait_read0();  // this warp's previous reduce has read its box
      __syncwarp();
      if (lane == 0 && quad == 0 && n < 256) ZP_BSTAMP(1024 + n * 4 + 2);
#pragma unroll
      for (int j = 0; j < 32; ++j) st_shared_f32(box + lane * 4 + j * 128, __uint_as_float(r0[j]));
#pragma unroll
      for (int j = 0; j < 32; ++j) st_shared_f32(box + lane * 4 + (32 + j) * 128, __uint_as_float(r1[j]));
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_reduce_add_2d(&tm_dq, box, h * kD + 32 * quad, cur.row());
        bulk_commit();
      }
      if (lane == 0 && quad == 0 && n < 256) ZP_BSTAMP(1024 + n * 4 + 1);
    }
    if (lane == 0) bulk_wait0();
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
#ifdef ZP_TRACE
  if (threadIdx.x == 0) ZP_BITEM(2, gtimer());
#endif
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// Delta[h][row] = sum_d dO[row,h,d] * O[row,h,d] (fp32), one warp per (row, head).
__global__ void bwd_delta_kernel(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
                                 float* __restrict__ delta, int rows, int hq, int stride) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= rows * hq) return;
  const int row = w / hq, h = w % hq;
  const size_t base = (size_t(row) * hq + h) * kD + lane * 4;
  const uint2 a = *reinterpret_cast<const uint2*>(o + base);
  const uint2 b = *reinterpret_cast<const uint2*>(dout + base);
  const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
  const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b);
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float2 x = __bfloat1622float2(a2[i]), y = __bfloat1622float2(b2[i]);
    s += x.x * y.x + x.y * y.y;
  }
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
  if (lane == 0) delta[size_t(h) * stride + row] = s;
}

}  // namespace bwd
}  // namespace zp

// ------------------------------------------------------------------ host side
#include "zp_host.h"

#ifdef ZP_TRACE
extern "C" ZP_API int zp_debug_bitems(unsigned long long* host, int n) {
  return cudaMemcpyFromSymbol(host, zp::bwd::g_zp_bitems, sizeof(unsigned long long) * (n < 65536 ? n : 65536)) ==
                 cudaSuccess ? 0 : -1;
}
extern "C" ZP_API int zp_debug_btrace(unsigned long long* host, int n) {
  return cudaMemcpyFromSymbol(host, zp::bwd::g_zp_btrace, sizeof(unsigned long long) * (n < 4096 ? n : 4096)) ==
                 cudaSuccess ? 0 : -1;
}
#endif

extern "C" int zp_attn_bwd_prep(const void* o, const void* dout, int rows, int hq, int head_dim, float* delta,
                                int delta_stride, void* stream) {
  using namespace zp::bwd;
  if (head_dim != kD) return zp_fail(ZP_EINVAL, "zp_attn_bwd_prep: head_dim must be 128");
  if (rows < 0 || hq <= 0 || delta_stride < rows) return zp_fail(ZP_EINVAL, "zp_attn_bwd_prep: bad sizes");
  if (rows == 0) return ZP_OK;
  if (!o || !dout || !delta) return zp_fail(ZP_EINVAL, "zp_attn_bwd_prep: null pointer");
  if (zp_check_device() != ZP_OK) return ZP_ENODEV;
  const long long warps = (long long)rows * hq;
  const int blocks = int((warps * 32 + 255) / 256);
  bwd_delta_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const __nv_bfloat16*>(o), reinterpret_cast<const __nv_bfloat16*>(dout), delta, rows, hq,
      delta_stride);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return zp_fail_cuda(e, "zp_attn_bwd_prep: launch");
  return ZP_OK;
}

extern "C" int zp_attn_bwd(const void* q, const void* k, const void* v, const void* dout, int q_rows, int kv_rows,
                           int kv_row_stride, int hq, int hkv, int head_dim, const float* lse, const float* delta,
                           int lse_stride, float* dq, float* dk, float* dv, const zp_bwd_item* items, int n_items,
                           const zp_kv_seg* qsegs, float softmax_scale, void* stream) {
  using namespace zp::bwd;
  if (head_dim != kD) return zp_fail(ZP_EINVAL, "zp_attn_bwd: head_dim must be 128");
  if (hq <= 0 || hkv <= 0 || hq % hkv != 0) return zp_fail(ZP_EINVAL, "zp_attn_bwd: need hq % hkv == 0");
  if (n_items < 0 || q_rows < 0 || kv_rows < 0 || kv_row_stride < hkv * kD)
    return zp_fail(ZP_EINVAL, "zp_attn_bwd: bad sizes");
  if (n_items == 0) return ZP_OK;
  if (q_rows == 0 || kv_rows == 0) return zp_fail(ZP_EINVAL, "zp_attn_bwd: empty q or kv with items");
  if (!q || !k || !v || !dout || !lse || !delta || !dq || !dk || !dv || !items || !qsegs)
    return zp_fail(ZP_EINVAL, "zp_attn_bwd: null pointer");
  if (zp_check_device() != ZP_OK) return ZP_ENODEV;

  CUtensorMap tq, tdo, tk, tv, tdq;
  int rc;
  if ((rc = zp_make_tmap_2d_bf16(&tq, q, uint64_t(hq) * kD, uint64_t(q_rows), uint64_t(hq) * kD * 2, 64, kBQ)) !=
      ZP_OK)
    return rc;
  if ((rc = zp_make_tmap_2d_bf16(&tdo, dout, uint64_t(hq) * kD, uint64_t(q_rows), uint64_t(hq) * kD * 2, 64,
                                 kBQ)) != ZP_OK)
    return rc;
  if ((rc = zp_make_tmap_2d_bf16(&tk, k, uint64_t(hkv) * kD, uint64_t(kv_rows), uint64_t(kv_row_stride) * 2, 64,
                                 kBK)) != ZP_OK)
    return rc;
  if ((rc = zp_make_tmap_2d_bf16(&tv, v, uint64_t(hkv) * kD, uint64_t(kv_rows), uint64_t(kv_row_stride) * 2, 64,
                                 kBK)) != ZP_OK)
    return rc;
  if ((rc = zp_make_tmap_2d_f32(&tdq, dq, uint64_t(hq) * kD, uint64_t(q_rows), uint64_t(hq) * kD * 4, 32, kBQ)) !=
      ZP_OK)
    return rc;
  static bool attr_done[64] = {};  // per device: the attribute is per device and function
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return zp_fail(ZP_ENODEV, "zp_attn_bwd: device");
  if (!attr_done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(kSmemBytes));
    if (e != cudaSuccess) return zp_fail_cuda(e, "zp_attn_bwd: smem attribute");
    attr_done[dev] = true;
  }
  BwdArgs a;
  a.items = items;
  a.qsegs = qsegs;
  a.lse = lse;
  a.delta = delta;
  a.lse_stride = lse_stride;
  a.dq = dq;
  a.dk = dk;
  a.dv = dv;
  a.hq = hq;
  a.hkv = hkv;
  a.group = hq / hkv;
  a.q_rows = q_rows;
  a.kv_rows = kv_rows;
  a.scale = softmax_scale;
  a.scale_log2 = softmax_scale * 1.4426950408889634f;
  attn_bwd_kernel<<<n_items, kThreads, kSmemBytes, reinterpret_cast<cudaStream_t>(stream)>>>(tq, tdo, tk, tv, tdq,
                                                                                              a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return zp_fail_cuda(e, "zp_attn_bwd: launch");
  return ZP_OK;
}
