// Causal varlen / ring-round flash attention forward for sm_100a.
//
// Executes what the reference only counts: for every query row q and every
// key k of the same sequence with global position k <= q
// (attention_engine.py:113-136, visible_pairs), O = softmax(q.K^T/sqrt(d)) V.
// LocalTask work (attention_engine.py:260-265) is one launch over all local
// fragments; each RingRound (attention_engine.py:229-244) is one launch against
// the KV set held by the ring position (i-r) mod g, resuming the running
// softmax state of the previous round (exact online-softmax continuation).
//
// Work item = 128 query rows x 2 query heads of one GQA group.  Two variants of
// one kernel template:
//
//   single (kPair=false): one CTA per item, M=128 tcgen05.mma (cta_group::1).
//   pair   (kPair=true):  a cluster of 2 CTAs on one TPC runs items 2p and 2p+1
//       (heads 4g..4g+3 of one KV head) as M=256 tcgen05.mma.cta_group::2: each
//       CTA holds its own Q rows, HALF of every K tile (64 keys) and HALF of
//       every V tile (64 dims); the leader CTA issues all MMAs for the pair and
//       each CTA's TMEM receives its own 128 rows.  Per SM this halves the
//       shared-memory operand traffic of B (K, V) and the K/V bytes fetched,
//       which is what bounds the single-CTA M=128 pipeline.
//
// Roles inside a CTA (384 threads):
//   warp 0      TMA producer (Q, then K/V tiles through smem rings); in the
//               pair the leader's producer also claims work items
//   warp 1      TMEM allocator + tcgen05.mma issuer (single thread; leader only)
//   warps 2-3   idle (keep warpgroup 0 whole for setmaxnreg)
//   warps 4-7   softmax / rescale / epilogue for head tile 0 (thread == row)
//   warps 8-11  softmax / rescale / epilogue for head tile 1 (thread == row)
// A warp may only touch TMEM lanes 32*(warp%4)..+31.  Warpgroup 0 gives its
// registers to the two softmax warpgroups (setmaxnreg), which hold a whole
// 128-column S row per thread.
// TMEM (512 columns): S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512);
// P_t (bf16x2 packed, 64 columns) aliases S_t columns [64,128) and feeds the
// PV product as the TMEM A operand.  Shared memory: Q0,Q1 (2x32 KB) and the
// K and V rings, all SWIZZLE_128B as written by TMA.
#include <cstdlib>

#include "zp_ptx.cuh"
#include "../../include/zeppelin_b200.h"

namespace zp {

constexpr int kHeadDim = 128;
constexpr int kBM = 128;  // query rows per CTA tile
constexpr int kBN = 128;  // key rows per tile
constexpr int kThreads = 384;
constexpr uint32_t kTileBytes = kBM * kHeadDim * 2;   // 32 KB
constexpr uint32_t kBoxBytes = 128 * 64 * 2;          // 16 KB (one 64-column x 128-row TMA box)
constexpr int kSchedSlots = 4;
#ifndef ZP_MMA_UNROLL
#define ZP_MMA_UNROLL 8
#endif
#ifndef ZP_WG0_REGS
#define ZP_WG0_REGS 88  // producer / MMA warpgroup
#endif
#ifndef ZP_SM_REGS
#define ZP_SM_REGS 208  // each softmax warpgroup (thread = one 128-column S row)
#endif
constexpr int kMmaUnroll = ZP_MMA_UNROLL;

// Diagnostic build only (-DZP_TRACE): SM clock stamps of CTA 0's softmax
// stages and MMA issue points, read back with zp_debug_trace().
#ifdef ZP_TRACE
__device__ unsigned long long g_zp_trace[8192];  // CTA 0 at [0, 4096), CTA 1 at [4096, 8192)
#define ZP_STAMP(slot)                                                              \
  do {                                                                              \
    if (blockIdx.x < 2 && (slot) >= 0 && (slot) < 4096) {                           \
      unsigned long long c_;                                                        \
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(c_)::"memory");                  \
      g_zp_trace[blockIdx.x * 4096 + (slot)] = c_;                                  \
    }                                                                               \
  } while (0)
#else
#define ZP_STAMP(slot) \
  do {                 \
  } while (0)
#endif
static_assert(ZP_WG0_REGS * 128 + ZP_SM_REGS * 256 <= 168 * 384, "setmaxnreg exceeds the launch register pool");

template <bool kPair>
struct Cfg {
  static constexpr int kKStages = kPair ? 4 : 2;
  static constexpr int kVStages = kPair ? 4 : 2;
  // bytes of one K / V ring stage in THIS CTA (the pair splits each tile)
  static constexpr uint32_t kKBytes = kPair ? kTileBytes / 2 : kTileBytes;
  static constexpr uint32_t kVBytes = kPair ? kTileBytes / 2 : kTileBytes;
  static constexpr uint32_t kKRows = kPair ? kBN / 2 : kBN;  // key rows of K per CTA
  static constexpr uint32_t kKBox = kKRows * 128;            // one 64-column K box
  static constexpr uint32_t kSmemQ = 0;
  static constexpr uint32_t kSmemK = 2 * kTileBytes;
  static constexpr uint32_t kSmemV = kSmemK + kKStages * kKBytes;
  static constexpr uint32_t kSmemBar = kSmemV + kVStages * kVBytes;
  static constexpr uint32_t kSmemSched = kSmemBar + 512;            // schedule ring: kSchedSlots x SchedSlot
  static constexpr uint32_t kSmemBytes = kSmemSched + 256 + 1024;  // + alignment slack
  static constexpr uint32_t kPFullCount = kPair ? 8 : 4;          // one arrival per softmax warp (x CTAs)
  static constexpr uint32_t kSchedConsumers = kPair ? 18 : 9;
};

// barrier slots (ring stages <= 4)
enum : int {
  B_QFULL = 0,
  B_KFULL = 1,          // +stage
  B_KEMPTY = 5,         // +stage
  B_VFULL = 9,          // +stage
  B_VEMPTY = 13,        // +stage
  B_SFULL = 17,         // +tile
  B_PFULL = 19,         // +2*tile+half: P columns of keys [0,64) / [64,128) stored
  B_ODONE = 23,         // +tile
  B_QEMPTY = 25,
  B_SCHED_FULL = 26,    // +slot (4): item index published by the producer
  B_SCHED_EMPTY = 30,   // +slot (4): consumed by the MMA issuer and the softmax warps
  B_QFULL1 = 34,        // head tile 1's Q (B_QFULL / B_QEMPTY: head tile 0), so each head's
  B_QEMPTY1 = 35,       // next Q streams in as soon as that head's last QK^T is done
  B_COUNT = 36
};
static_assert(Cfg<true>::kKStages <= 4 && Cfg<true>::kVStages <= 4, "ring depth <= 4");
static_assert(Cfg<true>::kSmemBytes <= 232448 && Cfg<false>::kSmemBytes <= 232448, "smem budget");

struct AttnArgs {
  const zp_attn_item* items;
  int n_units;     // items (single) or item pairs (pair)
  int* next_unit;  // global work counter (zeroed before the launch)
  const zp_kv_seg* segs;
  void* o;  // bf16 [rows, hq, 128]; fp32 in the parity mode
  float* lse;
  float* st_o;
  float* st_ml;
  int lse_stride;
  int state_rows;
  int hq;
  int group;  // hq / hkv
  float scale_log2;
  int q_rows;   // bounds of q / o and k / v (checked in -DZP_CHECKS builds)
  int kv_rows;
};

// Walks the KV tiles an item needs, in order: tiles of each segment up to the
// item's last visible key (causal pruning; fully-masked tiles never issued).
struct TileCursor {
  const zp_kv_seg* segs;
  int s, first, end, max_qpos, ti, nt;
  zp_kv_seg g, g0;  // g0: segs[first], handed over through the schedule ring
  __device__ __forceinline__ TileCursor(const zp_kv_seg* sg, int b, int c, int mq)
      : segs(sg), s(b - 1), first(-1), end(b + c), max_qpos(mq), ti(0), nt(0) {}
  __device__ __forceinline__ TileCursor(const zp_kv_seg* sg, int b, int c, int mq, const zp_kv_seg& seg0)
      : segs(sg), s(b - 1), first(b), end(b + c), max_qpos(mq), ti(0), nt(0), g0(seg0) {}
  __device__ __forceinline__ bool next() {
    if (++ti < nt) return true;
    while (++s < end) {
      g = s == first ? g0 : segs[s];
      if (g.len > 0 && g.pos0 <= max_qpos) {
        nt = (min(g.len, max_qpos - g.pos0 + 1) + kBN - 1) / kBN;
        ti = 0;
        return true;
      }
    }
    return false;
  }
  __device__ __forceinline__ int row() const { return g.row0 + ti * kBN; }
  __device__ __forceinline__ int pos() const { return g.pos0 + ti * kBN; }
  __device__ __forceinline__ int valid() const { return min(kBN, g.len - ti * kBN); }
};

#ifndef ZP_RESCALE_LOG2
#define ZP_RESCALE_LOG2 8.0f
#endif
constexpr float kRescaleLog2 = ZP_RESCALE_LOG2;  // lazy-rescale threshold (log2 units)
#ifndef ZP_SPEC_EXP
#define ZP_SPEC_EXP 1
#endif
constexpr bool kSpecExp = ZP_SPEC_EXP != 0;  // speculative exps with the running max

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

#ifndef ZP_EMU_OF8
#define ZP_EMU_OF8 2
#endif
constexpr int kEmuOf8 = ZP_EMU_OF8;  // column pairs per 8 whose exp2 runs on the FMA pipe

// 2^x for a pair on the FMA pipe: round-to-nearest split x = j + f (magic
// constant 1.5*2^23), degree-3 minimax polynomial for 2^f on [-1/2, 1/2]
// (max rel. error 7.5e-5, far below bf16's 3.9e-3), exponent add for 2^j.
// x is clamped at -125 so the exponent add never underflows (2^-125 ~ 0);
// used on unmasked tiles only (masked keys need an exact 0).
__device__ __forceinline__ float2 exp2_poly(float2 x) {
  x.x = fmaxf(x.x, -125.f);
  x.y = fmaxf(x.y, -125.f);
  const float2 y = __fadd2_rn(x, make_float2(12582912.f, 12582912.f));
  const float2 j = __fadd2_rn(y, make_float2(-12582912.f, -12582912.f));
  const float2 f = __ffma2_rn(j, make_float2(-1.f, -1.f), x);
  float2 p = __ffma2_rn(make_float2(0.055171608583694395f, 0.055171608583694395f), f,
                        make_float2(0.2426111175727868f, 0.2426111175727868f));
  p = __ffma2_rn(p, f, make_float2(0.6932609966238247f, 0.6932609966238247f));
  p = __ffma2_rn(p, f, make_float2(0.9999280741082696f, 0.9999280741082696f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(y.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(y.y) << 23)));
}

// P = 2^(s*scale_log2 - m) for one half (64 keys) of a 128-column row,
// packed to bf16x2 and stored to the half's 32 P columns in TMEM; row sum
// accumulated in two float2.  kEmu: a fixed share of the column pairs takes
// the FMA-pipe exp2 (relieves the MUFU pipe, 16 ex2/clk/SM).
template <int kHalf, bool kEmu, bool kF16>
__device__ __forceinline__ void exp_half(const float (&s)[128], float2 sl2x2, float2 negm, uint32_t tP,
                                         float2& acc0, float2& acc1) {
#pragma unroll
  for (int c = 2 * kHalf; c < 2 * kHalf + 2; ++c) {
    uint32_t pk[16];
#pragma unroll
    for (int v = 0; v < 16; ++v) {
      const float2 x = __ffma2_rn(make_float2(s[c * 32 + 2 * v], s[c * 32 + 2 * v + 1]), sl2x2, negm);
      float2 p;
      if (kEmu && ((c * 16 + v) & 7) < kEmuOf8) {
        p = exp2_poly(x);
      } else {
        p.x = ex2(x.x);
        p.y = ex2(x.y);
      }
      if (v & 1) acc1 = __fadd2_rn(acc1, p); else acc0 = __fadd2_rn(acc0, p);
      pk[v] = pack_p<kF16>(p.x, p.y);
    }
    tmem_st16(tP + c * 16, pk);
  }
}

// Issued by the whole MMA warp (warp-uniform operands), one elected lane.
template <bool kPair>
__device__ __forceinline__ void commit(uint32_t bar) {
  if constexpr (kPair) tc_commit_pair_w(bar, 0x3);
  else tc_commit_w(bar);
}

// Descriptor start addresses are in 16-byte units in the low 14 bits, so a
// byte offset inside shared memory is added to a base descriptor as off>>4.
// K tile (this CTA's rows) is K-major: 16 dims per MMA, the two 64-dim halves
// are one K box apart.
template <bool kPair>
__device__ __forceinline__ void issue_qk(uint32_t d_tmem, uint64_t q_desc, uint64_t k_desc,
                                         uint32_t idesc) {
#pragma unroll kMmaUnroll
  for (int kk = 0; kk < kHeadDim / 16; ++kk) {
    const uint64_t qoff = ((kk >> 2) * kBoxBytes + (kk & 3) * 32) >> 4;
    const uint64_t koff = ((kk >> 2) * Cfg<kPair>::kKBox + (kk & 3) * 32) >> 4;
    if constexpr (kPair) mma_ss_pair_w(d_tmem, q_desc + qoff, k_desc + koff, idesc, kk > 0 ? 1u : 0u);
    else mma_ss_w(d_tmem, q_desc + qoff, k_desc + koff, idesc, kk > 0 ? 1u : 0u);
  }
}

// V tile is [128 keys x dims], dims contiguous: MN-major B operand.  16 keys
// per MMA = 2 groups of 8 rows (SBO 1 KB); in the single kernel the two 64-dim
// swizzle atoms are one TMA box apart (LBO 16 KB), in the pair each CTA holds
// one 64-dim atom.  P (A operand) is 8 TMEM columns per 16 keys.
template <bool kPair>
__device__ __forceinline__ void issue_pv(uint32_t d_tmem, uint32_t p_tmem, uint64_t v_desc,
                                         uint32_t idesc, bool accumulate, int half) {
#pragma unroll
  for (int kk = 4 * half; kk < 4 * half + 4; ++kk) {
    const uint32_t acc = (accumulate || kk > 0) ? 1u : 0u;
    if constexpr (kPair) mma_ts_pair_w(d_tmem, p_tmem + kk * 8, v_desc + uint64_t(kk * (2048 >> 4)), idesc, acc);
    else mma_ts_w(d_tmem, p_tmem + kk * 8, v_desc + uint64_t(kk * (2048 >> 4)), idesc, acc);
  }
}

// One published work unit of the schedule ring: the claimed index plus what
// every consumer needs to start it without global loads (this CTA's item, its
// tile count, its first KV segment).
struct SchedSlot {
  int idx, n_tiles, pad0, pad1;
  zp_attn_item item;
  zp_kv_seg seg0;
};
static_assert(sizeof(SchedSlot) == 64, "schedule slot layout");

__device__ __forceinline__ int count_tiles(const zp_kv_seg* segs, const zp_attn_item& it) {
  int n = 0;
  TileCursor cur(segs, it.seg_begin, it.seg_count, it.q_pos0 + it.q_len - 1);
  while (cur.next()) ++n;
  return n;
}

// Persistent, dynamically scheduled CTAs (CTA pairs): the producer thread (the
// leader's, in a pair) claims the next unit of the longest-first list with one
// atomicAdd (greedy LPT across SMs) and publishes it to every consumer through
// a 4-slot smem ring (both CTAs' rings in a pair).
template <bool kPair, bool kParity>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q,
                    const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const AttnArgs args) {
  using C = Cfg<kPair>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t sbase = (raw + 1023u) & ~1023u;
  uint8_t* sgen = smem_raw + (sbase - raw);
  const uint32_t bar0 = sbase + C::kSmemBar;
  auto bar = [&](int i) -> uint32_t { return bar0 + 8u * uint32_t(i); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sgen + C::kSmemBar + 8 * B_COUNT);
  SchedSlot* ring = reinterpret_cast<SchedSlot*>(sgen + C::kSmemSched);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_units = args.n_units;
  const uint32_t cta = kPair ? cluster_ctarank() : 0u;
  // barrier of the MMA-issuing (leader) CTA, as a shared::cluster address
  auto lead = [&](int i) -> uint32_t { return kPair ? mapa_shared(bar(i), 0) : bar(i); };

  if (threadIdx.x == 0) {
    mbar_init(bar(B_QFULL), 1);
    mbar_init(bar(B_QEMPTY), 1);
    mbar_init(bar(B_QFULL1), 1);
    mbar_init(bar(B_QEMPTY1), 1);
    for (int k = 0; k < kSchedSlots; ++k) {
      mbar_init(bar(B_SCHED_FULL + k), 1);
      mbar_init(bar(B_SCHED_EMPTY + k), C::kSchedConsumers);
    }
    for (int s = 0; s < C::kKStages; ++s) {
      mbar_init(bar(B_KFULL + s), 1);
      mbar_init(bar(B_KEMPTY + s), 1);
    }
    for (int s = 0; s < C::kVStages; ++s) {
      mbar_init(bar(B_VFULL + s), 1);
      mbar_init(bar(B_VEMPTY + s), 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(bar(B_SFULL + s), 1);
      mbar_init(bar(B_PFULL + 2 * s), C::kPFullCount);
      mbar_init(bar(B_PFULL + 2 * s + 1), C::kPFullCount);
      mbar_init(bar(B_ODONE + s), 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    if constexpr (kPair) tmem_alloc_pair(smem_u32(tmem_slot), 512);
    else tmem_alloc(smem_u32(tmem_slot), 512);
  }
  tc_fence_before();
  if constexpr (kPair) cluster_sync_all();  // peer barriers initialised before any remote arrive
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) ZP_STAMP(4095);  // cluster-sync release: aligns the two CTAs' clocks

  // Next work unit for a consumer: wait for the slot, then release it to the
  // publishing producer (leader's ring in a pair).
  auto sched_wait = [&](uint32_t k) -> SchedSlot {
    const uint32_t slot = k % kSchedSlots;
    // the peer CTA's ring is written remotely by the leader: cluster-scope acquire
    if (kPair && cta != 0) mbar_wait_cluster(bar(B_SCHED_FULL + slot), (k / kSchedSlots) & 1);
    else mbar_wait(bar(B_SCHED_FULL + slot), (k / kSchedSlots) & 1);
    return ring[slot];
  };
  // The slot was copied to registers before this arrive (release.cta: the
  // cluster-scope release of the P hand-off cost ~1,000 cycles per arrive).
  auto sched_release = [&](uint32_t k) {
    const uint32_t slot = k % kSchedSlots;
    if constexpr (kPair) mbar_arrive_remote(lead(B_SCHED_EMPTY + slot));
    else mbar_arrive(bar(B_SCHED_EMPTY + slot));
  };

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(ZP_WG0_REGS));
    if (warp == 0 && lane == 0) {
      // ---------------- producer: per item Q (2 heads), then K_j / V_j rings
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_last();
      uint32_t jg = 0, qn = 0;
      for (uint32_t k = 0;; ++k) {
        SchedSlot u;
        if (cta == 0) {
          const uint32_t slot = k % kSchedSlots;
          if (k >= kSchedSlots) {
            if constexpr (kPair) mbar_wait_cluster(bar(B_SCHED_EMPTY + slot), ((k / kSchedSlots) - 1) & 1);
            else mbar_wait(bar(B_SCHED_EMPTY + slot), ((k / kSchedSlots) - 1) & 1);
          }
          u.idx = atomicAdd(args.next_unit, 1);
          u.n_tiles = 0;
          u.pad0 = u.pad1 = 0;
          zp_attn_item o{};
          if (u.idx < n_units) {
            u.item = args.items[kPair ? 2 * u.idx : u.idx];
            if constexpr (kPair) {
              // contract: items 2p / 2p+1 are the same tile for head pairs 2g / 2g+1
              o = args.items[2 * u.idx + 1];
              const zp_attn_item& it = u.item;
              if (o.q_row0 != it.q_row0 || o.q_pos0 != it.q_pos0 || o.q_len != it.q_len ||
                  o.seg_begin != it.seg_begin || o.seg_count != it.seg_count || o.state_row0 != it.state_row0 ||
                  o.flags != it.flags || it.head_pair != (o.head_pair ^ 1) || (it.head_pair & 1) != 0)
                __trap();
            }
            u.n_tiles = count_tiles(args.segs, u.item);
            if (u.item.seg_count > 0) u.seg0 = args.segs[u.item.seg_begin];
          }
          ring[slot] = u;
          if constexpr (kPair) {
            // the peer CTA's slot: same unit, its own item (head pair 2g+1)
            const int4* w = reinterpret_cast<const int4*>(&u);
            const int4* wo = reinterpret_cast<const int4*>(&o);
            const uint32_t peer = mapa_shared(smem_u32(ring + slot), 1);
            st_cluster_v4(peer, w[0]);
            st_cluster_v4(peer + 16, wo[0]);
            st_cluster_v4(peer + 32, wo[1]);
            st_cluster_v4(peer + 48, w[3]);
            mbar_arrive_cluster(mapa_shared(bar(B_SCHED_FULL + slot), 1));
          }
          mbar_arrive(bar(B_SCHED_FULL + slot));
        } else {
          u = sched_wait(k);
          sched_release(k);
        }
        if (u.idx >= n_units) break;
        const zp_attn_item it = u.item;
        if (u.n_tiles == 0) continue;
        ZP_CHECK(it.q_len >= 1 && it.q_len <= kBM && it.q_row0 >= 0 && it.q_row0 + it.q_len <= args.q_rows,
                 "fwd item q rows", it.q_row0, it.q_len);
        ZP_CHECK(it.q_row0 + it.q_len <= args.lse_stride, "fwd item lse row", it.q_row0 + it.q_len, args.lse_stride);
        ZP_CHECK(2 * it.head_pair + 1 < args.hq, "fwd item head pair", it.head_pair, args.hq);
        ZP_CHECK(!(it.flags & (ZP_ITEM_LOAD_STATE | ZP_ITEM_STORE_STATE)) ||
                     (args.st_o != nullptr && it.state_row0 >= 0 && it.state_row0 + it.q_len <= args.state_rows),
                 "fwd item state rows", it.state_row0, args.state_rows);
        const int kvh = (2 * it.head_pair) / args.group;
        // Q of head tile t, once that head's last QK^T of the previous item is done
        auto load_q = [&](int t) {
          const int qf = t ? B_QFULL1 : B_QFULL;
          if (qn > 0) mbar_wait(bar(t ? B_QEMPTY1 : B_QEMPTY), (qn - 1) & 1);
          if (cta == 0) mbar_expect_tx(bar(qf), (kPair ? 2 : 1) * kTileBytes);
          for (int b = 0; b < 2; ++b) {
            const uint32_t dst = sbase + C::kSmemQ + t * kTileBytes + b * kBoxBytes;
            const int x = (2 * it.head_pair + t) * kHeadDim + b * 64;
            if constexpr (kPair) tma_load_2d_pair(dst, &tm_q, lead(qf), x, it.q_row0, pol_q);
            else tma_load_2d(dst, &tm_q, bar(qf), x, it.q_row0, pol_q);
          }
        };
        load_q(0);
        TileCursor cur(args.segs, it.seg_begin, it.seg_count, it.q_pos0 + it.q_len - 1, u.seg0);
        for (int jj = 0; cur.next(); ++jg, ++jj) {
          if (jj == 1) load_q(1);  // after the first K/V tile: head 1's Q is needed later
          const int kst = int(jg % C::kKStages), vst = int(jg % C::kVStages);
          const uint32_t ku = jg / C::kKStages, vu = jg / C::kVStages;
          const int row = cur.row();
          ZP_CHECK(cur.g.row0 >= 0 && cur.g.len >= 0 && cur.g.row0 + cur.g.len <= args.kv_rows, "fwd kv segment",
                   cur.g.row0, cur.g.len);
          if (jg >= uint32_t(C::kKStages)) mbar_wait(bar(B_KEMPTY + kst), (ku - 1) & 1);
          if (cta == 0) mbar_expect_tx(bar(B_KFULL + kst), (kPair ? 2 : 1) * C::kKBytes);
          for (int b = 0; b < 2; ++b) {
            const uint32_t dst = sbase + C::kSmemK + kst * C::kKBytes + b * C::kKBox;
            if constexpr (kPair)
              tma_load_2d_pair(dst, &tm_k, lead(B_KFULL + kst), kvh * kHeadDim + b * 64,
                               row + int(cta) * (kBN / 2), pol_kv);
            else
              tma_load_2d(dst, &tm_k, bar(B_KFULL + kst), kvh * kHeadDim + b * 64, row, pol_kv);
          }
          if (jg >= uint32_t(C::kVStages)) mbar_wait(bar(B_VEMPTY + vst), (vu - 1) & 1);
          if (cta == 0) mbar_expect_tx(bar(B_VFULL + vst), (kPair ? 2 : 1) * C::kVBytes);
          if constexpr (kPair) {
            tma_load_2d_pair(sbase + C::kSmemV + vst * C::kVBytes, &tm_v, lead(B_VFULL + vst),
                             kvh * kHeadDim + int(cta) * 64, row, pol_kv);
          } else {
            for (int b = 0; b < 2; ++b)
              tma_load_2d(sbase + C::kSmemV + vst * C::kVBytes + b * kBoxBytes, &tm_v, bar(B_VFULL + vst),
                          kvh * kHeadDim + b * 64, row, pol_kv);
          }
        }
        if (u.n_tiles == 1) load_q(1);
        ++qn;
      }
    } else if (warp == 1 && cta == 0) {
      // ---------------- MMA issuer (whole warp; one elected lane issues each
      // tcgen05 op).  Global tile stream: at tile g it issues
      // PV_t(g-1) then S_t(g) for t = 0, 1 (the S/P TMEM aliasing relies on
      // tcgen05 MMAs executing in issue order).
      constexpr uint32_t idesc_qk = idesc_bf16_f32(kPair ? 256 : 128, 128, 0, 0);
      // parity mode: P (TMEM A) and V (smem B) are fp16
      constexpr uint32_t idesc_pv = kParity ? idesc_f16_f32(kPair ? 256 : 128, 128, 0, 1)
                                            : idesc_bf16_f32(kPair ? 256 : 128, 128, 0, 1);
      const uint32_t tS[2] = {tmem + 0, tmem + 128};
      const uint32_t tO[2] = {tmem + 256, tmem + 384};
      const uint64_t q_desc0 = umma_desc_sw128(sbase + C::kSmemQ, 16, 1024);
      const uint64_t k_desc0 = umma_desc_sw128(sbase + C::kSmemK, 16, 1024);
      const uint64_t v_desc0 = umma_desc_sw128(sbase + C::kSmemV, kBoxBytes, 1024);
      constexpr uint64_t q_step = kTileBytes >> 4, k_step = C::kKBytes >> 4, v_step = C::kVBytes >> 4;
      uint32_t jg = 0, qn = 0;
      bool prev_acc = false;  // accumulate flag of the pending PV (tile jg-1)
      // PV_t of the previous tile, one 64-key half as soon as its P lands
      auto pv_prev = [&](int t, int pvs) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          mbar_wait(bar(B_PFULL + 2 * t + h), (jg - 1) & 1);
          tc_fence_after();
          if (lane == 0 && jg < 200) ZP_STAMP(2560 + int(jg - 1) * 6 + 3 * t + h);
          issue_pv<kPair>(tO[t], tS[t] + 64, v_desc0 + v_step * pvs, idesc_pv, prev_acc, h);
        }
        commit<kPair>(bar(B_ODONE + t));
      };
      for (uint32_t k = 0;; ++k) {
        const SchedSlot u = sched_wait(k);
        __syncwarp();
        if (lane == 0) sched_release(k);
        if (u.idx >= n_units) break;
        const zp_attn_item it = u.item;
        const int n = u.n_tiles;
        if (n == 0) continue;
        const bool resume = (it.flags & ZP_ITEM_LOAD_STATE) != 0;
        for (int j = 0; j < n; ++j, ++jg) {
          const int kst = int(jg % C::kKStages);
          const uint32_t kpar = (jg / C::kKStages) & 1;
          const int pvs = int((jg - 1) % C::kVStages);
          if (jg > 0) {
            mbar_wait(bar(B_VFULL + pvs), ((jg - 1) / C::kVStages) & 1);
            tc_fence_after();
          }
          // PV_t of the previous tile (possibly the previous item's last),
          // then S_t of this tile; at an item start S_t waits for head t's Q
          for (int t = 0; t < 2; ++t) {
            if (jg > 0) pv_prev(t, pvs);
            if (j == 0) mbar_wait(bar(t ? B_QFULL1 : B_QFULL), qn & 1);
            if (t == 0) mbar_wait(bar(B_KFULL + kst), kpar);
            tc_fence_after();
            issue_qk<kPair>(tS[t], q_desc0 + q_step * t, k_desc0 + k_step * kst, idesc_qk);
            commit<kPair>(bar(B_SFULL + t));
            if (j == n - 1) commit<kPair>(bar(t ? B_QEMPTY1 : B_QEMPTY));  // Q_t free once this S lands
            if (lane == 0 && jg < 200) ZP_STAMP(2560 + int(jg) * 6 + 3 * t + 2);
          }
          if (jg > 0) commit<kPair>(bar(B_VEMPTY + pvs));
          commit<kPair>(bar(B_KEMPTY + kst));
          prev_acc = resume || j > 0;
        }
        ++qn;
      }
      if (jg > 0) {
        const int pvs = int((jg - 1) % C::kVStages);
        mbar_wait(bar(B_VFULL + pvs), ((jg - 1) / C::kVStages) & 1);
        tc_fence_after();
        for (int t = 0; t < 2; ++t) pv_prev(t, pvs);
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(ZP_SM_REGS));
    // ---------------- softmax / correction / epilogue (thread == row)
    const int t = (warp - 4) >> 2;
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    const uint32_t lane_bits = uint32_t(quad * 32) << 16;
    const uint32_t tS = tmem + lane_bits + uint32_t(t * 128);
    const uint32_t tP = tS + 64;
    const uint32_t tO = tmem + lane_bits + 256u + uint32_t(t * 128);
    const uint32_t pfull = lead(B_PFULL + 2 * t);  // + 8 bytes: second half
    const float sl2 = args.scale_log2;
    uint32_t jg = 0;
#ifdef ZP_TRACE
    // item-level stamps: 3760 + (item * 2 + t) * 4 + {epilogue start, epilogue end, next item claimed, tiles counted}
    int tri = -4;
    auto item_stamp = [&](int e) {
      if (quad == 0 && lane == 0 && tri >= 0 && tri < 41) ZP_STAMP(3760 + (tri * 2 + t) * 4 + e);
    };
#else
    auto item_stamp = [](int) {};
#endif
    for (uint32_t k = 0;; ++k) {
      const SchedSlot u = sched_wait(k);
      __syncwarp();
      if (lane == 0) sched_release(k);
      item_stamp(2);
      if (u.idx >= n_units) break;
      const zp_attn_item it = u.item;
      TileCursor cur(args.segs, it.seg_begin, it.seg_count, it.q_pos0 + it.q_len - 1, u.seg0);
      if (u.n_tiles == 0) continue;
#ifdef ZP_TRACE
      ++tri;
#endif
      item_stamp(3);
      const bool resume = (it.flags & ZP_ITEM_LOAD_STATE) != 0;
      const int h = 2 * it.head_pair + t;
      const int qpos = it.q_pos0 + row;
      const bool ok = row < it.q_len;
      float m = -INFINITY, l = 0.f;

      if (resume) {
        // O_t is free: the previous item's epilogue (this thread) drained it.
        const int srow = it.state_row0 + row;
        if (ok) {
          m = args.st_ml[size_t(h) * args.state_rows + srow];
          l = args.st_ml[size_t(args.hq + h) * args.state_rows + srow];
        }
        const uint8_t* src = reinterpret_cast<const uint8_t*>(args.st_o + (size_t(srow) * args.hq + h) * kHeadDim);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t rr[32];
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            if (ok) {
              ldg_v8(src + c * 128 + v * 32, rr + 8 * v);
            } else {
#pragma unroll
              for (int e = 0; e < 8; ++e) rr[8 * v + e] = 0u;
            }
          }
          tmem_st32(tO + c * 32, rr);
        }
        tmem_wait_st();
      }

      for (int j = 0; cur.next(); ++j, ++jg) {
        mbar_wait(bar(B_SFULL + t), jg & 1);
        tc_fence_after();
        const int tr = (lane == 0 && quad == 0 && jg < 256) ? t * 1280 + int(jg) * 5 : -1;
        ZP_STAMP(tr);
        float s[128];
        {
          uint32_t r0[32], r1[32], r2[32], r3[32];
          tmem_ld32(tS + 0, r0);
          tmem_ld32(tS + 32, r1);
          tmem_ld32(tS + 64, r2);
          tmem_ld32(tS + 96, r3);
          tmem_wait_ld();
          ZP_STAMP(tr < 0 ? -1 : tr + 1);
#pragma unroll
          for (int v = 0; v < 32; ++v) {
            s[v] = __uint_as_float(r0[v]);
            s[32 + v] = __uint_as_float(r1[v]);
            s[64 + v] = __uint_as_float(r2[v]);
            s[96 + v] = __uint_as_float(r3[v]);
          }
        }
        const int kpos0 = cur.pos();
        const int kv_valid = cur.valid();
        const bool masked = kv_valid < kBN || kpos0 + kBN - 1 > it.q_pos0;
        if (masked) {
          const int lim = min(kv_valid - 1, qpos - kpos0);  // last visible column
#pragma unroll
          for (int c = 0; c < 128; ++c)
            if (c > lim) s[c] = -INFINITY;
        }
        float mx;  // row max in log2 units
        bool have_mx = false;
        if (kSpecExp && __all_sync(0xffffffffu, m > -INFINITY)) {
          // Speculative path: with a finite reference max, the first half's
          // exponentials start right away with it while the row max is folded
          // in alongside (ALU next to MUFU); only if some row exceeds the
          // reference by more than the lazy threshold is the work redone.
          const float2 sl2x2 = make_float2(sl2, sl2), negm = make_float2(-m, -m);
          float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
          uint32_t pa0[16], pa1[16];
          float c0 = -INFINITY, c1 = -INFINITY, c2 = -INFINITY, c3 = -INFINITY;
#pragma unroll
          for (int v = 0; v < 32; ++v) {
            const float2 x = __ffma2_rn(make_float2(s[2 * v], s[2 * v + 1]), sl2x2, negm);
            float2 p;
            p.x = ex2(x.x);
            p.y = ex2(x.y);
            if (v & 1) a1 = __fadd2_rn(a1, p); else a0 = __fadd2_rn(a0, p);
            if (v < 16) pa0[v] = pack_p<kParity>(p.x, p.y); else pa1[v - 16] = pack_p<kParity>(p.x, p.y);
            if (v & 1) {
              c0 = fmax3(c0, s[2 * v], s[2 * v + 1]);
              c1 = fmax3(c1, s[64 + 2 * v], s[64 + 2 * v + 1]);
            } else {
              c2 = fmax3(c2, s[2 * v], s[2 * v + 1]);
              c3 = fmax3(c3, s[64 + 2 * v], s[64 + 2 * v + 1]);
            }
          }
          mx = fmax3(c0, c1, fmaxf(c2, c3)) * sl2;
          have_mx = true;
          if (!__any_sync(0xffffffffu, mx > m + kRescaleLog2)) {
            tmem_st16(tP, pa0);
            tmem_st16(tP + 16, pa1);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              if constexpr (kPair) mbar_arrive_remote(pfull);
              else mbar_arrive(pfull);
            }
            ZP_STAMP(tr < 0 ? -1 : tr + 2);
            ZP_STAMP(tr < 0 ? -1 : tr + 3);
            if (masked) exp_half<1, false, kParity>(s, sl2x2, negm, tP, a0, a1);
            else exp_half<1, true, kParity>(s, sl2x2, negm, tP, a0, a1);
            const float2 acc = __fadd2_rn(a0, a1);
            l += acc.x + acc.y;
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              if constexpr (kPair) mbar_arrive_remote(pfull + 8);
              else mbar_arrive(pfull + 8);
            }
            ZP_STAMP(tr < 0 ? -1 : tr + 4);
            continue;
          }
        }
        if (!have_mx) {
          // row max with 3-input max (FMNMX3), four independent chains
          float mx0 = fmax3(s[0], s[1], s[2]), mx1 = fmax3(s[3], s[4], s[5]);
          float mx2 = fmax3(s[6], s[7], s[8]), mx3 = fmax3(s[9], s[10], s[11]);
#pragma unroll
          for (int c = 12; c < 124; c += 8) {
            mx0 = fmax3(mx0, s[c], s[c + 1]);
            mx1 = fmax3(mx1, s[c + 2], s[c + 3]);
            mx2 = fmax3(mx2, s[c + 4], s[c + 5]);
            mx3 = fmax3(mx3, s[c + 6], s[c + 7]);
          }
          mx0 = fmax3(mx0, s[124], s[125]);
          mx1 = fmax3(mx1, s[126], s[127]);
          mx = fmax3(mx0, mx1, fmaxf(mx2, mx3)) * sl2;
        }
#ifdef ZP_TRACE
        asm volatile("" ::"f"(mx));
        ZP_STAMP(tr < 0 ? -1 : tr + 2);
#endif
        // Lazy rescale: keep the reference max unless this tile exceeds it by
        // more than 2^8; P <= 256 is exact enough in bf16 / fp32 and O, l stay
        // consistent with the reference actually used.
        const bool bump = mx > m + kRescaleLog2;
        const float m_new = bump ? mx : m;
        const float m_use = (m_new == -INFINITY) ? 0.f : m_new;
        const float alpha = bump ? ex2(m - m_use) : 1.f;
        // O_t must hold PV(g-1) before it is rescaled, and PV(g) is issued only
        // after this warp's first P arrival, so rescale first — and wait for
        // PV(g-1) only when this warp actually rescales.
        if ((j > 0 || resume) && __any_sync(0xffffffffu, bump)) {
          if (j > 0) {
            mbar_wait(bar(B_ODONE + t), (jg - 1) & 1);
            tc_fence_after();
          }
          const float2 a2 = make_float2(alpha, alpha);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t rr[32];
            tmem_ld32(tO + c * 32, rr);
            tmem_wait_ld();
#pragma unroll
            for (int v = 0; v < 16; ++v) {
              const float2 o2 = __fmul2_rn(make_float2(__uint_as_float(rr[2 * v]), __uint_as_float(rr[2 * v + 1])), a2);
              rr[2 * v] = __float_as_uint(o2.x);
              rr[2 * v + 1] = __float_as_uint(o2.y);
            }
            tmem_st32(tO + c * 32, rr);
          }
        }
        // P in two 64-key halves; the MMA issues PV over the first half while
        // the second half's exponentials run.
        const float2 sl2x2 = make_float2(sl2, sl2), negm = make_float2(-m_use, -m_use);
        float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
        if (masked) exp_half<0, false, kParity>(s, sl2x2, negm, tP, acc0, acc1);
        else exp_half<0, true, kParity>(s, sl2x2, negm, tP, acc0, acc1);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (kPair) mbar_arrive_remote(pfull);
          else mbar_arrive(pfull);
        }
        ZP_STAMP(tr < 0 ? -1 : tr + 3);
        if (masked) exp_half<1, false, kParity>(s, sl2x2, negm, tP, acc0, acc1);
        else exp_half<1, true, kParity>(s, sl2x2, negm, tP, acc0, acc1);
        const float2 acc = __fadd2_rn(acc0, acc1);
        l = l * alpha + (acc.x + acc.y);
        m = m_new;
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (kPair) mbar_arrive_remote(pfull + 8);
          else mbar_arrive(pfull + 8);
        }
        ZP_STAMP(tr < 0 ? -1 : tr + 4);
      }

      // ---------------- epilogue of this item (overlaps the next item's S MMAs)
      mbar_wait(bar(B_ODONE + t), (jg - 1) & 1);
      tc_fence_after();
      item_stamp(0);
      if (it.flags & ZP_ITEM_STORE_STATE) {
        const int srow = it.state_row0 + row;
        uint8_t* dst = reinterpret_cast<uint8_t*>(args.st_o + (size_t(srow) * args.hq + h) * kHeadDim);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t rr[32];
          tmem_ld32(tO + c * 32, rr);
          tmem_wait_ld();
          if (ok) {
#pragma unroll
            for (int v = 0; v < 4; ++v) stg_v8(dst + c * 128 + v * 32, rr + 8 * v);
          }
        }
        if (ok) {
          args.st_ml[size_t(h) * args.state_rows + srow] = m;
          args.st_ml[size_t(args.hq + h) * args.state_rows + srow] = l;
        }
      } else {
        const float inv_l = l > 0.f ? 1.f / l : 0.f;
        // one 256-bit store per 16 dims (8 fp32 dims in the parity mode):
        // full 32-byte sectors of the row
        const size_t orow = (size_t(it.q_row0 + row) * args.hq + h) * kHeadDim;
        uint8_t* dst = kParity ? reinterpret_cast<uint8_t*>(static_cast<float*>(args.o) + orow)
                               : reinterpret_cast<uint8_t*>(static_cast<__nv_bfloat16*>(args.o) + orow);
        const float2 il2 = make_float2(inv_l, inv_l);
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          uint32_t rr[64];  // two TMEM loads in flight per wait
          tmem_ld32(tO + cc * 64, *reinterpret_cast<uint32_t(*)[32]>(rr));
          tmem_ld32(tO + cc * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(rr + 32));
          tmem_wait_ld();
          if (ok) {
            if constexpr (kParity) {
#pragma unroll
              for (int v = 0; v < 32; ++v) {
                const float2 x =
                    __fmul2_rn(make_float2(__uint_as_float(rr[2 * v]), __uint_as_float(rr[2 * v + 1])), il2);
                rr[2 * v] = __float_as_uint(x.x);
                rr[2 * v + 1] = __float_as_uint(x.y);
              }
#pragma unroll
              for (int w = 0; w < 8; ++w) stg_v8(dst + cc * 256 + w * 32, rr + 8 * w);
            } else {
              uint32_t pk[32];
#pragma unroll
              for (int v = 0; v < 32; ++v) {
                const float2 x =
                    __fmul2_rn(make_float2(__uint_as_float(rr[2 * v]), __uint_as_float(rr[2 * v + 1])), il2);
                pk[v] = pack_bf16(x.x, x.y);
              }
#pragma unroll
              for (int w = 0; w < 4; ++w) stg_v8(dst + cc * 128 + w * 32, pk + 8 * w);
            }
          }
        }
        if (ok) {
          const float lse = l > 0.f ? (m + __log2f(l)) * 0.69314718055994531f : -INFINITY;
          args.lse[size_t(h) * args.lse_stride + it.q_row0 + row] = lse;
        }
      }
      item_stamp(1);
    }
  }

  __syncwarp();
  tc_fence_before();
  if constexpr (kPair) cluster_sync_all();  // the peer's last MMAs / arrivals are done
  else __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    if constexpr (kPair) tmem_dealloc_pair(tmem, 512);
    else tmem_dealloc(tmem, 512);
  }
}



}  // namespace zp

// ------------------------------------------------------------------ host side
#include "zp_host.h"

namespace {

int g_sm_reserve = 0;  // zp_attn_set_sm_reserve

// ZP_ATTN_VARIANT (A/B measurements only): "single" = one-CTA kernel;
// default = CTA pair (when the GQA group allows it).
int variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("ZP_ATTN_VARIANT");
    v = !e ? 1 : (e[0] == 's' ? 0 : 1);
  }
  return v;
}

// Per-device launch facts (the smem attribute is per device and function; the
// resident CTA / cluster count comes from that device's occupancy query).
struct LaunchCache {
  bool done = false;
  int max_units = 0;  // resident CTAs (single) or CTA pairs (pair)
};
constexpr int kMaxDevices = 64;

template <bool kPair, bool kParity>
int launch_attn(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, zp::AttnArgs a,
                int n_units, cudaStream_t stream) {
  using namespace zp;
  constexpr uint32_t smem = Cfg<kPair>::kSmemBytes;
  auto kernel = attn_fwd_kernel<kPair, kParity>;
  static LaunchCache cache[kMaxDevices];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices)
    return zp_fail(ZP_ENODEV, "zp_attn_fwd: no current device");
  LaunchCache& lc = cache[dev];
  if (!lc.done) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return zp_fail_cuda(e, "zp_attn_fwd: smem attribute");
    const int sms = zp_device_sm_count();
    if (sms <= 0) return zp_fail(ZP_ENODEV, "zp_attn_fwd: cannot query SM count");
    int units = sms;
    if (kPair) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(2 * (sms / 2));
      cfg.blockDim = dim3(kThreads);
      cfg.dynamicSmemBytes = smem;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int clusters = 0;
      e = cudaOccupancyMaxActiveClusters(&clusters, kernel, &cfg);
      if (e != cudaSuccess || clusters <= 0) {
        cudaGetLastError();
        clusters = sms / 2;
      }
      units = clusters;
    }
    lc.max_units = units;
    lc.done = true;
  }
  a.n_units = n_units;
  // persistent; g_sm_reserve SMs (whole units) stay free for concurrent comm kernels
  const int per_unit = kPair ? 2 : 1;
  int cap = lc.max_units - (g_sm_reserve + per_unit - 1) / per_unit;
  if (cap < 1) cap = 1;
  const int units = n_units < cap ? n_units : cap;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  if (kPair) {
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(2 * units);
  } else {
    cfg.gridDim = dim3(units);
  }
  cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, tq, tk, tv, a);
  if (e != cudaSuccess) return zp_fail_cuda(e, "zp_attn_fwd: launch");
  return ZP_OK;
}

int attn_fwd_common(bool parity, const void* q, const void* k, const void* v, int q_rows, int kv_rows,
                    int kv_row_stride, int hq, int hkv, int head_dim, void* o, float* lse, int lse_stride,
                    const zp_attn_item* items, int n_items, const zp_kv_seg* segs, float* state_o,
                    float* state_ml, int state_rows, float softmax_scale, void* workspace, void* stream) {
  using namespace zp;
  if (head_dim != kHeadDim) return zp_fail(ZP_EINVAL, "zp_attn_fwd: head_dim must be 128");
  if (hq <= 0 || hkv <= 0 || hq % hkv != 0 || (hq / hkv) % 2 != 0)
    return zp_fail(ZP_EINVAL, "zp_attn_fwd: need hq % hkv == 0 and an even GQA group size");
  if (n_items < 0 || q_rows < 0 || kv_rows < 0 || kv_row_stride < hkv * kHeadDim)
    return zp_fail(ZP_EINVAL, "zp_attn_fwd: bad sizes");
  if (n_items == 0) return ZP_OK;
  if (q_rows == 0 || kv_rows == 0) return zp_fail(ZP_EINVAL, "zp_attn_fwd: empty q or kv with items");
  if (!q || !k || !v || !o || !lse || !items || !segs || !workspace)
    return zp_fail(ZP_EINVAL, "zp_attn_fwd: null pointer");
  if (zp_check_device() != ZP_OK) return ZP_ENODEV;

  // CTA pairs need both head pairs of a pair item to share the KV head
  // (GQA group a multiple of 4) and the item list in aligned pairs.
  const int var = variant();
  const bool pair = (hq / hkv) % 4 == 0 && n_items % 2 == 0 && var != 0;
  CUtensorMap tq, tk, tv;
  int rc;
  if ((rc = zp_make_tmap_2d_bf16(&tq, q, uint64_t(hq) * kHeadDim, uint64_t(q_rows),
                                 uint64_t(hq) * kHeadDim * 2, 64, 128)) != ZP_OK)
    return rc;
  if ((rc = zp_make_tmap_2d_bf16(&tk, k, uint64_t(hkv) * kHeadDim, uint64_t(kv_rows),
                                 uint64_t(kv_row_stride) * 2, 64, pair ? 64 : 128)) != ZP_OK)
    return rc;
  // (parity: v holds fp16; a 2-byte TMA copy moves the bits unchanged)
  if ((rc = zp_make_tmap_2d_bf16(&tv, v, uint64_t(hkv) * kHeadDim, uint64_t(kv_rows),
                                 uint64_t(kv_row_stride) * 2, 64, 128)) != ZP_OK)
    return rc;

  AttnArgs a;
  a.items = items;
  a.next_unit = reinterpret_cast<int*>(workspace);
  a.segs = segs;
  a.o = o;
  a.lse = lse;
  a.st_o = state_o;
  a.st_ml = state_ml;
  a.lse_stride = lse_stride;
  a.state_rows = state_rows;
  a.hq = hq;
  a.group = hq / hkv;
  a.q_rows = q_rows;
  a.kv_rows = kv_rows;
  a.scale_log2 = softmax_scale * 1.4426950408889634f;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t me = cudaMemsetAsync(workspace, 0, sizeof(int), s);
  if (me != cudaSuccess) return zp_fail_cuda(me, "zp_attn_fwd: workspace reset");
  if (parity)
    return pair ? launch_attn<true, true>(tq, tk, tv, a, n_items / 2, s)
                : launch_attn<false, true>(tq, tk, tv, a, n_items, s);
  return pair ? launch_attn<true, false>(tq, tk, tv, a, n_items / 2, s)
              : launch_attn<false, false>(tq, tk, tv, a, n_items, s);
}

}  // namespace

#ifdef ZP_TRACE
extern "C" ZP_API int zp_debug_trace(unsigned long long* host, int n) {
  return cudaMemcpyFromSymbol(host, zp::g_zp_trace, sizeof(unsigned long long) * (n < 8192 ? n : 8192)) ==
                 cudaSuccess ? 0 : -1;
}
#endif

extern "C" int zp_attn_set_sm_reserve(int sms) {
  const int prev = g_sm_reserve;
  g_sm_reserve = sms < 0 ? 0 : sms;
  return prev;
}

extern "C" int zp_attn_fwd(const void* q, const void* k, const void* v, int q_rows, int kv_rows,
                           int kv_row_stride, int hq, int hkv, int head_dim, void* o, float* lse,
                           int lse_stride, const zp_attn_item* items, int n_items,
                           const zp_kv_seg* segs, float* state_o, float* state_ml,
                           int state_rows, float softmax_scale, void* workspace, void* stream) {
  return attn_fwd_common(false, q, k, v, q_rows, kv_rows, kv_row_stride, hq, hkv, head_dim, o, lse, lse_stride,
                         items, n_items, segs, state_o, state_ml, state_rows, softmax_scale, workspace, stream);
}

extern "C" int zp_attn_fwd_parity(const void* q, const void* k, const void* v_f16, int q_rows, int kv_rows,
                                  int kv_row_stride, int hq, int hkv, int head_dim, float* o, float* lse,
                                  int lse_stride, const zp_attn_item* items, int n_items,
                                  const zp_kv_seg* segs, float* state_o, float* state_ml,
                                  int state_rows, float softmax_scale, void* workspace, void* stream) {
  return attn_fwd_common(true, q, k, v_f16, q_rows, kv_rows, kv_row_stride, hq, hkv, head_dim, o, lse,
                         lse_stride, items, n_items, segs, state_o, state_ml, state_rows, softmax_scale,
                         workspace, stream);
}
