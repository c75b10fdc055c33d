/*
 * zeppelin_b200.h — C ABI of the B200 (sm_100a) per-layer hot path of Zeppelin
 * (arXiv 2509.21841): the varlen / ring-round causal attention engine and the
 * attention<->linear remapping layer.
 *
 * The reference (`/root/reference/pkg/src/varlenplan`) is a pure-Python cost
 * model: it counts causal (q,k) pairs and KV tokens but never computes them.
 * Each entry point below is the device execution of one thing the reference
 * only charges a cost for:
 *
 *   zp_attn_fwd        LocalTask / RingRound compute
 *                        attention_engine.py:113-141  (visible_pairs: mask semantics)
 *                        attention_engine.py:229-244  (_ring_schedule: src=(i-r)%g)
 *                        attention_engine.py:260-265  (LocalTask: whole-sequence causal)
 *                        simulator.py:142-148,181-187 (where the cost model charges it)
 *   zp_copy_rows       ring KV pack (held KV set of a ring position) and the
 *                      remap kept-row/tail copies
 *                        attention_engine.py:247-251  (KV rotates i -> i+1)
 *                        remapping.py:187-245         (transfer matrix M rows)
 *   zp_attn_fwd_parity the same compute with fp16 P / V and fp32 O: the checkable
 *                      form of the north star's mean-rel 1e-3 tolerance
 *   zp_ring_hop        one RingRound KV forward (position i -> i+1) as a pull by
 *   (+ zp_stream_*)    i+1: stream-waited epoch flags + one copy-engine transfer
 *                        attention_engine.py:237,247-251; simulator.py:150-174
 *   zp_remap_pull/push fused remap: rows of M[i][j] moved between peer buffers
 *                      over NVLink, bracketed by ready/done epoch flags
 *                        remapping.py:187-255, simulator.py:282-302,336-347
 *   zp_attn_bwd        the backward the reference charges as a multiple of the
 *   (+ zp_add_f32)     forward (topology.py:37, simulator.py:304); ring dK/dV
 *                      totals travel with the KV sets (README.md:119-124)
 *
 * Conventions: all pointers are device pointers (except where noted); the
 * library never allocates device memory; every call is asynchronous on the
 * given cudaStream_t (passed as void*).  Return 0 on success or a negative
 * ZP_E* code; zp_last_error() returns a static description of the last error.
 * There is no CPU fallback: without an sm_100a device every call fails.
 */
#ifndef ZEPPELIN_B200_H
#define ZEPPELIN_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define ZP_API __attribute__((visibility("default")))
#else
#define ZP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define ZP_OK 0
#define ZP_EINVAL (-1)   /* bad argument / unsupported shape */
#define ZP_ETMA (-2)     /* tensor-map encode failed */
#define ZP_ECUDA (-3)    /* CUDA runtime error (launch, attribute, ...) */
#define ZP_ENODEV (-4)   /* no sm_100 device */

/* One attention work item: a tile of <=128 query rows of one sequence
 * fragment (contiguous global positions), for a PAIR of query heads
 * (2*head_pair, 2*head_pair+1) that share one KV head (GQA group size even).
 * The item attends to `seg_count` KV segments starting at `seg_begin`. */
typedef struct zp_attn_item {
  int32_t q_row0;     /* physical row of the first query row in q/o */
  int32_t q_pos0;     /* global in-sequence position of that row */
  int32_t q_len;      /* valid rows, 1..128 */
  int32_t head_pair;  /* query heads 2*head_pair and 2*head_pair+1 */
  int32_t seg_begin;  /* index into the KV segment table */
  int32_t seg_count;  /* number of KV segments (same sequence) */
  int32_t state_row0; /* row of this tile in the ring partial-state buffers */
  int32_t flags;      /* ZP_ITEM_* */
} zp_attn_item;

/* A contiguous run of KV rows of one sequence: rows [row0,row0+len) of k/v
 * hold global positions [pos0, pos0+len). */
typedef struct zp_kv_seg {
  int32_t row0;
  int32_t pos0;
  int32_t len;
  int32_t reserved;
} zp_kv_seg;

#define ZP_ITEM_LOAD_STATE 1  /* resume from (m, l, O_acc) partial state */
#define ZP_ITEM_STORE_STATE 2 /* write partial state instead of final O/LSE */

/* Causal flash attention over a work-item list (bf16 in, fp32 accumulate).
 * q: [q_rows, hq, 128] bf16; k, v: [kv_rows, hkv, 128] bf16 with row stride
 * kv_row_stride elements (>= hkv*128; lets K and V live interleaved in one
 * ring buffer); o: [q_rows, hq, 128] bf16; lse: [hq, lse_stride] fp32 (natural
 * log).  Mask: key position <= query position (global in-sequence positions).
 * state_o: [state_rows, hq, 128] fp32 unnormalised accumulator, state_ml:
 * [2, hq, state_rows] fp32 (running max in log2 units, running sum); only
 * touched by items carrying ZP_ITEM_*_STATE.  Items must be device-resident.
 * workspace: >= ZP_ATTN_WORKSPACE_BYTES of device memory owned by the caller
 * (the persistent CTAs' work counter; zeroed by the call on `stream`).  Items
 * are claimed in list order, so pass them longest-first.
 * When (hq/hkv) % 4 == 0 the kernel runs CTA pairs (cta_group::2): items 2p
 * and 2p+1 must then describe the same query tile for head pairs 2g and 2g+1
 * (the order worklist.build_worklist emits); a violation traps the kernel. */
#define ZP_ATTN_WORKSPACE_BYTES 16
ZP_API int zp_attn_fwd(const void* q, const void* k, const void* v, int q_rows, int kv_rows,
                int kv_row_stride, int hq, int hkv, int head_dim, void* o, float* lse,
                int lse_stride, const zp_attn_item* items, int n_items, const zp_kv_seg* segs,
                float* state_o, float* state_ml, int state_rows, float softmax_scale,
                void* workspace, void* stream);

/* Parity mode of zp_attn_fwd (same work items, same kernel pipeline): v_f16
 * holds V converted to fp16 (same layout / strides as zp_attn_fwd's v), the
 * probabilities P are staged as fp16 instead of bf16 for the P.V product, and
 * o is written as fp32 [q_rows, hq, 128] (unrounded).  This isolates the
 * kernel's arithmetic from the bf16 output rounding so that the north star's
 * mean-relative tolerance (1e-3 vs fp32) is checkable; the production path is
 * zp_attn_fwd. */
ZP_API int zp_attn_fwd_parity(const void* q, const void* k, const void* v_f16, int q_rows, int kv_rows,
                int kv_row_stride, int hq, int hkv, int head_dim, float* o, float* lse,
                int lse_stride, const zp_attn_item* items, int n_items, const zp_kv_seg* segs,
                float* state_o, float* state_ml, int state_rows, float softmax_scale,
                void* workspace, void* stream);

/* ---------------------------------------------------------------- backward
 * (the reference charges backward as a multiple of the
 * forward, topology.py:37 / simulator.py:304; executed here for the same
 * LocalTask and RingRound work, attention_engine.py:229-265.)
 *
 * One backward work item: up to 128 keys (rows [kv_row0, +kv_len) of k/v,
 * global positions [kv_pos0, ...)) of KV head kv_head, against every query of
 * the query segments [qseg_begin, +qseg_count) (zp_kv_seg rows/positions of
 * q) that can see them, for all hq/hkv query heads of the group. */
typedef struct zp_bwd_item {
  int32_t kv_row0;
  int32_t kv_pos0;
  int32_t kv_len;     /* 1..128 */
  int32_t kv_head;
  int32_t qseg_begin;
  int32_t qseg_count;
  int32_t flags;      /* ZP_BWD_* */
  int32_t reserved;
} zp_bwd_item;

#define ZP_BWD_ACCUMULATE 1 /* add dK/dV into dk/dv instead of overwriting */

/* delta[h * delta_stride + row] = sum_d o[row,h,d] * dout[row,h,d] (fp32);
 * o, dout: [rows, hq, 128] bf16. */
ZP_API int zp_attn_bwd_prep(const void* o, const void* dout, int rows, int hq, int head_dim,
                     float* delta, int delta_stride, void* stream);

/* Causal flash attention backward over a work-item list (bf16 in, fp32
 * accumulate).  q, dout: [q_rows, hq, 128] bf16 (row-contiguous); k, v as in
 * zp_attn_fwd; lse (natural log, the forward's FINAL value) and delta:
 * [hq, lse_stride] fp32.  dq: [q_rows, hq, 128] fp32, ACCUMULATED with
 * atomic adds (zero it before the first call); dk, dv: [kv_rows, hkv, 128]
 * fp32, each item writes (or, with ZP_BWD_ACCUMULATE, adds to) its own rows —
 * items of one call must cover disjoint (key row, kv head) tiles. */
ZP_API int zp_attn_bwd(const void* q, const void* k, const void* v, const void* dout, int q_rows,
                int kv_rows, int kv_row_stride, int hq, int hkv, int head_dim, const float* lse,
                const float* delta, int lse_stride, float* dq, float* dk, float* dv,
                const zp_bwd_item* items, int n_items, const zp_kv_seg* qsegs,
                float softmax_scale, void* stream);

/* Row-range copy with 16-byte vector loads/stores.  For each range i:
 * dst rows [dst_row0[i], +n_rows[i]) <- src rows [src_row0[i], +n_rows[i]).
 * ranges: device int32 [n_ranges][3] = {dst_row0, src_row0, n_rows}.
 * row_bytes, strides and both base pointers must be 16-byte aligned. */
ZP_API int zp_copy_rows(void* dst, int64_t dst_stride_bytes, const void* src, int64_t src_stride_bytes,
                 int64_t row_bytes, const int32_t* ranges, int n_ranges, int max_rows_per_range,
                 void* stream);

/* dst[i] += src[i] for n fp32 values (n % 4 == 0, 16-byte aligned): the ring
 * backward adds the dK/dV partial sum received for a travelling KV set to this
 * position's contribution before forwarding it (README.md:119-124 charges
 * the g sends of a ring). */
ZP_API int zp_add_f32(float* dst, const float* src, int64_t n, void* stream);

/* Fused remap push (collective: every rank calls it with the same epoch).
 * flags_ptrs[r] points at rank r's int32[2*world] flag block (IPC-mapped):
 * [0,world) "done from sender s", [world,2*world) "ready from rank s".
 *  1. ready: release-store `epoch` into every peer's ready slot, then wait
 *     until each destination d (count[d] > 0) has announced `epoch` — so no
 *     rank overwrites a buffer its owner is still reading;
 *  2. push: rows [src_row0[d], +count[d]) of `src` are stored straight into
 *     dst_ptrs[d] (a peer pointer valid in this process) at row dst_row0[d],
 *     16-byte vector stores over NVLink;
 *  3. done: release-store `epoch` into each destination's done slot, then
 *     acquire-wait for `epoch` from every sender s with expect[s] != 0.
 * Epochs must increase from call to call.  All tables are device arrays of
 * length world (int64 pointers, int32 counts/rows). */
ZP_API int zp_remap_push(const void* src, int64_t row_bytes, const int64_t* dst_ptrs,
                  const int32_t* src_row0, const int32_t* dst_row0, const int32_t* count,
                  const int64_t* flags_ptrs, const int32_t* expect, int world, int my_rank,
                  int32_t epoch, int max_count, void* stream);

/* Fused remap, pull form (collective): rank `my_rank` copies rows
 * [src_row0[s], +count[s]) of source rank s's buffer src_ptrs[s] (peer
 * pointer) into its local `dst` at row dst_row0[s] — peer LDG.128 over
 * NVLink.  Handshake as zp_remap_push with the roles of the flags swapped:
 * ready = "my rows are final for `epoch`", done = "I finished reading your
 * rows"; the call returns (on `stream`) only after every rank with
 * readers[r] != 0 has read this rank's rows. */
ZP_API int zp_remap_pull(void* dst, int64_t row_bytes, const int64_t* src_ptrs,
                  const int32_t* src_row0, const int32_t* dst_row0, const int32_t* count,
                  const int64_t* flags_ptrs, const int32_t* readers, int world, int my_rank,
                  int32_t epoch, int max_count, void* stream);

/* zp_remap_push / zp_remap_pull with a subset of their three stages:
 * phases bit 1 = ready handshake, 2 = row move, 4 = done handshake (7 = the
 * whole call).  Lets ranks emulated in one process on one GPU enqueue every
 * rank's ready stage before any rank's move (the single-GPU tests). */
ZP_API int zp_remap_push_phased(const void* src, int64_t row_bytes, const int64_t* dst_ptrs,
                  const int32_t* src_row0, const int32_t* dst_row0, const int32_t* count,
                  const int64_t* flags_ptrs, const int32_t* expect, int world, int my_rank,
                  int32_t epoch, int max_count, int phases, void* stream);
ZP_API int zp_remap_pull_phased(void* dst, int64_t row_bytes, const int64_t* src_ptrs,
                  const int32_t* src_row0, const int32_t* dst_row0, const int32_t* count,
                  const int64_t* flags_ptrs, const int32_t* readers, int world, int my_rank,
                  int32_t epoch, int max_count, int phases, void* stream);

/* Bound of every handshake spin (ready / done flags of the remap): a rank
 * that waits longer prints the ranks and epochs involved and traps, so a
 * crashed peer fails the job instead of hanging the GPU.  ms <= 0 restores
 * the default (30 s).  Returns the previous bound in ms. */
ZP_API int zp_set_spin_timeout_ms(int64_t ms);

/* Same contract as zp_remap_pull, but the row blocks are moved by the copy
 * engines (one cudaMemcpyAsync per source rank, enqueued between the ready
 * and done handshake kernels), leaving every SM free for concurrent compute.
 * Row tables are HOST arrays here; count_dev / readers_dev are their device
 * copies for the handshake kernels. */
ZP_API int zp_remap_pull_ce(void* dst, int64_t row_bytes, const int64_t* src_ptrs_host,
                     const int32_t* src_row0_host, const int32_t* dst_row0_host,
                     const int32_t* count_host, const int64_t* flags_ptrs,
                     const int32_t* count_dev, const int32_t* readers_dev, int world,
                     int my_rank, int32_t epoch, void* stream);

/* zp_remap_push with the row blocks written by the sender's copy engines
 * (one cudaMemcpyAsync per destination into its IPC-mapped buffer) between
 * the ready and done handshake kernels.  Host row tables + device copies of
 * count / expect for the handshake. */
ZP_API int zp_remap_push_ce(const void* src, int64_t row_bytes, const int64_t* dst_ptrs_host,
                     const int32_t* src_row0_host, const int32_t* dst_row0_host,
                     const int32_t* count_host, const int64_t* flags_ptrs,
                     const int32_t* count_dev, const int32_t* expect_dev, int world,
                     int my_rank, int32_t epoch, void* stream);

/* ---------------------------------------------------------------- ring KV exchange
 * (attention_engine.py:247-251: after round r position i forwards the KV set
 * it holds to position i+1; simulator.py:150-174 charges it.)  Executed as a
 * PULL by position i+1 with no SM involvement: stream memory operations wait
 * on / write int32 epoch flags and one copy-engine transfer moves the bytes
 * over NVLink, so a hop overlaps a ring round that occupies every SM.
 * Flags are compared with wrap-around ">=" (int32)(*flag - epoch) >= 0. */

/* Enqueue on `stream`: wait until *flag >= epoch (flag: device memory of the
 * calling GPU, written by peers). */
ZP_API int zp_stream_wait_flag(const int32_t* flag, int32_t epoch, void* stream);

/* Enqueue on `stream`: *flag = epoch after every earlier operation of the
 * stream (memory barrier), flag may be a peer (IPC-mapped) address. */
ZP_API int zp_stream_write_flag(int32_t* flag, int32_t epoch, void* stream);

/* One hop, pull form, enqueued on `stream`:
 *  1. wait *full_flag >= full_epoch     (the predecessor's set is in `src`);
 *  2. if free_flag: wait *free_flag >= free_epoch   (the successor finished
 *     reading what `dst` held before);
 *  3. copy `bytes` from src (predecessor's IPC-mapped buffer) to dst;
 *  4. *consumed_flag = consumed_epoch   (in the predecessor's flag block);
 *  5. if next_full_flag: *next_full_flag = next_full_epoch   (in the
 *     successor's flag block: dst now holds the set it pulls next). */
ZP_API int zp_ring_hop(void* dst, const void* src, int64_t bytes, const int32_t* full_flag,
                int32_t full_epoch, const int32_t* free_flag, int32_t free_epoch,
                int32_t* consumed_flag, int32_t consumed_epoch, int32_t* next_full_flag,
                int32_t next_full_epoch, void* stream);

/* Stream-ordered device copy (copy engine; src may be a peer's IPC-mapped
 * address: the ring backward pulls the predecessor's dK/dV partial sums with
 * it between zp_stream_wait_flag / zp_stream_write_flag) and memset. */
ZP_API int zp_memcpy_async(void* dst, const void* src, int64_t bytes, void* stream);
ZP_API int zp_memset_async(void* dst, int value, int64_t bytes, void* stream);

/* ---- full transformer block (config 5): elementwise kernels around the
 * cuBLAS GEMMs of the linear modules, which run on the balanced (linear)
 * layout as in the reference's linear phase (simulator.py:291-299). */

/* y = x / sqrt(mean(x^2) + eps) * w, rows x hidden bf16 (hidden % 8 == 0, <= 8192). */
ZP_API int zp_rmsnorm(const void* x, const void* w, void* y, int rows, int hidden, float eps,
               void* stream);

/* Split qkv [rows, (hq+2*hkv)*128] bf16 (attention layout) into q [rows,hq,128],
 * k, v [rows,hkv,128]; q and k rotated (rotate-half RoPE) at each row's GLOBAL
 * in-sequence position pos[row], cos/sin from fp32 tables [max_pos, 64]. */
ZP_API int zp_rope_split(const void* qkv, const int32_t* pos, const float* cos_table,
                  const float* sin_table, void* q, void* k, void* v, int rows, int hq,
                  int hkv, int head_dim, void* stream);

/* a = silu(g) * u for gu = [rows, 2*inter] = [g | u] bf16 -> out [rows, inter]. */
ZP_API int zp_swiglu(const void* gu, void* out, int rows, int inter, void* stream);

/* CUDA IPC helpers for zp_remap_push (host pointers to 64-byte handles).
 * get_handle exports the allocation containing dev_ptr and returns dev_ptr's
 * byte offset inside it; a peer maps it with open_handle and adds the offset. */
ZP_API int zp_ipc_get_handle(void* dev_ptr, void* handle_out64, int64_t* offset_out);
ZP_API int zp_ipc_open_handle(const void* handle64, void** dev_ptr_out);
ZP_API int zp_ipc_close_handle(void* dev_ptr);

/* SMs the persistent attention launches leave free (rounded up to whole CTA
 * pairs), process-wide; 0 (default) = every SM.  Ring rounds set it while a
 * KV hop is in flight so the communication kernels (NCCL P2P) are not queued
 * behind a kernel that holds every SM.  Returns the previous value. */
ZP_API int zp_attn_set_sm_reserve(int sms);

/* Misc. */
ZP_API const char* zp_last_error(void);
ZP_API int zp_device_sm_count(void);
ZP_API int zp_version(void);  /* 2 since round 2 (parity kernel, ring hops, phased remap) */

#ifdef __cplusplus
}
#endif
#endif /* ZEPPELIN_B200_H */
