// KV-tile walk shared by the forward kernel and the backward's dQ pass.
#pragma once
#include "zp_ptx.cuh"
#include "../../include/zeppelin_b200.h"

namespace zp {

constexpr int kTileKeys = 128;  // keys per KV tile

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
        nt = (min(g.len, max_qpos - g.pos0 + 1) + kTileKeys - 1) / kTileKeys;
        ti = 0;
        return true;
      }
    }
    return false;
  }
  __device__ __forceinline__ int row() const { return g.row0 + ti * kTileKeys; }
  __device__ __forceinline__ int pos() const { return g.pos0 + ti * kTileKeys; }
  __device__ __forceinline__ int valid() const { return min(kTileKeys, g.len - ti * kTileKeys); }
};


}  // namespace zp
