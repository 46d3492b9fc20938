// cache.cuh -- NEXT-3 internals shared by cache.cu (directory kernels) and features.cu (the
// gather entry point): the HBM feature cache's workspace layout and its per-batch step.
#pragma once

#include "common.cuh"

namespace cmb {

// Workspace of an HBM software cache of `capacity` feature rows over a host-resident table:
//   slot_of[N]   int32  cache slot of node v, or -1
//   node_of[C]   int32  node cached in slot s, or -1
//   used[C]      uint32 tag of the last batch that referenced slot s (protects it from eviction
//                       inside that batch)
//   ref[C]       uint8  CLOCK reference bit (second chance: an approximation of LRU)
//   hand         uint64 CLOCK hand (monotone counter, slot = hand % C)
//   counters     uint64 [0] misses of the current batch
//   slot_i[R]    int32  slot of the batch's i-th unique node (R = max rows per batch)
//   miss_i[R]    int32  indices i of the batch's misses
//   gslot[E]     int32  slot of the src node of every last-hop edge (E = max last-hop edges)
struct CacheWs {
  WsHeader* hdr;
  int32_t* slot_of;
  int32_t* node_of;
  uint32_t* used;
  uint8_t* ref;
  unsigned long long* hand;
  unsigned long long* counters;
  int32_t* slot_i;
  int32_t* miss_i;
  int32_t* gslot;
};

inline CacheWs carve_cache_ws(void* base, int64_t n, int64_t cap, int64_t rows, int64_t edges,
                              size_t* bytes) {
  Carver c(base);
  CacheWs w;
  w.hdr = c.take<WsHeader>(1);
  w.slot_of = c.take<int32_t>(n);
  w.node_of = c.take<int32_t>(cap);
  w.used = c.take<uint32_t>(cap);
  w.ref = c.take<uint8_t>(cap);
  w.hand = c.take<unsigned long long>(1);
  w.counters = c.take<unsigned long long>(4);
  w.slot_i = c.take<int32_t>(rows);
  w.miss_i = c.take<int32_t>(rows);
  w.gslot = c.take<int32_t>(edges);
  if (bytes) *bytes = c.bytes();
  return w;
}

// lookup + insert + fill for the batch's unique nodes nodes[0:*n_rows) and the slot map of the
// last-hop edges; afterwards every node of the batch is resident (capacity >= rows).
cmb_status cache_prepare(const CacheWs& w, int64_t cap, const int32_t* nodes,
                         const int64_t* n_rows_dev, int64_t rows_cap, const int32_t* last_idx,
                         const int64_t* n_edges_dev, int64_t edges_cap, const float* host_x,
                         int64_t host_ld, int32_t feat_dim, float* cache_rows, int64_t cache_ld,
                         uint32_t batch_tag, int64_t* stats, int sms, cudaStream_t s);

}  // namespace cmb
