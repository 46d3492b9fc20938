// cache.cu -- NEXT-3: an HBM software cache of feature rows over a host-resident (pinned,
// UVA-mapped) feature table, the paper's second setting (S6.5.1: DGL's GPU cache of
// 4M node features with LRU replacement in front of UVA transfers).  Per batch:
//   lookup   every unique node of the batch: hit if its directory entry is live; hits mark
//            their slot used by this batch (protected) and referenced (CLOCK bit)
//   insert   every miss claims a victim slot with the CLOCK hand -- skip slots used by this
//            batch, give referenced slots a second chance -- and takes over its directory entry
//   fill     the missed rows are copied from host memory (zero-copy UVA loads over the host
//            link) into their slots, one warp per row
//   gslot    slot of the src node of every last-hop edge, so the fused gather+aggregate reads
//            every row from HBM
// Hits and misses are a pure function of the cache state; the choice of victims depends on the
// order of the atomic hand increments (not deterministic), the gathered bytes never do.
#include <cuda_runtime.h>

#include <cstring>

#include "cache.cuh"

namespace cmb {
namespace {

__global__ void k_cache_reset(int32_t* slot_of, int64_t n, int32_t* node_of, uint32_t* used,
                              uint8_t* ref, int64_t cap, unsigned long long* hand) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = t; i < n; i += st) slot_of[i] = -1;
  for (int64_t i = t; i < cap; i += st) {
    node_of[i] = -1;
    used[i] = 0xFFFFFFFFu;
    ref[i] = 0;
  }
  if (t == 0) *hand = 0;
}

__global__ void k_cache_lookup(const int32_t* __restrict__ nodes, const int64_t* n_rows_dev,
                               int64_t rows_cap, const int32_t* __restrict__ slot_of,
                               const int32_t* __restrict__ node_of, uint32_t* used, uint8_t* ref,
                               uint32_t tag, int32_t* slot_i, int32_t* miss_i,
                               unsigned long long* counters) {
  const int64_t n = min(*n_rows_dev, rows_cap);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = nodes[i];
    const int32_t s = slot_of[v];
    if (s >= 0 && node_of[s] == v) {
      used[s] = tag;
      ref[s] = 1;
      slot_i[i] = s;
    } else {
      const unsigned long long k = atomicAdd(counters, 1ull);
      miss_i[k] = static_cast<int32_t>(i);
    }
  }
}

__global__ void k_cache_insert(const int32_t* __restrict__ nodes, int64_t cap,
                               int32_t* slot_of, int32_t* node_of, uint32_t* used, uint8_t* ref,
                               unsigned long long* hand, uint32_t tag,
                               const int32_t* __restrict__ miss_i, int32_t* slot_i,
                               const unsigned long long* counters) {
  const int64_t nm = static_cast<int64_t>(*counters);
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nm;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t i = miss_i[k];
    const int32_t v = nodes[i];
    int64_t t;
    for (;;) {  // CLOCK: capacity >= rows per batch, so a victim always exists
      t = static_cast<int64_t>(atomicAdd(hand, 1ull) % static_cast<unsigned long long>(cap));
      const uint32_t u = used[t];
      if (u == tag) continue;                  // referenced (or just claimed) by this batch
      if (ref[t]) {                            // second chance
        ref[t] = 0;
        continue;
      }
      if (atomicCAS(&used[t], u, tag) == u) break;  // claimed
    }
    const int32_t old = node_of[t];
    if (old >= 0 && slot_of[old] == static_cast<int32_t>(t)) slot_of[old] = -1;
    node_of[t] = v;
    slot_of[v] = static_cast<int32_t>(t);
    ref[t] = 1;
    slot_i[i] = static_cast<int32_t>(t);
  }
}

// one warp per missed row: host (UVA) -> cache slot
__global__ void k_cache_fill(const int32_t* __restrict__ nodes, const int32_t* __restrict__ miss_i,
                             const int32_t* __restrict__ slot_i,
                             const unsigned long long* counters, const float* __restrict__ host_x,
                             int64_t host_ld, int32_t feat_dim, float* cache_rows,
                             int64_t cache_ld) {
  const int64_t nm = static_cast<int64_t>(*counters);
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool vec = (host_ld % 4 == 0) && (cache_ld % 4 == 0) && (feat_dim % 4 == 0);
  for (int64_t k = w0; k < nm; k += nw) {
    const int32_t i = miss_i[k];
    const float* src = host_x + static_cast<int64_t>(nodes[i]) * host_ld;
    float* dst = cache_rows + static_cast<int64_t>(slot_i[i]) * cache_ld;
    if (vec) {
      for (int c = lane; c < feat_dim / 4; c += 32)
        reinterpret_cast<float4*>(dst)[c] = reinterpret_cast<const float4*>(src)[c];
    } else {
      for (int c = lane; c < feat_dim; c += 32) dst[c] = src[c];
    }
  }
}

__global__ void k_cache_edge_slots(const int32_t* __restrict__ idx, const int64_t* n_edges_dev,
                                   int64_t edges_cap, const int32_t* __restrict__ slot_i,
                                   int32_t* gslot, const int64_t* n_rows_dev,
                                   const unsigned long long* counters, int64_t* stats) {
  const int64_t n = min(*n_edges_dev, edges_cap);
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int64_t e = t; e < n; e += (int64_t)gridDim.x * blockDim.x) gslot[e] = slot_i[idx[e]];
  if (t == 0 && stats) {
    stats[0] += *n_rows_dev;
    stats[1] += static_cast<int64_t>(*counters);
  }
}

}  // namespace

cmb_status cache_prepare(const CacheWs& w, int64_t cap, const int32_t* nodes,
                         const int64_t* n_rows_dev, int64_t rows_cap, const int32_t* last_idx,
                         const int64_t* n_edges_dev, int64_t edges_cap, const float* host_x,
                         int64_t host_ld, int32_t feat_dim, float* cache_rows, int64_t cache_ld,
                         uint32_t batch_tag, int64_t* stats, int sms, cudaStream_t s) {
  const int grid = sms * 4, blk = 256;
  CMB_CUDA(cudaMemsetAsync(w.counters, 0, sizeof(unsigned long long), s));
  k_cache_lookup<<<grid, blk, 0, s>>>(nodes, n_rows_dev, rows_cap, w.slot_of, w.node_of, w.used,
                                      w.ref, batch_tag, w.slot_i, w.miss_i, w.counters);
  k_cache_insert<<<grid, blk, 0, s>>>(nodes, cap, w.slot_of, w.node_of, w.used, w.ref, w.hand,
                                      batch_tag, w.miss_i, w.slot_i, w.counters);
  k_cache_fill<<<sms * 8, blk, 0, s>>>(nodes, w.miss_i, w.slot_i, w.counters, host_x, host_ld,
                                       feat_dim, cache_rows, cache_ld);
  k_cache_edge_slots<<<grid, blk, 0, s>>>(last_idx, n_edges_dev, edges_cap, w.slot_i, w.gslot,
                                          n_rows_dev, w.counters, stats);
  CMB_CUDA(cudaGetLastError());
  return CMB_OK;
}

}  // namespace cmb

using namespace cmb;

extern "C" {

size_t cmb_feature_cache_bytes(int64_t num_nodes, int64_t capacity, int64_t max_rows,
                               int64_t max_edges) {
  size_t b = 0;
  carve_cache_ws(nullptr, num_nodes, capacity, max_rows, max_edges, &b);
  return b;
}

cmb_status cmb_feature_cache_init(void* workspace, size_t workspace_bytes, int64_t num_nodes,
                                  int64_t capacity, int64_t max_rows, int64_t max_edges,
                                  void* stream) {
  CMB_ARG(workspace && (reinterpret_cast<uintptr_t>(workspace) & 255) == 0,
          "cmb_feature_cache_init: workspace must be 256-B aligned");
  CMB_ARG(num_nodes >= 1 && capacity >= max_rows && max_rows >= 1 && capacity <= INT32_MAX,
          "cmb_feature_cache_init: need 1 <= max_rows <= capacity");
  const size_t need = cmb_feature_cache_bytes(num_nodes, capacity, max_rows, max_edges);
  CMB_ARG(workspace_bytes >= need, "cmb_feature_cache_init: workspace < %zu bytes", need);
  CacheWs w = carve_cache_ws(workspace, num_nodes, capacity, max_rows, max_edges, nullptr);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CMB_CUDA(cudaMemsetAsync(w.hdr, 0, sizeof(WsHeader), s));
  k_cache_reset<<<1184, 256, 0, s>>>(w.slot_of, num_nodes, w.node_of, w.used, w.ref, capacity,
                                     w.hand);
  CMB_CUDA(cudaGetLastError());
  return CMB_OK;
}

}  // extern "C"
