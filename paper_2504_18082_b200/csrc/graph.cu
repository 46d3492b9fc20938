// graph.cu -- a0: community offsets and per-row intra-community segments.
//
// A community-ordered graph (community c owns the id range
// [cbeg[c], cbeg[c+1])) with strictly ascending rows has, in every row v, its
// intra-community neighbours (S4.2 P:688; reading R5) in ONE contiguous
// segment [lo, hi).  Storing (lo, hi) per row (8 B/node) replaces the paper's
// per-edge probability tensor (P:717, 4 B/edge): the sampler splits a row into
// intra / inter parts with one 8-byte load and no per-edge work.
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace cmb {
namespace {

// Validation of community order (one thread per node) + community offsets.
__global__ void k_comm_offsets(const int32_t* __restrict__ comm, int64_t n, int32_t ncomm,
                               int32_t* __restrict__ cbeg, int32_t* status) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = comm[v];
    const int32_t prev = v == 0 ? -1 : comm[v - 1];
    if (c < 0 || c >= ncomm || c < prev || c > prev + 1) {
      raise_status(status, CMB_ERR_NOT_COMMUNITY_ORDERED);  // unordered, gap or out of range
      continue;
    }
    if (c != prev) cbeg[c] = static_cast<int32_t>(v);
    if (v == n - 1) {
      if (c != ncomm - 1) raise_status(status, CMB_ERR_NOT_COMMUNITY_ORDERED);
      cbeg[ncomm] = static_cast<int32_t>(n);
    }
  }
}

// indptr[0] == 0, indptr[n] == nnz, rows inside [0, nnz), strictly ascending with ids in
// [0, n): one warp per row (a row whose offsets leave [0, nnz) is flagged before any read).
__global__ void k_validate_rows(const int64_t* __restrict__ indptr,
                                const int32_t* __restrict__ indices, int64_t n, int64_t nnz,
                                int32_t* status) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  if (warp == 0 && lane == 0 && (indptr[0] != 0 || indptr[n] != nnz))
    raise_status(status, CMB_ERR_INVALID_GRAPH);
  for (int64_t v = warp; v < n; v += nwarps) {
    const int64_t rs = indptr[v], re = indptr[v + 1];
    bool bad = re < rs || rs < 0 || re > nnz;
    for (int64_t e = rs + lane; e < re && !bad; e += 32) {
      const int32_t u = indices[e];
      bad |= (u < 0) || (u >= n) || (e + 1 < re && indices[e + 1] <= u);
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) raise_status(status, CMB_ERR_INVALID_GRAPH);
  }
}

__device__ __forceinline__ int64_t lower_bound(const int32_t* __restrict__ a, int64_t lo,
                                               int64_t hi, int32_t key) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// (lo, hi) = row offsets of the first neighbour >= cbeg[c(v)] and >= cbeg[c(v)+1].
// With `rec`, also the packed row record the sampler reads instead of indptr[v], indptr[v+1]
// and bounds[v] (two or three random 32-B sectors -> one): x = row start bits 0..31,
// y = start bits 32..39 | degree << 8, z = lo, w = hi; a row of degree >= 2^24 - 1 stores the
// degree field 0xFFFFFF (read the three arrays instead).  Used when nnz < 2^40.
__global__ void k_intra_bounds(const int64_t* __restrict__ indptr,
                               const int32_t* __restrict__ indices,
                               const int32_t* __restrict__ comm, const int32_t* __restrict__ cbeg,
                               int32_t ncomm, int64_t n, uint2* __restrict__ bounds,
                               uint4* __restrict__ rec) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rs = indptr[v], re = indptr[v + 1];
    const int32_t c = min(max(comm[v], 0), ncomm - 1);  // memory-safe on unvalidated input
    const int64_t a = lower_bound(indices, rs, re, cbeg[c]);
    const int64_t b = lower_bound(indices, a, re, cbeg[c + 1]);
    bounds[v] = make_uint2(static_cast<uint32_t>(a - rs), static_cast<uint32_t>(b - rs));
    if (rec) {
      const uint64_t deg = static_cast<uint64_t>(re - rs);
      const uint32_t df = deg < kRecDegSlow ? static_cast<uint32_t>(deg) : kRecDegSlow;
      rec[v] = make_uint4(static_cast<uint32_t>(rs),
                          (static_cast<uint32_t>(static_cast<uint64_t>(rs) >> 32) & 0xFFu) | (df << 8),
                          static_cast<uint32_t>(a - rs), static_cast<uint32_t>(b - rs));
    }
  }
}

struct GraphWs {
  WsHeader* hdr;
  int32_t* cbeg;
  uint2* bounds;
  uint4* rec;
};

GraphWs carve_graph_ws(void* base, int64_t n, int32_t ncomm, size_t* bytes) {
  Carver c(base);
  GraphWs w;
  w.hdr = c.take<WsHeader>(1);
  w.cbeg = c.take<int32_t>(static_cast<size_t>(ncomm) + 1);
  w.bounds = c.take<uint2>(static_cast<size_t>(n));
  w.rec = c.take<uint4>(static_cast<size_t>(n));
  if (bytes) *bytes = c.bytes();
  return w;
}

}  // namespace
}  // namespace cmb

using namespace cmb;

extern "C" {

size_t cmb_graph_workspace_bytes(int64_t num_nodes, int32_t num_communities) {
  size_t b = 0;
  carve_graph_ws(nullptr, num_nodes, num_communities, &b);
  return b;
}

cmb_status cmb_load_graph(const cmb_graph_desc* d, void* stream, cmb_graph** out) {
  CMB_NVTX("cmb.a0.load_graph");
  CMB_ARG(d != nullptr && out != nullptr, "cmb_load_graph: null desc/out");
  *out = nullptr;
  CMB_ARG(d->num_nodes > 0 && d->num_nodes < (int64_t(1) << 31),
          "cmb_load_graph: num_nodes %lld outside [1, 2^31)", (long long)d->num_nodes);
  CMB_ARG(d->num_edges >= 0, "cmb_load_graph: negative num_edges");
  CMB_ARG(d->indptr && (d->indices || d->num_edges == 0) && d->community,
          "cmb_load_graph: null indptr/indices/community");
  CMB_ARG(d->num_communities >= 1 && d->num_communities <= d->num_nodes,
          "cmb_load_graph: num_communities %d outside [1, N]", d->num_communities);
  if (d->features) {
    CMB_ARG(d->feat_dim >= 1 && d->feat_ld >= d->feat_dim,
            "cmb_load_graph: feat_dim %d / feat_ld %lld invalid", d->feat_dim,
            (long long)d->feat_ld);
  }
  size_t need = cmb_graph_workspace_bytes(d->num_nodes, d->num_communities);
  CMB_ARG(d->workspace && d->workspace_bytes >= need &&
              (reinterpret_cast<uintptr_t>(d->workspace) & 255) == 0,
          "cmb_load_graph: workspace must be 256-B aligned and >= %zu bytes", need);
  cmb_status st = require_sm100();
  if (st != CMB_OK) return st;

  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool use_rec = d->num_edges < (int64_t(1) << 40);  // the record's 40-bit row start
  GraphWs w = carve_graph_ws(d->workspace, d->num_nodes, d->num_communities, nullptr);
  CMB_CUDA(cudaMemsetAsync(w.hdr, 0, sizeof(WsHeader), s));
  int dev = 0, sms = 148;
  CMB_CUDA(cudaGetDevice(&dev));
  CMB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int grid = sms * 8;
  k_comm_offsets<<<grid, 256, 0, s>>>(d->community, d->num_nodes, d->num_communities, w.cbeg,
                                      &w.hdr->status);
  CMB_CUDA(cudaGetLastError());
  if (d->validate) {
    k_validate_rows<<<grid, 256, 0, s>>>(d->indptr, d->indices, d->num_nodes, d->num_edges,
                                         &w.hdr->status);
    CMB_CUDA(cudaGetLastError());
    int32_t hs = 0;
    CMB_CUDA(cudaMemcpyAsync(&hs, &w.hdr->status, 4, cudaMemcpyDeviceToHost, s));
    CMB_CUDA(cudaStreamSynchronize(s));
    if (hs != 0) {
      set_error("cmb_load_graph: device validation failed (%s)",
                cmb_status_string(static_cast<cmb_status>(hs)));
      return static_cast<cmb_status>(hs);
    }
  }
  k_intra_bounds<<<grid, 256, 0, s>>>(d->indptr, d->indices, d->community, w.cbeg,
                                      d->num_communities, d->num_nodes,
                                      w.bounds, use_rec ? w.rec : nullptr);
  CMB_CUDA(cudaGetLastError());

  // 64-byte aligned (the embedded CUtensorMap requires it)
  const size_t gbytes = (sizeof(cmb_graph) + 63) / 64 * 64;
  cmb_graph* g = static_cast<cmb_graph*>(std::aligned_alloc(64, gbytes));
  if (g) std::memset(static_cast<void*>(g), 0, gbytes);
  if (!g) {
    set_error("cmb_load_graph: out of host memory");
    return CMB_ERR_INVALID_ARGUMENT;
  }
  g->d.n = d->num_nodes;
  g->d.nnz = d->num_edges;
  g->d.indptr = d->indptr;
  g->d.indices = d->indices;
  g->d.comm = d->community;
  g->d.ncomm = d->num_communities;
  g->d.cbeg = w.cbeg;
  g->d.bounds = w.bounds;
  g->d.rec = use_rec ? w.rec : nullptr;
  g->d.x = d->features;
  g->d.f = d->features ? d->feat_dim : 0;
  g->d.ld = d->features ? d->feat_ld : 0;
  g->status = &w.hdr->status;
  g->device = dev;
  g->num_sms = sms;
  *out = g;
  return CMB_OK;
}

cmb_status cmb_free_graph(cmb_graph* g) {
  std::free(g);
  return CMB_OK;
}

cmb_status cmb_graph_arrays(const cmb_graph* g, const int32_t** cbeg, const uint32_t** bounds) {
  CMB_ARG(g != nullptr, "cmb_graph_arrays: null graph");
  if (cbeg) *cbeg = g->d.cbeg;
  if (bounds) *bounds = reinterpret_cast<const uint32_t*>(g->d.bounds);
  return CMB_OK;
}

}  // extern "C"
