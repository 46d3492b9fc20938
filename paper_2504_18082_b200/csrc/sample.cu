// sample.cu -- a2 (Knob-2 biased fanout sampling) + a3 (dedup/relabel into per-hop blocks).
//
// PAPER.md S4.2 P:683-691, S5 P:717: intra-community edges get unnormalised weight p,
// inter-community edges 1-p, and DGL's NeighborSampler draws `fanout` neighbours per node
// WITHOUT replacement (reading R1).  With two weight classes that law factorises exactly:
// the class sequence of successive draws is an urn (P(intra) = wi*ri / (wi*ri + wo*ro)),
// and given K intra picks the intra (inter) subset is uniform -> Floyd's subset sampler.
// So a row costs O(f) Philox draws whatever its degree.  Alg. 1 P:541-542 then builds the
// sub-graph: the src list of hop h is the dst list followed by the new neighbours in order
// of first occurrence (readings R7, R8).
//
// B200 mapping:
//   k_count     1 thread / dst row           cnt = min(f, #eligible)     (8 B bounds + 16 B indptr)
//   scan        CUB DeviceScan                indptr_h (exclusive)
//   k_sample<G> G lanes / dst row (G = pow2 >= f): lane s owns Philox slot s; urn via
//               shuffles, Floyd membership via ballots, ascending emit via shuffle ranks
//   k_insert    1 thread / edge; __match_any_sync collapses duplicates inside a warp, the
//               leader claims the key in an open-addressing table (L2-resident, <= 50 %
//               load) and atomicMin's its edge position into the value
//   k_flag      edge e is the first occurrence of a new node <=> value == (HB | e)
//   scan        CUB DeviceScan                new local ids
//   k_relabel   1 thread / edge: local id, append node, finalise the table value
// Every size lives on the device (sizes[]), grids are capacity-bounded: no host sync.
#include <cub/cub.cuh>

#include "common.cuh"

namespace cmb {
namespace {

constexpr uint32_t kEmpty = 0xFFFFFFFFu;
constexpr uint32_t kHB = 0x80000000u;  // value = HB | first edge position (not yet relabelled)

struct Table {
  uint32_t* keys;
  uint32_t* vals;
  uint32_t mask;   // slots - 1 (slots = 2^log2)
  int shift;       // 32 - log2(slots)
};

__device__ __forceinline__ uint32_t hash_slot(uint32_t u, const Table& t) {
  return (u * 0x9E3779B1u) >> t.shift;
}

// Find-or-claim the slot of key u (linear probing).  Returns mask+1 on a full table.
__device__ __forceinline__ uint32_t probe_insert(uint32_t u, const Table& t) {
  uint32_t h = hash_slot(u, t);
  for (uint32_t i = 0; i <= t.mask; ++i) {
    const uint32_t k = __ldcg(t.keys + h);
    if (k == u) return h;
    if (k == kEmpty) {
      const uint32_t old = atomicCAS(t.keys + h, kEmpty, u);
      if (old == kEmpty || old == u) return h;
    }
    h = (h + 1) & t.mask;
  }
  return t.mask + 1;
}

// Batch start: nodes[0:n0) = roots, roots inserted with their final local id.
__global__ void k_init_roots(const int32_t* __restrict__ roots, int64_t n0, Table t,
                             int32_t* __restrict__ nodes, int64_t* __restrict__ sizes,
                             int n_sizes, int32_t* status) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n_sizes) sizes[i] = (i == 0) ? n0 : 0;
  if (i >= n0) return;
  const uint32_t u = static_cast<uint32_t>(roots[i]);
  nodes[i] = static_cast<int32_t>(u);
  uint32_t h = hash_slot(u, t);
  for (uint32_t k = 0; k <= t.mask; ++k) {
    const uint32_t old = atomicCAS(t.keys + h, kEmpty, u);
    if (old == kEmpty) {
      t.vals[h] = static_cast<uint32_t>(i);
      return;
    }
    if (old == u) {  // duplicate root: precondition violated
      raise_status(status, CMB_ERR_INVALID_INPUT);
      return;
    }
    h = (h + 1) & t.mask;
  }
  raise_status(status, CMB_ERR_CAPACITY);
}

struct RowInfo {
  int64_t rs, deg, ni_e, no_e;
  uint32_t lo, hi;
};

__device__ __forceinline__ RowInfo row_info(const DevGraph& g, int32_t v, uint32_t wi,
                                            uint32_t wo) {
  RowInfo r;
  r.rs = __ldg(g.indptr + v);
  r.deg = __ldg(g.indptr + v + 1) - r.rs;
  const uint2 b = __ldg(g.bounds + v);
  r.lo = b.x;
  r.hi = b.y;
  const int64_t ni = static_cast<int64_t>(b.y) - b.x;
  r.ni_e = wi ? ni : 0;
  r.no_e = wo ? r.deg - ni : 0;
  return r;
}

// cnt[i] = min(f, m_i) for i < n_h, 0 for n_h <= i <= cap (so the scan over cap+1 is exact)
__global__ void k_count(DevGraph g, const int32_t* __restrict__ nodes,
                        const int64_t* __restrict__ sizes, int hop, int f, uint32_t wi,
                        uint32_t wo, int64_t cap, int32_t* __restrict__ cnt) {
  const int64_t n_h = sizes[hop];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= cap;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t c = 0;
    if (i < n_h) {
      const RowInfo r = row_info(g, nodes[i], wi, wo);
      const int64_t m = r.ni_e + r.no_e;
      c = static_cast<int32_t>(m < f ? m : f);
    }
    cnt[i] = c;
  }
}

template <int G>
__global__ void __launch_bounds__(256) k_sample(DevGraph g, const int32_t* __restrict__ nodes,
                                                int64_t* __restrict__ sizes, int hop, int L,
                                                int f, uint32_t wi, uint32_t wo, uint32_t k0,
                                                uint32_t k1, uint32_t batch,
                                                const int32_t* __restrict__ indptr_h,
                                                int32_t* __restrict__ out) {
  const int64_t n_h = sizes[hop];
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid == 0) sizes[L + 1 + hop] = indptr_h[n_h];  // e_h
  const int64_t row = tid / G;
  if (row >= n_h) return;  // whole groups leave together
  const int lane = threadIdx.x & (G - 1);
  const int wl = threadIdx.x & 31;
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (wl & ~(G - 1)));

  const int32_t v = nodes[row];
  const RowInfo r = row_info(g, v, wi, wo);
  const int32_t* __restrict__ nb = g.indices + r.rs;
  int32_t* __restrict__ o = out + indptr_h[row];
  const int64_t m = r.ni_e + r.no_e;
  if (f >= m) {  // whole eligible neighbourhood (reading R4), ascending position, no RNG
    if (r.ni_e && r.no_e) {
      for (int64_t q = lane; q < r.deg; q += G) o[q] = __ldg(nb + q);
    } else if (r.ni_e) {
      for (int64_t q = lane; q < r.ni_e; q += G) o[q] = __ldg(nb + r.lo + q);
    } else {
      for (int64_t q = lane; q < r.no_e; q += G)
        o[q] = __ldg(nb + (q < r.lo ? q : r.hi + (q - r.lo)));
    }
    return;
  }
  // lane s draws W_s = Philox(s, v, (1<<24)|hop, batch)
  PhiloxOut w{0u, 0u, 0u, 0u};
  if (lane < f)
    w = philox4x32_10(static_cast<uint32_t>(lane), static_cast<uint32_t>(v),
                      (kTagSample << 24) | static_cast<uint32_t>(hop), batch, k0, k1);
  const uint64_t u01 = lo64(w), u23 = hi64(w);

  // urn: number K of intra picks among f successive weighted draws
  uint64_t ri = static_cast<uint64_t>(r.ni_e), ro = static_cast<uint64_t>(r.no_e);
  int K = 0;
  for (int s = 0; s < f; ++s) {
    const uint64_t x = __shfl_sync(gmask, u01, s, G);
    const uint64_t wri = wi * ri;
    if (__umul64hi(x, wri + wo * ro) < wri) {
      ++K;
      --ri;
    } else {
      --ro;
    }
  }
  // Floyd: lanes [0,K) draw the intra subset, lanes [K,f) the inter subset
  const bool in = lane < K;
  const uint64_t n_cls = in ? static_cast<uint64_t>(r.ni_e) : static_cast<uint64_t>(r.no_e);
  const int k_cls = in ? K : f - K;
  const int t = in ? lane : lane - K;
  const uint32_t j = static_cast<uint32_t>(n_cls - static_cast<uint64_t>(k_cls) + t);
  const uint32_t rr = static_cast<uint32_t>(__umul64hi(u23, static_cast<uint64_t>(j) + 1u));
  uint32_t sel = kEmpty;
  for (int s = 0; s < f; ++s) {
    const uint32_t rs = __shfl_sync(gmask, rr, s, G);
    const bool same_cls = (lane < K) == (s < K);
    const unsigned hit = __ballot_sync(gmask, lane < s && same_cls && sel == rs);
    if (lane == s) sel = hit ? j : rr;
  }
  uint32_t pos = in ? r.lo + sel : (sel < r.lo ? sel : r.hi + (sel - r.lo));
  if (lane >= f) pos = kEmpty;
  int rank = 0;
  for (int s = 0; s < f; ++s) rank += __shfl_sync(gmask, pos, s, G) < pos;
  if (lane < f) o[rank] = __ldg(nb + pos);
}

__global__ void k_insert(const int32_t* __restrict__ nbr, const int64_t* __restrict__ sizes,
                         int e_idx, Table t, uint32_t* __restrict__ slot_out, int32_t* status) {
  const int64_t e_h = sizes[e_idx];
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool valid = e < e_h;
  const unsigned act = __ballot_sync(0xffffffffu, valid);
  if (!valid) return;
  const uint32_t u = static_cast<uint32_t>(nbr[e]);
  const unsigned peers = __match_any_sync(act, u);
  const int leader = __ffs(peers) - 1;
  const int lane = threadIdx.x & 31;
  uint32_t slot = 0;
  if (lane == leader) {
    slot = probe_insert(u, t);
    if (slot > t.mask) {
      raise_status(status, CMB_ERR_CAPACITY);
      slot = 0;
    } else {
      const uint32_t cur = __ldcg(t.vals + slot);
      if (cur == kEmpty || (cur & kHB)) atomicMin(t.vals + slot, kHB | static_cast<uint32_t>(e));
    }
  }
  slot = __shfl_sync(peers, slot, leader);
  slot_out[e] = slot;
}

__global__ void k_flag(const int64_t* __restrict__ sizes, int e_idx, int64_t e_cap, Table t,
                       const uint32_t* __restrict__ slot, int32_t* __restrict__ flag,
                       uint32_t* __restrict__ mask_out) {
  const int64_t e_h = sizes[e_idx];
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  bool f = false;
  if (e < e_h) f = t.vals[slot[e]] == (kHB | static_cast<uint32_t>(e));
  if (e < e_cap) flag[e] = f ? 1 : 0;
  if (mask_out) {
    const unsigned word = __ballot_sync(0xffffffffu, f);
    if ((threadIdx.x & 31) == 0 && e < e_cap) mask_out[e >> 5] = word;
  }
}

__global__ void k_relabel(int64_t* __restrict__ sizes, int hop, int L, int64_t e_cap, Table t,
                          const uint32_t* __restrict__ slot, const int32_t* __restrict__ scan,
                          int32_t* __restrict__ idx, int32_t* __restrict__ nodes,
                          int32_t* __restrict__ gid_out) {
  const int64_t n_h = sizes[hop];
  const int64_t e_h = sizes[L + 1 + hop];
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e == 0) sizes[hop + 1] = n_h + (e_cap > 0 ? scan[e_cap - 1] : 0);
  if (e >= e_h) return;
  const uint32_t s = slot[e];
  const uint32_t val = __ldcg(t.vals + s);
  if (gid_out) gid_out[e] = idx[e];  // pre-relabel (global) src id, kept for the last hop
  uint32_t id;
  if (val & kHB) {
    const uint32_t ef = val & ~kHB;
    id = static_cast<uint32_t>(n_h) + static_cast<uint32_t>(scan[ef]) - 1u;
    if (ef == static_cast<uint32_t>(e)) {  // first occurrence: append + finalise the value
      nodes[id] = idx[e];
      t.vals[s] = id;
    }
  } else {
    id = val;
  }
  idx[e] = static_cast<int32_t>(id);
}

struct SampleWs {
  WsHeader* hdr;
  int32_t* cnt;
  int32_t* flag;
  int32_t* scan;
  uint32_t* slot;
  Table tab;
  size_t tab_bytes;
  void* temp;
  size_t temp_bytes;
};

SampleWs carve_sample_ws(void* base, int64_t n_roots, const int32_t* fanouts, int32_t L,
                         int64_t num_nodes, size_t* bytes) {
  int64_t n_cap[CMB_MAX_HOPS + 1], e_cap[CMB_MAX_HOPS];
  cmb_blocks_capacity(n_roots, fanouts, L, num_nodes, n_cap, e_cap);
  int64_t max_n = 0, max_e = 0;
  for (int h = 0; h < L; ++h) {
    if (n_cap[h] > max_n) max_n = n_cap[h];
    if (e_cap[h] > max_e) max_e = e_cap[h];
  }
  int log2s = 8;
  while ((int64_t(1) << log2s) < 2 * n_cap[L]) ++log2s;
  Carver c(base);
  SampleWs w;
  w.hdr = c.take<WsHeader>(1);
  w.cnt = c.take<int32_t>(static_cast<size_t>(max_n) + 1);
  w.flag = c.take<int32_t>(static_cast<size_t>(max_e) + 1);
  w.scan = c.take<int32_t>(static_cast<size_t>(max_e) + 1);
  w.slot = c.take<uint32_t>(static_cast<size_t>(max_e) + 1);
  const size_t slots = size_t(1) << log2s;
  w.tab.keys = c.take<uint32_t>(slots);
  w.tab.vals = c.take<uint32_t>(slots);
  w.tab.mask = static_cast<uint32_t>(slots - 1);
  w.tab.shift = 32 - log2s;
  w.tab_bytes = slots * 2 * sizeof(uint32_t);
  size_t a = 0, b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, a, (int32_t*)nullptr, (int32_t*)nullptr,
                                static_cast<int>(max_n + 1));
  cub::DeviceScan::InclusiveSum(nullptr, b, (int32_t*)nullptr, (int32_t*)nullptr,
                                static_cast<int>(max_e + 1));
  w.temp_bytes = a > b ? a : b;
  w.temp = c.take<char>(w.temp_bytes);
  if (bytes) *bytes = c.bytes();
  return w;
}

template <int G>
void launch_sample(int64_t n_cap, cudaStream_t s, const DevGraph& g, const int32_t* nodes,
                   int64_t* sizes, int hop, int L, int f, uint32_t wi, uint32_t wo, uint32_t k0,
                   uint32_t k1, uint32_t batch, const int32_t* indptr_h, int32_t* out) {
  const int64_t threads = n_cap * G;
  const int grid = static_cast<int>((threads + 255) / 256);
  k_sample<G><<<grid > 0 ? grid : 1, 256, 0, s>>>(g, nodes, sizes, hop, L, f, wi, wo, k0, k1,
                                                   batch, indptr_h, out);
}

}  // namespace
}  // namespace cmb

using namespace cmb;

extern "C" {

size_t cmb_sample_workspace_bytes(int64_t n_roots, const int32_t* fanouts, int32_t n_hops,
                                  int64_t num_nodes) {
  if (!fanouts || n_hops < 1 || n_hops > CMB_MAX_HOPS) return 0;
  size_t b = 0;
  carve_sample_ws(nullptr, n_roots, fanouts, n_hops, num_nodes, &b);
  return b;
}

cmb_status cmb_sample_blocks(const cmb_graph* g, const int32_t* roots, int64_t n_roots,
                             const int32_t* fanouts, int32_t n_hops, double p_intra, uint64_t seed,
                             uint32_t batch_id, cmb_blocks* out, void* workspace,
                             size_t workspace_bytes, void* stream) {
  CMB_ARG(g && roots && fanouts && out, "cmb_sample_blocks: null graph/roots/fanouts/out");
  CMB_ARG(n_hops >= 1 && n_hops <= CMB_MAX_HOPS, "cmb_sample_blocks: n_hops %d outside [1,%d]",
          n_hops, CMB_MAX_HOPS);
  CMB_ARG(n_roots >= 1 && n_roots <= g->d.n, "cmb_sample_blocks: n_roots %lld outside [1, N]",
          (long long)n_roots);
  CMB_ARG(p_intra >= 0.0 && p_intra <= 1.0, "cmb_sample_blocks: p_intra outside [0, 1]");
  for (int h = 0; h < n_hops; ++h)
    CMB_ARG(fanouts[h] >= 1 && fanouts[h] <= CMB_MAX_FANOUT,
            "cmb_sample_blocks: fanout[%d] = %d outside [1, %d]", h, fanouts[h], CMB_MAX_FANOUT);
  int64_t n_cap[CMB_MAX_HOPS + 1], e_cap[CMB_MAX_HOPS];
  cmb_blocks_capacity(n_roots, fanouts, n_hops, g->d.n, n_cap, e_cap);
  CMB_ARG(out->nodes && out->sizes, "cmb_sample_blocks: null nodes/sizes");
  if (out->nodes_cap < n_cap[n_hops]) {
    set_error("cmb_sample_blocks: nodes_cap %lld < %lld", (long long)out->nodes_cap,
              (long long)n_cap[n_hops]);
    return CMB_ERR_CAPACITY;
  }
  for (int h = 0; h < n_hops; ++h) {
    CMB_ARG(out->indptr[h] && out->indices[h], "cmb_sample_blocks: null indptr/indices[%d]", h);
    if (out->indices_cap[h] < e_cap[h]) {
      set_error("cmb_sample_blocks: indices_cap[%d] %lld < %lld", h,
                (long long)out->indices_cap[h], (long long)e_cap[h]);
      return CMB_ERR_CAPACITY;
    }
    CMB_ARG(e_cap[h] < (int64_t(1) << 31) - 1, "cmb_sample_blocks: hop %d capacity exceeds int32",
            h);
  }
  const size_t need = cmb_sample_workspace_bytes(n_roots, fanouts, n_hops, g->d.n);
  CMB_ARG(workspace && workspace_bytes >= need && (reinterpret_cast<uintptr_t>(workspace) & 255) == 0,
          "cmb_sample_blocks: workspace must be 256-B aligned and >= %zu bytes", need);

  cudaStream_t s = static_cast<cudaStream_t>(stream);
  SampleWs w = carve_sample_ws(workspace, n_roots, fanouts, n_hops, g->d.n, nullptr);
  int32_t* status = &w.hdr->status;
  const uint32_t P16 = static_cast<uint32_t>(p_intra * 65536.0 + 0.5);
  const uint32_t wi = P16, wo = 65536u - P16;
  const uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
  const int L = n_hops;

  CMB_CUDA(cudaMemsetAsync(w.tab.keys, 0xFF, w.tab_bytes, s));  // keys and vals = EMPTY
  {
    const int64_t nthr = n_roots > 2 * L + 1 ? n_roots : 2 * L + 1;
    k_init_roots<<<ceil_div(nthr, 256), 256, 0, s>>>(roots, n_roots, w.tab, out->nodes,
                                                     out->sizes, 2 * L + 1, status);
    CMB_CUDA(cudaGetLastError());
  }
  for (int h = 0; h < L; ++h) {
    const int f = fanouts[h];
    const int64_t nc = n_cap[h], ec = e_cap[h];
    k_count<<<ceil_div(nc + 1, 256), 256, 0, s>>>(g->d, out->nodes, out->sizes, h, f, wi, wo, nc,
                                                  w.cnt);
    CMB_CUDA(cudaGetLastError());
    size_t tb = w.temp_bytes;
    CMB_CUDA(cub::DeviceScan::ExclusiveSum(w.temp, tb, w.cnt, out->indptr[h],
                                           static_cast<int>(nc + 1), s));
    if (f <= 4)
      launch_sample<4>(nc, s, g->d, out->nodes, out->sizes, h, L, f, wi, wo, k0, k1, batch_id,
                       out->indptr[h], out->indices[h]);
    else if (f <= 8)
      launch_sample<8>(nc, s, g->d, out->nodes, out->sizes, h, L, f, wi, wo, k0, k1, batch_id,
                       out->indptr[h], out->indices[h]);
    else if (f <= 16)
      launch_sample<16>(nc, s, g->d, out->nodes, out->sizes, h, L, f, wi, wo, k0, k1, batch_id,
                        out->indptr[h], out->indices[h]);
    else
      launch_sample<32>(nc, s, g->d, out->nodes, out->sizes, h, L, f, wi, wo, k0, k1, batch_id,
                        out->indptr[h], out->indices[h]);
    CMB_CUDA(cudaGetLastError());
    const int eg = ceil_div(ec > 0 ? ec : 1, 256);
    k_insert<<<eg, 256, 0, s>>>(out->indices[h], out->sizes, L + 1 + h, w.tab, w.slot, status);
    CMB_CUDA(cudaGetLastError());
    uint32_t* mask = (h == L - 1) ? out->new_src_mask : nullptr;
    k_flag<<<eg, 256, 0, s>>>(out->sizes, L + 1 + h, ec, w.tab, w.slot, w.flag, mask);
    CMB_CUDA(cudaGetLastError());
    if (ec > 0) {
      tb = w.temp_bytes;
      CMB_CUDA(cub::DeviceScan::InclusiveSum(w.temp, tb, w.flag, w.scan, static_cast<int>(ec), s));
    }
    k_relabel<<<eg, 256, 0, s>>>(out->sizes, h, L, ec, w.tab, w.slot, w.scan, out->indices[h],
                                 out->nodes, h == L - 1 ? out->last_src_ids : nullptr);
    CMB_CUDA(cudaGetLastError());
  }
  return CMB_OK;
}

}  // extern "C"
