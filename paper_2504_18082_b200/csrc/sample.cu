// sample.cu -- a2 (Knob-2 biased fanout sampling) + a3 (dedup/relabel into per-hop blocks):
// host side of cmb_sample_blocks.  The device schedule is the persistent cooperative kernel
// of sample_persist.cuh (one launch per batch, all hops, grid barriers between phases).
#include <cub/cub.cuh>

#include "sample_dev.cuh"
#include "sample_persist.cuh"

namespace cmb {
namespace {

constexpr int kMaxPersistBlocks = pst::kMaxBlocks;

// Workspace layout (all 256-B aligned).  The caller zero-initialises it once: the status word,
// the grid-barrier words, the tagged block aggregates, the tag counter, the tagged dedup map and
// the dst-order buckets start at zero and the kernel leaves them consistent after every batch
// (the barrier's arrival count returns to 0, aggregates and map entries are tagged by batch, the
// buckets are cleared after use) -- no per-batch memset.  A workspace belongs to one graph.
struct SampleWs {
  WsHeader* hdr;
  unsigned* bar;             // grid barrier {arrivals, generation}
  unsigned long long* pub;   // [3][kMaxPersistBlocks] tagged block aggregates / bases
  uint32_t* hist;            // [kOrderBuckets] dst rows of hop L-1 per node-id bucket
  uint64_t* prof;            // [kMaxPersistBlocks][64] sub-step timeline
  unsigned* tag_ctr;         // [2] batches sampled with this workspace, map width of the last
  void* map;                 // [N] tagged dedup map: 32-bit words, or 64-bit (wide_map)
  uint32_t* scan;            // [max e_cap]
  uint32_t* rank;            // [n_cap[L-1]] last-hop dst rows' ranks in their order buckets
};

// A batch needs 64-bit map words when one of its local ids or edge positions may reach 2^24
// (the 32-bit word's value field; sample_persist.cuh MapWord).
bool wide_map(int64_t n_roots, const int32_t* fanouts, int32_t L, int64_t num_nodes) {
  int64_t n_cap[CMB_MAX_HOPS + 1], e_cap[CMB_MAX_HOPS];
  cmb_blocks_capacity(n_roots, fanouts, L, num_nodes, n_cap, e_cap);
  bool wide = n_cap[L] > static_cast<int64_t>(pst::MapWord<uint32_t>::kVal);
  for (int h = 0; h < L; ++h) wide |= e_cap[h] > static_cast<int64_t>(pst::MapWord<uint32_t>::kVal);
  return wide;
}

SampleWs carve_sample_ws(void* base, int64_t n_roots, const int32_t* fanouts, int32_t L,
                         int64_t num_nodes, bool wide, size_t* bytes) {
  int64_t n_cap[CMB_MAX_HOPS + 1], e_cap[CMB_MAX_HOPS];
  cmb_blocks_capacity(n_roots, fanouts, L, num_nodes, n_cap, e_cap);
  int64_t max_e = 0;
  for (int h = 0; h < L; ++h)
    if (e_cap[h] > max_e) max_e = e_cap[h];
  Carver c(base);
  SampleWs w;
  w.hdr = c.take<WsHeader>(1);
  w.bar = c.take<unsigned>(64);
  // [3][kMaxPersistBlocks]: count and flag aggregates, then the last hop's block bases
  w.pub = c.take<unsigned long long>(3 * kMaxPersistBlocks);  // follows bar contiguously
  w.hist = c.take<uint32_t>(pst::kOrderBuckets);
  w.prof = c.take<uint64_t>(static_cast<size_t>(kMaxPersistBlocks) * 64);
  w.tag_ctr = c.take<unsigned>(2);  // {batch counter, map width of the last batch}
  if (wide)
    w.map = c.take<unsigned long long>(static_cast<size_t>(num_nodes));
  else
    w.map = c.take<unsigned>(static_cast<size_t>(num_nodes));
  w.scan = c.take<uint32_t>(static_cast<size_t>(max_e) + 1);
  w.rank = c.take<uint32_t>(static_cast<size_t>(n_cap[L - 1]) + 1);
  if (bytes) *bytes = c.bytes();
  return w;
}

void fill_args(pst::PArgs& a, const cmb_graph* g, const int32_t* roots, int64_t n_roots,
               const int32_t* fanouts, int L, uint32_t wi, uint32_t wo, uint32_t k0, uint32_t k1,
               uint32_t batch_id, const cmb_blocks* out, const SampleWs& w, int law) {
  a.g = g->d;
  a.roots = roots;
  a.n_roots = n_roots;
  a.L = L;
  for (int h = 0; h < CMB_MAX_HOPS; ++h) {
    a.fan[h] = h < L ? fanouts[h] : 0;
    a.indptr[h] = h < L ? out->indptr[h] : nullptr;
    a.indices[h] = h < L ? out->indices[h] : nullptr;
  }
  a.wi = wi;
  a.wo = wo;
  a.k0 = k0;
  a.k1 = k1;
  a.batch = batch_id;
  a.nodes = out->nodes;
  a.mask = out->new_src_mask;
  a.last_src = out->last_src_ids;
  a.sizes = out->sizes;
  a.map = w.map;
  a.tag_ctr = w.tag_ctr;
  a.scan = w.scan;
  a.rank = w.rank;
  a.pub = w.pub;
  a.bar = w.bar;
  a.prof = w.prof;
  a.hist = w.hist;
  a.order = out->dst_order;
  int bits = 0;
  while ((int64_t{1} << bits) < g->d.n) ++bits;
  a.order_shift = bits > pst::kOrderBits ? bits - pst::kOrderBits : 0;
  a.status = &w.hdr->status;
  a.law = law;
}

// One 1024-thread block per SM (64 registers: the whole register file), co-resident by
// construction.  (One 512-thread block per SM measured 101 vs 78 us per batch; TWO 512-thread
// blocks per SM, of different batches -- CMB_SAMPLER_PB = 512, a layout experiment -- 172 vs
// 164 us per step at 6 batches per launch.)
#ifndef CMB_SAMPLER_PB
#define CMB_SAMPLER_PB 1024
#endif
cmb_status launch_persistent(const cmb_graph* g, pst::PMulti& m, bool wide, cudaStream_t s) {
  constexpr int kPB = CMB_SAMPLER_PB;
  int grid = g->num_sms * (1024 / kPB);
  if (grid > kMaxPersistBlocks) grid = kMaxPersistBlocks;
  grid -= grid % m.nb;    // equal virtual grids per batch
  void* args[] = {&m};
  const void* fn = wide ? reinterpret_cast<const void*>(&pst::k_sample_persistent<kPB, uint64_t>)
                        : reinterpret_cast<const void*>(&pst::k_sample_persistent<kPB, uint32_t>);
  const size_t smem = pst::smem_bytes<kPB>();
  CMB_SMEM(fn, smem);
  CMB_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kPB), args, smem, s));
  return CMB_OK;
}

// host-checkable validation of one batch (capacities, workspace)
cmb_status check_batch(const cmb_graph* g, const int32_t* roots, int64_t n_roots,
                       const int32_t* fanouts, int n_hops, const cmb_blocks* out,
                       const void* workspace, size_t workspace_bytes, bool wide) {
  CMB_ARG(roots && out, "cmb_sample_blocks: null roots/out");
  CMB_ARG(n_roots >= 1 && n_roots <= g->d.n, "cmb_sample_blocks: n_roots %lld outside [1, N]",
          (long long)n_roots);
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
  size_t need = 0;  // the launch's map width (wide if any batch of it needs 64-bit words)
  carve_sample_ws(nullptr, n_roots, fanouts, n_hops, g->d.n, wide, &need);
  CMB_ARG(workspace && workspace_bytes >= need && (reinterpret_cast<uintptr_t>(workspace) & 255) == 0,
          "cmb_sample_blocks: workspace must be 256-B aligned and >= %zu bytes", need);
  return CMB_OK;
}

}  // namespace
}  // namespace cmb

using namespace cmb;

extern "C" {

size_t cmb_sample_workspace_bytes(int64_t n_roots, const int32_t* fanouts, int32_t n_hops,
                                  int64_t num_nodes) {
  if (!fanouts || n_hops < 1 || n_hops > CMB_MAX_HOPS) return 0;
  size_t b = 0;
  carve_sample_ws(nullptr, n_roots, fanouts, n_hops, num_nodes,
                  wide_map(n_roots, fanouts, n_hops, num_nodes), &b);
  return b;
}

cmb_status cmb_sample_blocks_multi(const cmb_graph* g, const cmb_batch* batches,
                                   int32_t n_batches, const int32_t* fanouts, int32_t n_hops,
                                   double p_intra, int32_t law, uint64_t seed, void* stream) {
  CMB_NVTX("cmb.a2a3.sample_relabel");
  CMB_ARG(g && batches && fanouts, "cmb_sample_blocks: null graph/batches/fanouts");
  CMB_ARG(n_batches >= 1 && n_batches <= CMB_MAX_BATCHES_PER_LAUNCH,
          "cmb_sample_blocks_multi: n_batches %d outside [1, %d]", n_batches,
          CMB_MAX_BATCHES_PER_LAUNCH);
  CMB_ARG(n_hops >= 1 && n_hops <= CMB_MAX_HOPS, "cmb_sample_blocks: n_hops %d outside [1,%d]",
          n_hops, CMB_MAX_HOPS);
  CMB_ARG(p_intra >= 0.0 && p_intra <= 1.0, "cmb_sample_blocks: p_intra outside [0, 1]");
  CMB_ARG(law == CMB_LAW_A || law == CMB_LAW_SLOT, "cmb_sample_blocks: unknown law %d", law);
  for (int h = 0; h < n_hops; ++h)
    CMB_ARG(fanouts[h] >= 1 && fanouts[h] <= CMB_MAX_FANOUT,
            "cmb_sample_blocks: fanout[%d] = %d outside [1, %d]", h, fanouts[h], CMB_MAX_FANOUT);
  bool wide = false;
  for (int i = 0; i < n_batches; ++i)
    wide |= wide_map(batches[i].n_roots, fanouts, n_hops, g->d.n);
  for (int i = 0; i < n_batches; ++i) {
    const cmb_status st = check_batch(g, batches[i].roots, batches[i].n_roots, fanouts, n_hops,
                                      batches[i].out, batches[i].workspace,
                                      batches[i].workspace_bytes, wide);
    if (st != CMB_OK) return st;
    for (int j = 0; j < i; ++j)
      CMB_ARG(batches[j].workspace != batches[i].workspace,
              "cmb_sample_blocks_multi: batches %d and %d share a workspace", j, i);
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint32_t P16 = static_cast<uint32_t>(p_intra * 65536.0 + 0.5);
  const uint32_t wi = P16, wo = 65536u - P16;
  const uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
  pst::PMulti m;
  m.nb = n_batches;
  for (int i = 0; i < n_batches; ++i) {
    const cmb_batch& b = batches[i];
    SampleWs w = carve_sample_ws(b.workspace, b.n_roots, fanouts, n_hops, g->d.n, wide, nullptr);
    fill_args(m.a[i], g, b.roots, b.n_roots, fanouts, n_hops, wi, wo, k0, k1, b.batch_id, b.out,
              w, law);
  }
  return launch_persistent(g, m, wide, s);
}

cmb_status cmb_sample_blocks(const cmb_graph* g, const int32_t* roots, int64_t n_roots,
                             const int32_t* fanouts, int32_t n_hops, double p_intra, uint64_t seed,
                             uint32_t batch_id, cmb_blocks* out, void* workspace,
                             size_t workspace_bytes, void* stream) {
  CMB_ARG(g && roots && fanouts && out, "cmb_sample_blocks: null graph/roots/fanouts/out");
  cmb_batch b{roots, n_roots, batch_id, out, workspace, workspace_bytes};
  return cmb_sample_blocks_multi(g, &b, 1, fanouts, n_hops, p_intra, CMB_LAW_A, seed, stream);
}

cmb_status cmb_sample_blocks_law(const cmb_graph* g, const int32_t* roots, int64_t n_roots,
                                 const int32_t* fanouts, int32_t n_hops, double p_intra,
                                 int32_t law, uint64_t seed, uint32_t batch_id, cmb_blocks* out,
                                 void* workspace, size_t workspace_bytes, void* stream) {
  CMB_ARG(g && roots && fanouts && out, "cmb_sample_blocks: null graph/roots/fanouts/out");
  cmb_batch b{roots, n_roots, batch_id, out, workspace, workspace_bytes};
  return cmb_sample_blocks_multi(g, &b, 1, fanouts, n_hops, p_intra, law, seed, stream);
}

}  // extern "C"
