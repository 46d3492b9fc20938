// runtime.cu -- the native step executor: one C call enqueues a whole launch group (the
// multi-batch sampler launch + the fused gather/aggregate of every batch, optionally bracketed
// by caller-owned CUDA events), so a Python driver pays one foreign call per group instead of
// one per launch (host enqueue cost per group of 4 batches: ~180 us -> see DESIGN.md).
#include <cuda_runtime.h>

#include "common.cuh"

using namespace cmb;

extern "C" {

cmb_status cmb_step_group(const cmb_graph* g, const cmb_batch* batches,
                          const cmb_batch_features* feats, int32_t n_batches,
                          const int32_t* fanouts, int32_t n_hops, double p_intra, int32_t law,
                          uint64_t seed, void* const* events, void* stream) {
  CMB_NVTX("cmb.step_group");
  CMB_ARG(g && batches && feats && fanouts, "cmb_step_group: null argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto rec = [&](int i) -> cmb_status {
    if (events && events[i]) CMB_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(events[i]), s));
    return CMB_OK;
  };
  cmb_status st = rec(0);
  if (st != CMB_OK) return st;
  st = cmb_sample_blocks_multi(g, batches, n_batches, fanouts, n_hops, p_intra, law, seed, stream);
  if (st != CMB_OK) return st;
  if ((st = rec(1)) != CMB_OK) return st;
  // the a4 + a5 of every batch of the group in ONE launch (one walk over all their dst rows)
  // when every operand is 16-byte aligned (the per-batch events bracket that launch: the first
  // batch's pair spans it, the others are recorded at its end); otherwise one
  // cmb_gather_aggregate per batch (its scalar path handles unaligned rows)
  auto a16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  bool one_launch = g->d.x && a16(g->d.x) && g->d.ld % 4 == 0;
  for (int i = 0; i < n_batches && one_launch; ++i)
    one_launch = a16(feats[i].x_in) && a16(feats[i].h_out) && feats[i].x_in_ld % 4 == 0 &&
                 feats[i].h_ld % 4 == 0;
  if (one_launch) {
    if ((st = rec(2)) != CMB_OK) return st;
    const cmb_blocks* blocks[CMB_MAX_BATCHES_PER_LAUNCH];
    for (int i = 0; i < n_batches; ++i) blocks[i] = batches[i].out;
    st = cmb_gather_aggregate_multi(g, blocks, feats, n_batches, n_hops, stream);
    if (st != CMB_OK) return st;
    for (int i = 0; i < n_batches; ++i) {
      if (i > 0 && (st = rec(2 + 2 * i)) != CMB_OK) return st;
      if ((st = rec(3 + 2 * i)) != CMB_OK) return st;
    }
    return CMB_OK;
  }
  for (int i = 0; i < n_batches; ++i) {
    if ((st = rec(2 + 2 * i)) != CMB_OK) return st;
    const cmb_batch_features& f = feats[i];
    st = cmb_gather_aggregate(g, batches[i].out, n_hops, f.n_last_dst_cap, f.nodes_cap, f.x_in,
                              f.x_in_ld, f.h_out, f.h_ld, stream);
    if (st != CMB_OK) return st;
    if ((st = rec(3 + 2 * i)) != CMB_OK) return st;
  }
  return CMB_OK;
}

}  // extern "C"
