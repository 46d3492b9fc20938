// shard.cu -- a6: the row-sharded input-feature exchange (papers100M-scale tables; north_star:
// "the feature table is row-sharded, with an NCCL all-to-all over NVLink for remote rows").
//
// Rank r of W owns feature rows [r*S, min(N, (r+1)*S)), S = rows_per_shard.  For a batch's input
// nodes nodes[0:U) the exchange is
//   plan     stable bucketing of nodes by owner = id / S: send_ids (owner-major, original order
//            inside an owner), perm (position in X_in of every send slot), counts[W]
//   (NCCL)   all-to-all of counts, then of ids          -- torch.distributed, host side
//   gather   every rank gathers the requested rows from its shard (cmb_gather_rows)
//   (NCCL)   all-to-all of the rows back
//   scatter  X_in[perm[k]] = received row k              (cmb_scatter_rows)
// so X_in is byte-identical to the replicated gather (oracle O5).
#include <cub/cub.cuh>

#include "common.cuh"

namespace cmb {
namespace {

__global__ void k_owner_keys(const int32_t* __restrict__ nodes, const int64_t* __restrict__ n_dev,
                             int64_t n_cap, int64_t rows_per_shard, int32_t world,
                             uint32_t* __restrict__ keys, int32_t* __restrict__ pos,
                             unsigned long long* __restrict__ counts, int32_t* status) {
  const int64_t n = min(*n_dev, n_cap);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_cap;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t k = static_cast<uint32_t>(world);  // padding slots sort last
    if (i < n) {
      const int64_t o = nodes[i] / rows_per_shard;
      if (o < 0 || o >= world) {
        raise_status(status, CMB_ERR_INVALID_INPUT);
      } else {
        k = static_cast<uint32_t>(o);
        atomicAdd(counts + o, 1ull);
      }
    }
    keys[i] = k;
    pos[i] = static_cast<int32_t>(i);
  }
}

__global__ void k_send_ids(const int32_t* __restrict__ nodes, const int32_t* __restrict__ perm,
                           const int64_t* __restrict__ n_dev, int64_t n_cap,
                           int32_t* __restrict__ send_ids) {
  const int64_t n = min(*n_dev, n_cap);
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    send_ids[k] = nodes[perm[k]];
}

// out[perm[k]] = rows[k] for k < n (float4 lanes when aligned)
__global__ void k_scatter_rows(const float* __restrict__ rows, int64_t rows_ld,
                               const int32_t* __restrict__ perm, const int64_t* __restrict__ n_dev,
                               int64_t n_cap, int f, float* __restrict__ out, int64_t out_ld,
                               int vec) {
  const int64_t n = min(*n_dev, n_cap);
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t k = w0; k < n; k += nw) {
    const int64_t dst = perm[k];
    if (vec) {
      const float4* s = reinterpret_cast<const float4*>(rows + k * rows_ld);
      float4* d = reinterpret_cast<float4*>(out + dst * out_ld);
      for (int c = lane; c < (f + 3) / 4; c += 32) d[c] = s[c];
    } else {
      for (int c = lane; c < f; c += 32) out[dst * out_ld + c] = rows[k * rows_ld + c];
    }
  }
}

struct PlanWs {
  WsHeader* hdr;
  uint32_t* keys;
  uint32_t* keys_out;
  int32_t* pos;
  void* temp;
  size_t temp_bytes;
};

PlanWs carve_plan_ws(void* base, int64_t n_cap, size_t* bytes) {
  Carver c(base);
  PlanWs w;
  w.hdr = c.take<WsHeader>(1);
  w.keys = c.take<uint32_t>(static_cast<size_t>(n_cap) + 1);
  w.keys_out = c.take<uint32_t>(static_cast<size_t>(n_cap) + 1);
  w.pos = c.take<int32_t>(static_cast<size_t>(n_cap) + 1);
  size_t t = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (int32_t*)nullptr, (int32_t*)nullptr,
                                  static_cast<int>(n_cap > 0 ? n_cap : 1));
  w.temp_bytes = t;
  w.temp = c.take<char>(t);
  if (bytes) *bytes = c.bytes();
  return w;
}

int bits_for_world(int32_t world) {
  int b = 1;
  while ((1 << b) <= world) ++b;  // keys in [0, world] (world = padding)
  return b;
}

}  // namespace
}  // namespace cmb

using namespace cmb;

extern "C" {

size_t cmb_shard_plan_workspace_bytes(int64_t n_cap) {
  size_t b = 0;
  carve_plan_ws(nullptr, n_cap, &b);
  return b;
}

cmb_status cmb_shard_plan(const int32_t* nodes, const int64_t* n_dev, int64_t n_cap,
                          int64_t rows_per_shard, int32_t world, int64_t* counts,
                          int32_t* send_ids, int32_t* perm, void* workspace,
                          size_t workspace_bytes, void* stream) {
  CMB_NVTX("cmb.a6.shard_plan");
  CMB_ARG(nodes && n_dev && counts && send_ids && perm, "cmb_shard_plan: null argument");
  CMB_ARG(n_cap >= 1 && n_cap < (int64_t(1) << 31), "cmb_shard_plan: n_cap outside [1, 2^31)");
  CMB_ARG(world >= 1 && world <= 1024 && rows_per_shard >= 1,
          "cmb_shard_plan: world %d / rows_per_shard %lld invalid", world,
          (long long)rows_per_shard);
  const size_t need = cmb_shard_plan_workspace_bytes(n_cap);
  CMB_ARG(workspace && workspace_bytes >= need && (reinterpret_cast<uintptr_t>(workspace) & 255) == 0,
          "cmb_shard_plan: workspace must be 256-B aligned and >= %zu bytes", need);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  PlanWs w = carve_plan_ws(workspace, n_cap, nullptr);
  int dev = 0, sms = 148;
  CMB_CUDA(cudaGetDevice(&dev));
  CMB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CMB_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * world, s));
  k_owner_keys<<<sms * 4, 256, 0, s>>>(nodes, n_dev, n_cap, rows_per_shard, world, w.keys, w.pos,
                                       reinterpret_cast<unsigned long long*>(counts),
                                       &w.hdr->status);
  CMB_CUDA(cudaGetLastError());
  size_t tb = w.temp_bytes;
  // stable LSD radix sort on the owner (a few bits): owner-major, original order inside
  CMB_CUDA(cub::DeviceRadixSort::SortPairs(w.temp, tb, w.keys, w.keys_out, w.pos, perm,
                                           static_cast<int>(n_cap), 0, bits_for_world(world), s));
  k_send_ids<<<sms * 4, 256, 0, s>>>(nodes, perm, n_dev, n_cap, send_ids);
  CMB_CUDA(cudaGetLastError());
  return CMB_OK;
}

cmb_status cmb_gather_rows(const float* x, int64_t ld, int64_t row0, int32_t feat_dim,
                           const int32_t* ids, const int64_t* n_dev, int64_t n_cap, float* out,
                           int64_t out_ld, void* stream);

cmb_status cmb_scatter_rows(const float* rows, int64_t rows_ld, const int32_t* perm,
                            const int64_t* n_dev, int64_t n_cap, int32_t feat_dim, float* out,
                            int64_t out_ld, void* stream) {
  CMB_NVTX("cmb.a6.scatter_rows");
  CMB_ARG(rows && perm && n_dev && out, "cmb_scatter_rows: null argument");
  CMB_ARG(feat_dim >= 1 && rows_ld >= feat_dim && out_ld >= feat_dim && n_cap >= 0,
          "cmb_scatter_rows: bad feat_dim / ld / n_cap");
  if (n_cap == 0) return CMB_OK;
  int dev = 0, sms = 148;
  CMB_CUDA(cudaGetDevice(&dev));
  CMB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int vec = ((reinterpret_cast<uintptr_t>(rows) | reinterpret_cast<uintptr_t>(out)) & 15) == 0 &&
                  rows_ld % 4 == 0 && out_ld % 4 == 0 && rows_ld >= (feat_dim + 3) / 4 * 4 &&
                  out_ld >= (feat_dim + 3) / 4 * 4;
  k_scatter_rows<<<sms * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      rows, rows_ld, perm, n_dev, n_cap, feat_dim, out, out_ld, vec);
  CMB_CUDA(cudaGetLastError());
  return CMB_OK;
}

}  // extern "C"
