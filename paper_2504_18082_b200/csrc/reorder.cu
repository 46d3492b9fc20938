// reorder.cu -- NEXT-2 (iii): community reordering of a graph that is not community-ordered
// (reading R25).  New order = nodes sorted by (community, old id) (stable LSD radix sort of the
// community keys over an iota); rows are copied through inv (one warp per row) and re-sorted
// with a segmented sort; the community array is permuted.  B200 mapping: CUB sorts / scans and
// three bandwidth-bound elementwise kernels; the whole CSR moves once.  CUB's segmented sort
// counts items in int, so a CSR of more than 2^31 - 1 entries (papers100M: 3.2G) is sorted in
// row chunks of at most 2^30 entries (+ one row), each with offsets relative to its start.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <vector>

#include "common.cuh"

namespace cmb {
namespace {

__global__ void k_iota_keys(const int32_t* __restrict__ comm, int64_t n, uint32_t* key,
                            int32_t* val) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    key[i] = static_cast<uint32_t>(comm[i]);
    val[i] = static_cast<int32_t>(i);
  }
}

__global__ void k_inv_deg(const int32_t* __restrict__ perm, const int64_t* __restrict__ indptr,
                          const int32_t* __restrict__ comm, int64_t n, int32_t* inv, int64_t* deg,
                          int32_t* comm_out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i == n) {
      deg[n] = 0;
      continue;
    }
    const int32_t v = perm[i];
    inv[v] = static_cast<int32_t>(i);
    deg[i] = indptr[v + 1] - indptr[v];
    comm_out[i] = comm[v];
  }
}

// one warp per new row: old row perm[i] renamed through inv
__global__ void k_copy_rows(const int32_t* __restrict__ perm, const int64_t* __restrict__ indptr,
                            const int32_t* __restrict__ indices, const int32_t* __restrict__ inv,
                            const int64_t* __restrict__ indptr_out, int64_t n, int32_t* out) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int32_t v = perm[i];
    const int64_t b = indptr[v], d = indptr[v + 1] - b, o = indptr_out[i];
    for (int64_t k = lane; k < d; k += 32) out[o + k] = __ldg(inv + __ldg(indices + b + k));
  }
}

// c-th chunk boundary (c = 1 .. nchunks-1): the first row whose start offset is >= c * 2^30
__global__ void k_split_rows(const int64_t* __restrict__ indptr, int64_t n, int nchunks,
                             int64_t* __restrict__ split) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nchunks + 1) return;
  if (c == 0) { split[0] = 0; split[nchunks + 1] = indptr[0]; return; }
  if (c == nchunks) { split[nchunks] = n; split[2 * nchunks + 1] = indptr[n]; return; }
  const int64_t target = static_cast<int64_t>(c) << 30;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (indptr[mid] < target) lo = mid + 1; else hi = mid;
  }
  split[c] = lo;
  split[nchunks + 1 + c] = indptr[lo];
}

// offsets of a chunk relative to its first entry
struct MinusBase {
  int64_t base;
  __host__ __device__ int64_t operator()(int64_t x) const { return x - base; }
};

constexpr int64_t kSortChunk = int64_t{1} << 30;

struct ReorderWs {
  uint32_t *k0, *k1;
  int32_t *v0;
  int64_t* deg;
  int32_t* tmp;  // unsorted renamed rows
  int64_t* split;  // [2 * (nchunks + 1)] chunk start rows, then their start offsets
  void* temp;
  size_t temp_bytes;
};

ReorderWs carve_reorder_ws(void* base, int64_t n, int64_t nnz, size_t* bytes) {
  Carver c(base);
  ReorderWs w;
  w.k0 = c.take<uint32_t>(n);
  w.k1 = c.take<uint32_t>(n);
  w.v0 = c.take<int32_t>(n);
  w.deg = c.take<int64_t>(n + 1);
  w.tmp = c.take<int32_t>(nnz > 0 ? nnz : 1);
  const int64_t nchunks = nnz > INT32_MAX ? (nnz + kSortChunk - 1) / kSortChunk : 1;
  w.split = c.take<int64_t>(2 * (nchunks + 1));
  size_t a = 0, b = 0, d = 0;
  const int ni = static_cast<int>(n);
  cub::DeviceRadixSort::SortPairs(nullptr, a, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (int32_t*)nullptr, (int32_t*)nullptr, ni);
  cub::DeviceScan::ExclusiveSum(nullptr, b, (int64_t*)nullptr, (int64_t*)nullptr, ni + 1);
  // one chunk holds at most 2^30 entries plus one row (< 2^31 for any row shorter than 2^30)
  const int64_t items = nnz > INT32_MAX ? kSortChunk + (kSortChunk - 1) : nnz;
  cub::DeviceSegmentedSort::SortKeys(
      nullptr, d, (int32_t*)nullptr, (int32_t*)nullptr, static_cast<int>(items), ni,
      cub::TransformInputIterator<int64_t, MinusBase, const int64_t*>(nullptr, MinusBase{0}),
      cub::TransformInputIterator<int64_t, MinusBase, const int64_t*>(nullptr, MinusBase{0}));
  w.temp_bytes = a > b ? a : b;
  if (d > w.temp_bytes) w.temp_bytes = d;
  w.temp = c.take<char>(w.temp_bytes);
  if (bytes) *bytes = c.bytes();
  return w;
}

int bits_for_u32(uint32_t x) {
  int b = 1;
  while (b < 32 && (x >> b)) ++b;
  return b;
}

}  // namespace
}  // namespace cmb

using namespace cmb;

extern "C" {

size_t cmb_community_order_workspace_bytes(int64_t num_nodes, int64_t nnz) {
  if (num_nodes < 1 || num_nodes > INT32_MAX || nnz < 0) return 0;
  size_t b = 0;
  carve_reorder_ws(nullptr, num_nodes, nnz, &b);
  return b;
}

cmb_status cmb_community_order(const int64_t* indptr, const int32_t* indices,
                               const int32_t* community, int64_t num_nodes, int64_t nnz,
                               int32_t num_communities, int32_t* perm, int32_t* inv,
                               int64_t* indptr_out, int32_t* indices_out, int32_t* community_out,
                               void* workspace, size_t workspace_bytes, void* stream) {
  CMB_NVTX("cmb.next2.community_order");
  CMB_ARG(indptr && community && perm && inv && indptr_out && community_out &&
              (nnz == 0 || (indices && indices_out)),
          "cmb_community_order: null argument");
  CMB_ARG(num_nodes >= 1 && num_nodes <= INT32_MAX && nnz >= 0 && num_communities >= 1,
          "cmb_community_order: num_nodes outside [1, 2^31) or nnz < 0");
  const size_t need = cmb_community_order_workspace_bytes(num_nodes, nnz);
  CMB_ARG(workspace && workspace_bytes >= need &&
              (reinterpret_cast<uintptr_t>(workspace) & 255) == 0,
          "cmb_community_order: workspace must be 256-B aligned and >= %zu bytes", need);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ReorderWs w = carve_reorder_ws(workspace, num_nodes, nnz, nullptr);
  int dev = 0, sms = 148;
  CMB_CUDA(cudaGetDevice(&dev));
  CMB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int grid = sms * 4, blk = 256;
  const int ni = static_cast<int>(num_nodes);
  k_iota_keys<<<grid, blk, 0, s>>>(community, num_nodes, w.k0, w.v0);
  CMB_CUDA(cudaGetLastError());
  size_t tb = w.temp_bytes;
  CMB_CUDA(cub::DeviceRadixSort::SortPairs(w.temp, tb, w.k0, w.k1, w.v0, perm, ni, 0,
                                           bits_for_u32(static_cast<uint32_t>(num_communities)),
                                           s));
  k_inv_deg<<<grid, blk, 0, s>>>(perm, indptr, community, num_nodes, inv, w.deg, community_out);
  CMB_CUDA(cudaGetLastError());
  tb = w.temp_bytes;
  CMB_CUDA(cub::DeviceScan::ExclusiveSum(w.temp, tb, w.deg, indptr_out, ni + 1, s));
  if (nnz > 0) {
    k_copy_rows<<<sms * 8, blk, 0, s>>>(perm, indptr, indices, inv, indptr_out, num_nodes, w.tmp);
    CMB_CUDA(cudaGetLastError());
    using It = cub::TransformInputIterator<int64_t, MinusBase, const int64_t*>;
    if (nnz <= INT32_MAX) {
      tb = w.temp_bytes;
      CMB_CUDA(cub::DeviceSegmentedSort::SortKeys(w.temp, tb, w.tmp, indices_out,
                                                  static_cast<int>(nnz), ni, It(indptr_out, {0}),
                                                  It(indptr_out + 1, {0}), s));
    } else {  // row chunks of <= 2^30 entries (+ one row): the split rows are read back once
      const int nchunks = static_cast<int>((nnz + kSortChunk - 1) / kSortChunk);
      k_split_rows<<<(nchunks + 1 + 255) / 256, 256, 0, s>>>(indptr_out, num_nodes, nchunks,
                                                             w.split);
      CMB_CUDA(cudaGetLastError());
      std::vector<int64_t> sp(2 * (nchunks + 1));
      CMB_CUDA(cudaMemcpyAsync(sp.data(), w.split, sp.size() * sizeof(int64_t),
                               cudaMemcpyDeviceToHost, s));
      CMB_CUDA(cudaStreamSynchronize(s));
      for (int c = 0; c < nchunks; ++c) {
        const int64_t r0 = sp[c], r1 = sp[c + 1];
        const int64_t o0 = sp[nchunks + 1 + c], o1 = sp[nchunks + 2 + c];
        if (r1 <= r0 || o1 <= o0) continue;
        CMB_ARG(o1 - o0 <= INT32_MAX, "cmb_community_order: a row of more than 2^30 entries");
        tb = w.temp_bytes;
        CMB_CUDA(cub::DeviceSegmentedSort::SortKeys(
            w.temp, tb, w.tmp + o0, indices_out + o0, static_cast<int>(o1 - o0),
            static_cast<int>(r1 - r0), It(indptr_out + r0, MinusBase{o0}),
            It(indptr_out + r0 + 1, MinusBase{o0}), s));
      }
    }
  }
  return CMB_OK;
}

}  // extern "C"
