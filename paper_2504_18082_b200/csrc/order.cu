// order.cu -- a1: Knob-1 root ordering, once per epoch (Table 1, PAPER.md P:731-734;
// S4.1 P:653-680; readings R9, R10, R11 in DESIGN.md).
//
//   RAND   : train sorted by (key(v), v)              key(v)  = Philox(0, v, 2<<24, epoch).lo64
//   NORAND : train unchanged (static across epochs)
//   COMM(k): C_tr communities of the train set shuffled as blocks (sorted by (ckey, c),
//            ckey(c) = Philox(0, c, 3<<24, epoch).lo64), grouped into super-blocks of
//            S = max(1, floor(k*C_tr + 0.5)) consecutive shuffled communities, nodes
//            sorted by (super-block, key(v), v).
//
// B200 mapping: a few elementwise kernels plus stable LSD radix sorts (CUB DeviceRadixSort,
// the one library primitive used; n_train <= ~1.2M, once per epoch, not on the per-batch
// path).  Every tie-break falls out of stability: the input is ascending in v.
#include <cub/cub.cuh>

#include "common.cuh"

namespace cmb {
namespace {

__global__ void k_root_keys(const int32_t* __restrict__ train, int64_t n, int64_t num_nodes,
                            uint64_t seed, uint32_t epoch, uint64_t* __restrict__ keys,
                            int32_t* __restrict__ vals, int32_t* status) {
  const uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = train[i];
    if ((i > 0 && train[i - 1] >= v) || v < 0 || v >= num_nodes)
      raise_status(status, CMB_ERR_INVALID_INPUT);
    keys[i] = lo64(philox4x32_10(0u, static_cast<uint32_t>(v), kTagRoot << 24, epoch, k0, k1));
    vals[i] = static_cast<int32_t>(i);  // train position; ascending -> ties keep v order
  }
}

// community of train id v; an id outside [0, N) (already flagged by k_root_keys) reads node 0
__device__ __forceinline__ int32_t comm_of(const int32_t* __restrict__ comm, int32_t v,
                                           int64_t num_nodes) {
  return comm[(v >= 0 && v < num_nodes) ? v : 0];
}

// flag[i] = 1 where a new training community starts (train ascending + comm
// non-decreasing => comm[train[i]] non-decreasing).
__global__ void k_comm_flags(const int32_t* __restrict__ train, const int32_t* __restrict__ comm,
                             int64_t n, int64_t num_nodes, int32_t* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    flag[i] = (i == 0 || comm_of(comm, train[i], num_nodes) !=
                             comm_of(comm, train[i - 1], num_nodes)) ? 1 : 0;
  }
}

__global__ void k_comm_pad(int32_t ncomm, uint64_t* __restrict__ ckey, int32_t* __restrict__ cval) {
  for (int32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < ncomm; j += gridDim.x * blockDim.x) {
    ckey[j] = ~0ull;  // entries >= C_tr sort last (stable: after every real key)
    cval[j] = j;
  }
}

__global__ void k_comm_keys(const int32_t* __restrict__ train, const int32_t* __restrict__ comm,
                            const int32_t* __restrict__ flag, const int32_t* __restrict__ cpos,
                            int64_t n, int64_t num_nodes, uint64_t seed, uint32_t epoch,
                            uint64_t* __restrict__ ckey) {
  const uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (!flag[i]) continue;
    const int32_t c = comm_of(comm, train[i], num_nodes);
    ckey[cpos[i] - 1] = lo64(philox4x32_10(0u, static_cast<uint32_t>(c), kTagComm << 24, epoch,
                                           k0, k1));
  }
}

// super-block id of the community at shuffled rank r: r / S, S = max(1, floor(k*C_tr + .5))
__global__ void k_comm_superblock(const int32_t* __restrict__ cval_sorted,
                                  const int32_t* __restrict__ cpos, int64_t n, double mix,
                                  int32_t ncomm, uint32_t* __restrict__ sb_of_j) {
  const int64_t c_tr = cpos[n - 1];
  int64_t S = static_cast<int64_t>(__dadd_rn(__dmul_rn(mix, static_cast<double>(c_tr)), 0.5));
  if (S < 1) S = 1;
  for (int32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < ncomm && r < c_tr;
       r += gridDim.x * blockDim.x) {
    sb_of_j[cval_sorted[r]] = static_cast<uint32_t>(r / S);
  }
}

// static adjacent super-blocks (mode 3): one Philox key per super-block b < nsb (slot 1 of the
// community stream), padded with ~0 up to ncomm so the sort length is host-known
__global__ void k_static_sb_keys(const int32_t* __restrict__ cpos, int64_t n, double mix,
                                 int32_t ncomm, uint64_t seed, uint32_t epoch,
                                 uint64_t* __restrict__ key, int32_t* __restrict__ val) {
  const int64_t c_tr = cpos[n - 1];
  int64_t S = static_cast<int64_t>(__dadd_rn(__dmul_rn(mix, static_cast<double>(c_tr)), 0.5));
  if (S < 1) S = 1;
  const int64_t nsb = (c_tr + S - 1) / S;
  const uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
  for (int32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < ncomm; b += gridDim.x * blockDim.x) {
    key[b] = b < nsb ? lo64(philox4x32_10(1u, static_cast<uint32_t>(b), kTagComm << 24, epoch, k0,
                                          k1))
                     : ~0ull;
    val[b] = b;
  }
}

// sb_of_j[j] = rank of super-block j / S in the shuffled super-block order
__global__ void k_static_superblock(const int32_t* __restrict__ b_sorted,
                                    const int32_t* __restrict__ cpos, int64_t n, double mix,
                                    int32_t ncomm, uint32_t* __restrict__ ord,
                                    uint32_t* __restrict__ sb_of_j) {
  const int64_t c_tr = cpos[n - 1];
  int64_t S = static_cast<int64_t>(__dadd_rn(__dmul_rn(mix, static_cast<double>(c_tr)), 0.5));
  if (S < 1) S = 1;
  const int64_t nsb = (c_tr + S - 1) / S;
  // single block: ranks first, then the per-community lookup
  for (int32_t r = threadIdx.x; r < nsb; r += blockDim.x) ord[b_sorted[r]] = static_cast<uint32_t>(r);
  __syncthreads();
  for (int32_t j = threadIdx.x; j < ncomm && j < c_tr; j += blockDim.x)
    sb_of_j[j] = ord[j / S];
}

__global__ void k_node_superblock(const int32_t* __restrict__ pos_sorted,
                                  const int32_t* __restrict__ cpos,
                                  const uint32_t* __restrict__ sb_of_j, int64_t n,
                                  uint32_t* __restrict__ sbk) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    sbk[t] = sb_of_j[cpos[pos_sorted[t]] - 1];
  }
}

__global__ void k_emit(const int32_t* __restrict__ train, const int32_t* __restrict__ pos,
                       int64_t n, int32_t* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    out[t] = train[pos[t]];
  }
}

struct OrderWs {
  WsHeader* hdr;
  uint64_t *k0, *k1, *ck0, *ck1;
  int32_t *v0, *v1, *v2, *cpos, *flag, *cv0, *cv1;
  uint32_t *sbk, *sbk_out, *sb_of_j;
  void* temp;
  size_t temp_bytes;
};

size_t cub_temp_bytes(int64_t n, int32_t ncomm) {
  size_t a = 0, b = 0, c = 0, d = 0;
  const int ni = static_cast<int>(n);
  cub::DeviceRadixSort::SortPairs(nullptr, a, (uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (int32_t*)nullptr, (int32_t*)nullptr, ni);
  cub::DeviceRadixSort::SortPairs(nullptr, b, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (int32_t*)nullptr, (int32_t*)nullptr, ni);
  cub::DeviceRadixSort::SortPairs(nullptr, c, (uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (int32_t*)nullptr, (int32_t*)nullptr, static_cast<int>(ncomm));
  cub::DeviceScan::InclusiveSum(nullptr, d, (int32_t*)nullptr, (int32_t*)nullptr, ni);
  size_t m = a;
  if (b > m) m = b;
  if (c > m) m = c;
  if (d > m) m = d;
  return m;
}

OrderWs carve_order_ws(void* base, int64_t n, int32_t ncomm, size_t* bytes) {
  Carver c(base);
  OrderWs w;
  const size_t N = static_cast<size_t>(n), C = static_cast<size_t>(ncomm);
  w.hdr = c.take<WsHeader>(1);
  w.k0 = c.take<uint64_t>(N);
  w.k1 = c.take<uint64_t>(N);
  w.v0 = c.take<int32_t>(N);
  w.v1 = c.take<int32_t>(N);
  w.v2 = c.take<int32_t>(N);
  w.cpos = c.take<int32_t>(N);
  w.flag = c.take<int32_t>(N);
  w.sbk = c.take<uint32_t>(N);
  w.sbk_out = c.take<uint32_t>(N);
  w.ck0 = c.take<uint64_t>(C);
  w.ck1 = c.take<uint64_t>(C);
  w.cv0 = c.take<int32_t>(C);
  w.cv1 = c.take<int32_t>(C);
  w.sb_of_j = c.take<uint32_t>(C);
  w.temp_bytes = cub_temp_bytes(n, ncomm);
  w.temp = c.take<char>(w.temp_bytes);
  if (bytes) *bytes = c.bytes();
  return w;
}

int bits_for(int64_t maxval) {
  int b = 1;
  while (b < 32 && (int64_t(1) << b) <= maxval) ++b;
  return b;
}

}  // namespace
}  // namespace cmb

using namespace cmb;

extern "C" {

size_t cmb_order_roots_workspace_bytes(int64_t n_train, int32_t num_communities) {
  size_t b = 0;
  carve_order_ws(nullptr, n_train, num_communities, &b);
  return b;
}

cmb_status cmb_order_roots(const cmb_graph* g, const int32_t* train_ids, int64_t n_train,
                           cmb_roots_mode mode, double mix_fraction, uint64_t seed, uint32_t epoch,
                           int32_t* out_order, void* workspace, size_t workspace_bytes,
                           void* stream) {
  CMB_NVTX("cmb.a1.order_roots");
  CMB_ARG(g && train_ids && out_order, "cmb_order_roots: null graph/train_ids/out_order");
  CMB_ARG(n_train >= 1 && n_train <= g->d.n, "cmb_order_roots: n_train %lld outside [1, N]",
          (long long)n_train);
  CMB_ARG(mode == CMB_ROOTS_RAND || mode == CMB_ROOTS_NORAND || mode == CMB_ROOTS_COMM ||
              mode == CMB_ROOTS_COMM_STATIC,
          "cmb_order_roots: unknown mode %d", (int)mode);
  CMB_ARG(mix_fraction >= 0.0 && mix_fraction <= 1.0, "cmb_order_roots: mix_fraction outside [0,1]");
  const size_t need = cmb_order_roots_workspace_bytes(n_train, g->d.ncomm);
  CMB_ARG(workspace && workspace_bytes >= need && (reinterpret_cast<uintptr_t>(workspace) & 255) == 0,
          "cmb_order_roots: workspace must be 256-B aligned and >= %zu bytes", need);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (mode == CMB_ROOTS_NORAND) {
    CMB_CUDA(cudaMemcpyAsync(out_order, train_ids, sizeof(int32_t) * n_train,
                             cudaMemcpyDeviceToDevice, s));
    return CMB_OK;
  }
  OrderWs w = carve_order_ws(workspace, n_train, g->d.ncomm, nullptr);
  const int grid = g->num_sms * 4, blk = 256;
  const int ni = static_cast<int>(n_train);
  size_t tb = w.temp_bytes;
  k_root_keys<<<grid, blk, 0, s>>>(train_ids, n_train, g->d.n, seed, epoch, w.k0, w.v0,
                                   &w.hdr->status);
  CMB_CUDA(cudaGetLastError());
  // sort train positions by key(v) (stable: equal keys keep ascending v)
  CMB_CUDA(cub::DeviceRadixSort::SortPairs(w.temp, tb, w.k0, w.k1, w.v0, w.v1, ni, 0, 64, s));
  const int32_t* pos = w.v1;
  if (mode == CMB_ROOTS_COMM || mode == CMB_ROOTS_COMM_STATIC) {
    const int32_t C = g->d.ncomm;
    k_comm_flags<<<grid, blk, 0, s>>>(train_ids, g->d.comm, n_train, g->d.n, w.flag);
    CMB_CUDA(cudaGetLastError());
    tb = w.temp_bytes;
    CMB_CUDA(cub::DeviceScan::InclusiveSum(w.temp, tb, w.flag, w.cpos, ni, s));
    if (mode == CMB_ROOTS_COMM) {
      k_comm_pad<<<ceil_div(C, blk), blk, 0, s>>>(C, w.ck0, w.cv0);
      k_comm_keys<<<grid, blk, 0, s>>>(train_ids, g->d.comm, w.flag, w.cpos, n_train, g->d.n,
                                       seed, epoch, w.ck0);
      CMB_CUDA(cudaGetLastError());
      tb = w.temp_bytes;
      CMB_CUDA(
          cub::DeviceRadixSort::SortPairs(w.temp, tb, w.ck0, w.ck1, w.cv0, w.cv1, C, 0, 64, s));
      k_comm_superblock<<<ceil_div(C, blk), blk, 0, s>>>(w.cv1, w.cpos, n_train, mix_fraction, C,
                                                         w.sb_of_j);
    } else {
      k_static_sb_keys<<<ceil_div(C, blk), blk, 0, s>>>(w.cpos, n_train, mix_fraction, C, seed,
                                                        epoch, w.ck0, w.cv0);
      CMB_CUDA(cudaGetLastError());
      tb = w.temp_bytes;
      CMB_CUDA(
          cub::DeviceRadixSort::SortPairs(w.temp, tb, w.ck0, w.ck1, w.cv0, w.cv1, C, 0, 64, s));
      k_static_superblock<<<1, 1024, 0, s>>>(w.cv1, w.cpos, n_train, mix_fraction, C,
                                             reinterpret_cast<uint32_t*>(w.cv0), w.sb_of_j);
    }
    k_node_superblock<<<grid, blk, 0, s>>>(w.v1, w.cpos, w.sb_of_j, n_train, w.sbk);
    CMB_CUDA(cudaGetLastError());
    tb = w.temp_bytes;
    CMB_CUDA(cub::DeviceRadixSort::SortPairs(w.temp, tb, w.sbk, w.sbk_out, w.v1, w.v2, ni, 0,
                                             bits_for(C), s));
    pos = w.v2;
  }
  k_emit<<<grid, blk, 0, s>>>(train_ids, pos, n_train, out_order);
  CMB_CUDA(cudaGetLastError());
  return CMB_OK;
}

}  // extern "C"
