// common.cuh -- shared device/host helpers of the cmb CUDA library (sm_100a).
// Product code only: nothing here is shared with oracle/ (see DESIGN.md).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "cmb.h"

namespace cmb {

// ---------------------------------------------------------------- errors
void set_error(const char* fmt, ...);
cmb_status cuda_fail(cudaError_t e, const char* what);
cmb_status require_sm100();
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is a per-device setting: applied once per
// (kernel, current device) pair, thread-safe (capi.cu).
cmb_status ensure_dyn_smem(const void* kernel, size_t bytes);
#define CMB_SMEM(kernel, bytes)                                                             \
  do {                                                                                      \
    const cmb_status st_ = ::cmb::ensure_dyn_smem(reinterpret_cast<const void*>(kernel),    \
                                                  static_cast<size_t>(bytes));              \
    if (st_ != CMB_OK) return st_;                                                          \
  } while (0)

#define CMB_CUDA(call)                                        \
  do {                                                        \
    cudaError_t e_ = (call);                                  \
    if (e_ != cudaSuccess) return ::cmb::cuda_fail(e_, #call); \
  } while (0)

#define CMB_ARG(cond, ...)                         \
  do {                                             \
    if (!(cond)) {                                 \
      ::cmb::set_error(__VA_ARGS__);               \
      return CMB_ERR_INVALID_ARGUMENT;             \
    }                                              \
  } while (0)

// Sticky device status word (first 4 bytes of every workspace header).
struct WsHeader {
  int32_t status;
  int32_t pad[63];
};
static_assert(sizeof(WsHeader) == 256, "header is one 256-byte line");

__device__ __forceinline__ void raise_status(int32_t* st, int32_t code) {
  atomicCAS(st, 0, code);  // first error wins
}

// ---------------------------------------------------------------- tracing
// NVTX range around every entry point of the path (host enqueue span of one stage; nsys / ncu
// --nvtx show them per stage).  Header-only NVTX3: a no-op unless a tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define CMB_NVTX(name) ::cmb::NvtxRange cmb_nvtx_range_(name)

// ---------------------------------------------------------------- workspace carving
struct Carver {
  char* base;
  size_t off = 0;
  explicit Carver(void* b) : base(static_cast<char*>(b)) {}
  template <class T>
  T* take(size_t n) {
    off = (off + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += n * sizeof(T);
    return p;
  }
  size_t bytes() const { return (off + 255) & ~size_t(255); }
};

// ---------------------------------------------------------------- Philox4x32-10
// Salmon et al., SC'11.  Written independently of oracle/oracle.c.
struct PhiloxOut {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ PhiloxOut philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2,
                                                   uint32_t c3, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t a = 0xD2511F53u * c0;
    const uint32_t ah = __umulhi(0xD2511F53u, c0);
    const uint32_t b = 0xCD9E8D57u * c2;
    const uint32_t bh = __umulhi(0xCD9E8D57u, c2);
    const uint32_t n0 = bh ^ c1 ^ k0;
    const uint32_t n2 = ah ^ c3 ^ k1;
    c0 = n0;
    c1 = b;
    c2 = n2;
    c3 = a;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return PhiloxOut{c0, c1, c2, c3};
}

enum : uint32_t { kTagSample = 1u, kTagRoot = 2u, kTagComm = 3u };

__device__ __forceinline__ uint64_t lo64(const PhiloxOut& w) {
  return (static_cast<uint64_t>(w.y) << 32) | w.x;
}
__device__ __forceinline__ uint64_t hi64(const PhiloxOut& w) {
  return (static_cast<uint64_t>(w.w) << 32) | w.z;
}

// Graph as seen by kernels.
constexpr uint32_t kRecDegSlow = 0xFFFFFFu;  // row record degree field: "read indptr / bounds"
struct DevGraph {
  int64_t n;
  int64_t nnz;
  const int64_t* indptr;
  const int32_t* indices;
  const int32_t* comm;
  int32_t ncomm;
  const int32_t* cbeg;   // [C+1]
  const uint2* bounds;   // [N] (lo, hi) row offsets of the intra segment
  const uint4* rec;      // [N] or NULL: packed row record (graph.cu k_intra_bounds): row start,
                         // degree and intra segment of v in ONE 16-byte load
  const float* x;
  int32_t f;
  int64_t ld;
};

inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

// byte offset of element (row r, column c of half h) in a K-major SWIZZLE_128B bf16 operand image
// (the tcgen05 canonical layout) whose 128-byte-wide atoms hold `rows` rows each (atom = h*kh +
// c/64; 8-row groups 1 KB apart; 16-byte chunk j of row r stored at chunk j ^ (r & 7)).  Used by
// the layer kernels, the weight packer and the fused Adam + repack.
__host__ __device__ inline uint32_t sw128_off(int r, int h, int c, int kh, int rows) {
  const int atom = h * kh + (c >> 6);
  const int j = (c & 63) >> 3;
  return static_cast<uint32_t>(atom) * rows * 128u + (r >> 3) * 1024 + (r & 7) * 128 +
         ((j ^ (r & 7)) << 4) + ((c & 7) << 1);
}

}  // namespace cmb

struct cmb_graph {
  cmb::DevGraph d;
  int32_t* status;  // graph workspace header
  int device;
  int num_sms;
};
