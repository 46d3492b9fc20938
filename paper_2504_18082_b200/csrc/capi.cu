// capi.cu -- error plumbing, status queries and capacity helpers of the cmb C ABI.
#include <cstdarg>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"

namespace cmb {

static thread_local char g_msg[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_msg, sizeof(g_msg), fmt, ap);
  va_end(ap);
}

cmb_status cuda_fail(cudaError_t e, const char* what) {
  set_error("%s: %s", what, cudaGetErrorString(e));
  return CMB_ERR_CUDA;
}

cmb_status require_sm100() {
  int dev = 0;
  CMB_CUDA(cudaGetDevice(&dev));
  int major = 0;
  CMB_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  if (major != 10) {
    set_error("device %d has compute capability %d.x; this library is built for sm_100a (B200)",
              dev, major);
    return CMB_ERR_UNSUPPORTED_DEVICE;
  }
  return CMB_OK;
}

cmb_status ensure_dyn_smem(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;  // (kernel, device) -> bytes set
  int dev = 0;
  CMB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  size_t& have = done[{kernel, dev}];
  if (have < bytes) {
    CMB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(bytes)));
    have = bytes;
  }
  return CMB_OK;
}

}  // namespace cmb

extern "C" {

const char* cmb_last_error_message(void) { return cmb::g_msg; }

const char* cmb_status_string(cmb_status s) {
  switch (s) {
    case CMB_OK: return "CMB_OK";
    case CMB_ERR_INVALID_ARGUMENT: return "CMB_ERR_INVALID_ARGUMENT";
    case CMB_ERR_INVALID_GRAPH: return "CMB_ERR_INVALID_GRAPH";
    case CMB_ERR_NOT_COMMUNITY_ORDERED: return "CMB_ERR_NOT_COMMUNITY_ORDERED";
    case CMB_ERR_CAPACITY: return "CMB_ERR_CAPACITY";
    case CMB_ERR_CUDA: return "CMB_ERR_CUDA";
    case CMB_ERR_UNSUPPORTED_DEVICE: return "CMB_ERR_UNSUPPORTED_DEVICE";
    case CMB_ERR_INVALID_INPUT: return "CMB_ERR_INVALID_INPUT";
  }
  return "CMB_ERR_UNKNOWN";
}

int cmb_version(void) { return CMB_VERSION_MAJOR * 100 + CMB_VERSION_MINOR; }

cmb_status cmb_get_device_status(void* workspace, void* stream) {
  CMB_ARG(workspace != nullptr, "cmb_get_device_status: null workspace");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int32_t st = 0;
  CMB_CUDA(cudaMemcpyAsync(&st, workspace, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  CMB_CUDA(cudaStreamSynchronize(s));
  if (st != 0) {
    CMB_CUDA(cudaMemsetAsync(workspace, 0, sizeof(int32_t), s));
    CMB_CUDA(cudaStreamSynchronize(s));
    cmb::set_error("device-side status %d (%s)", st, cmb_status_string((cmb_status)st));
  }
  return static_cast<cmb_status>(st);
}

void cmb_blocks_capacity(int64_t n_roots, const int32_t* fanouts, int32_t n_hops,
                         int64_t num_nodes, int64_t* n_cap, int64_t* e_cap) {
  int64_t n = n_roots < num_nodes ? n_roots : num_nodes;
  n_cap[0] = n;
  for (int32_t h = 0; h < n_hops; ++h) {
    int64_t e = n * static_cast<int64_t>(fanouts[h]);
    e_cap[h] = e;
    int64_t nn = n + e;
    n = nn < num_nodes ? nn : num_nodes;
    n_cap[h + 1] = n;
  }
}

}  // extern "C"
